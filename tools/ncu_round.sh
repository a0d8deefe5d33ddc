#!/bin/bash
# ncu --set full of every hot kernel at the bench shapes (one GPU, short commands), reports under gpurun_out/
mkdir -p gpurun_out
A3="--batch 128 --layers 2 --context 32768 --cache 0.25 --steps 5 --gather memcpy"
for K in attend_bf16 select_plan finalize; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 \
    -o gpurun_out/prof3_$K -f python tools/profile_step.py $A3 > gpurun_out/ncu3_${K}.txt 2>&1
done
# cfg 2: all 28 layers, so the attention launches are the bench's (8 + 8 + 8 + 4 layers); the
# four launches of the second step are captured and their DRAM bytes averaged (traffic.json)
A2="--batch 32 --layers 28 --context 16384 --cache 1 --steps 3"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attend_bf16 -s 4 -c 4 \
  -o gpurun_out/prof2_attend_bf16 -f python tools/profile_step.py $A2 > gpurun_out/ncu2_attend.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:project_gemm -s 6 -c 1 \
  -o gpurun_out/prof_project -f python tools/proj_bench.py > gpurun_out/ncu_proj.txt 2>&1
# launch lists of the headline commands (per-launch device times; shares, not absolutes)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 3 --warmup 3 --burn-in 2 --no-cpu-baseline --no-e2e \
  > gpurun_out/launches_cfg3.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_cfg2.csv python bench.py --workload cfg2 --eager --steps 3 --warmup 3 --burn-in 2 \
  --no-cpu-baseline --no-e2e > gpurun_out/launches_cfg2.log 2>&1
