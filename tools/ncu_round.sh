#!/bin/bash
# ncu --set full of every hot kernel at the bench shapes (one GPU, short commands), reports under gpurun_out/
mkdir -p gpurun_out
A3="--batch 128 --layers 2 --context 32768 --cache 0.25 --steps 5 --gather memcpy"
for K in attend_bf16 select_plan finalize; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 \
    -o gpurun_out/prof3_$K -f python tools/profile_step.py $A3 > gpurun_out/ncu3_${K}.txt 2>&1
done
A2="--batch 32 --layers 4 --context 16384 --cache 1 --steps 5"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_bf16 -s 3 -c 1 \
  -o gpurun_out/prof2_attend_bf16 -f python tools/profile_step.py $A2 > gpurun_out/ncu2_attend.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:project_gemm -s 6 -c 1 \
  -o gpurun_out/prof_project -f python tools/proj_bench.py > gpurun_out/ncu_proj.txt 2>&1
