#!/bin/bash
# evidence run: ncu of the four kernels + launch list, other BASELINE configs, reference arm
mkdir -p gpurun_out
ARGS="--batch 128 --layers 2 --context 32768 --cache 0.25 --steps 5"
for K in attend_bf16 select_plan finalize gather_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 \
    -o gpurun_out/prof_$K -f python tools/profile_step.py $ARGS > gpurun_out/ncu_${K}_stdout.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --burn-in 4 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_stdout.txt 2>&1
for W in cfg1 cfg2 cfg4; do
  timeout 900 python bench.py --workload $W > gpurun_out/bench_$W.log 2>&1; echo rc=$? >> gpurun_out/bench_$W.log
done
timeout 900 python bench.py --workload cfg4 --selector infllmv2 --no-cpu-baseline > gpurun_out/bench_cfg4_infllmv2.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo rc=$? >> gpurun_out/bench_reference.log
