#!/bin/bash
mkdir -p gpurun_out
ARGS="--batch 32 --layers 2 --context 16384 --cache 1 --steps 6"
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for K in attend_bf16 finalize select_plan; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 6 -c 1 \
  -o gpurun_out/prof_cfg2_$K -f python tools/profile_step.py $ARGS > gpurun_out/ncu_${K}_stdout.txt 2>&1
done
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e --trace-out gpurun_out/tl_cfg2.txt > gpurun_out/bench_cfg2.log 2>&1
