#!/bin/bash
# tests + timing profile + the default bench (+ ncu of the hot kernels) on one GPU box
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/profile_step.py --batch 128 --layers 2 --context 32768 --cache 0.25 --steps 6 > gpurun_out/prof_offload.txt 2>&1
if [ "$1" == "full" ]; then
  timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
fi
if [ "$2" == "ncu" ]; then
  ARGS="--batch 128 --layers 2 --context 32768 --cache 0.25 --steps 5"
  for K in attend_bf16 select_plan finalize gather_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 \
      -o gpurun_out/prof_$K -f python tools/profile_step.py $ARGS > gpurun_out/ncu_${K}_stdout.txt 2>&1
  done
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/profile_step.py $ARGS > gpurun_out/ncu_launches_stdout.txt 2>&1
fi
