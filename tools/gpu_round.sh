#!/bin/bash
# tests + a small bench + the default bench on one GPU box; logs under gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/clocks0.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --layers 2 --batch 16 --steps 4 --warmup 3 > gpurun_out/bench_small.log 2>&1; echo rc=$? >> gpurun_out/bench_small.log
if [ "$1" == "full" ]; then
  timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
fi
