#!/bin/bash
# gather variants sweep (4 layers, steady state after burn-in inside profile_step) + bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "gather or golden" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
ARGS="--batch 128 --layers 4 --context 32768 --cache 0.25 --steps 12"
for V in 0 1 2 3; do
  for C in 8 12; do
    NOSA_GATHER_VARIANT=$V NOSA_GATHER_CTAS=$C timeout 300 python tools/profile_step.py $ARGS > gpurun_out/sweep_v${V}_c${C}.txt 2>&1
  done
done
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
