#!/bin/bash
# gather-path experiments: UVA kernel at several CTA counts vs the copy-engine batch path
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
ARGS="--batch 128 --layers 4 --context 32768 --cache 0.25 --steps 6"
for C in 8 16 32 64; do
  NOSA_GATHER_CTAS=$C timeout 300 python tools/profile_step.py $ARGS > gpurun_out/sweep_uva_$C.txt 2>&1
done
timeout 300 python tools/profile_step.py $ARGS --gather memcpy > gpurun_out/sweep_memcpy.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
timeout 900 python bench.py --gather memcpy --no-cpu-baseline > gpurun_out/bench_full_memcpy.log 2>&1; echo rc=$? >> gpurun_out/bench_full_memcpy.log
