#!/bin/bash
# gather-path experiments + tests + default bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
ARGS="--batch 128 --layers 4 --context 32768 --cache 0.25 --steps 6"
timeout 300 python tools/profile_step.py $ARGS > gpurun_out/sweep_uva_8.txt 2>&1
NOSA_GATHER_CTAS=4 timeout 300 python tools/profile_step.py $ARGS > gpurun_out/sweep_uva_4.txt 2>&1
timeout 300 python tools/profile_step.py $ARGS --gather tma > gpurun_out/sweep_tma_24.txt 2>&1
NOSA_GATHER_CTAS=48 timeout 300 python tools/profile_step.py $ARGS --gather tma > gpurun_out/sweep_tma_48.txt 2>&1
timeout 300 python tools/profile_step.py $ARGS --gather memcpy > gpurun_out/sweep_memcpy.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
