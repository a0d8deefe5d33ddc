#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python tools/profile_step.py --batch 128 --layers 4 --context 32768 --cache 0.25 --steps 5 --gather memcpy --sel-prof > gpurun_out/selprof3.txt 2>&1
timeout 600 python tools/profile_step.py --batch 32 --layers 4 --context 16384 --cache 1 --steps 5 --sel-prof > gpurun_out/selprof2.txt 2>&1
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1
