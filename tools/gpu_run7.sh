#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --trace-out gpurun_out/tl_cfg2.txt > gpurun_out/bench_cfg2.log 2>&1
NOSA_CHUNK=2 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_c2.log 2>&1
