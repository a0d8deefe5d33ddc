#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3_co.log 2>&1
NOSA_NO_CARVEOUT=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3_nco.log 2>&1
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_co.log 2>&1
NOSA_NO_CARVEOUT=1 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_nco.log 2>&1
