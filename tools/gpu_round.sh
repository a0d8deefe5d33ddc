#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "graph or gather_paths or shared or golden" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg2.log
NOSA_ONE_ATT_STREAM=1 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2_one.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg2_one.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
