#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg2.log
timeout 900 python bench.py --gather uva --no-cpu-baseline > gpurun_out/bench_full_uva.log 2>&1; echo rc=$? >> gpurun_out/bench_full_uva.log
