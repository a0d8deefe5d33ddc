#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e --trace-out gpurun_out/tl_cfg2.txt > gpurun_out/bench_cfg2.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --trace-out gpurun_out/tl_cfg3.txt > gpurun_out/bench_cfg3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
  python bench.py --workload cfg2 --steps 2 --warmup 1 --burn-in 4 --no-cpu-baseline --no-e2e --eager > gpurun_out/ncu_launches_stdout.txt 2>&1
