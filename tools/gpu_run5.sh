#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e --trace-out gpurun_out/tl_cfg2.txt > gpurun_out/bench_cfg2.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --trace-out gpurun_out/tl_cfg3.txt > gpurun_out/bench_cfg3.log 2>&1
