#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3_s$i.log 2>&1
NOSA_EXACT_SCAN=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3_x$i.log 2>&1
done
