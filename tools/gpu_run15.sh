#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "bitwise or graph or shared or resident" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for P in 0,0,1,1 0,0,0,0 0,0,1,2 0,1,2,3 1,0,0,0; do
NOSA_PRIO=$P timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_p$P.log 2>&1
done
NOSA_PRIO=0,0,1,1 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e --trace-out gpurun_out/tl_cfg2.txt > gpurun_out/bench_cfg2.log 2>&1
NOSA_PRIO=0,0,1,1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3_p0011.log 2>&1
NOSA_PRIO=0,0,0,0 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3_p0000.log 2>&1
