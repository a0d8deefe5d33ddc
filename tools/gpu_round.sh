#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg2.log
NOSA_NO_STREAM_PRIORITY=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_full_noprio.log 2>&1; echo rc=$? >> gpurun_out/bench_full_noprio.log
NOSA_NO_STREAM_PRIORITY=1 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2_noprio.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg2_noprio.log
