#!/bin/bash
mkdir -p gpurun_out
timeout 300 tools/bin/link_probe > gpurun_out/link_probe.txt 2>&1
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg2.log
timeout 900 python bench.py --workload cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg4.log
