#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --gather memcpy --no-cpu-baseline > gpurun_out/bench_full_memcpy.log 2>&1; echo rc=$? >> gpurun_out/bench_full_memcpy.log
timeout 900 python bench.py --workload cfg2 --graph --no-cpu-baseline > gpurun_out/bench_cfg2_graph.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg2_graph.log
timeout 900 python bench.py --graph --no-cpu-baseline > gpurun_out/bench_full_graph.log 2>&1; echo rc=$? >> gpurun_out/bench_full_graph.log
timeout 900 python bench.py --schedule serial --no-cpu-baseline > gpurun_out/bench_full_serial.log 2>&1; echo rc=$? >> gpurun_out/bench_full_serial.log
