#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --graph > gpurun_out/bench_full_graph.log 2>&1; echo rc=$? >> gpurun_out/bench_full_graph.log
timeout 900 python bench.py --workload cfg2 --graph --no-cpu-baseline > gpurun_out/bench_cfg2_graph.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg2_graph.log
