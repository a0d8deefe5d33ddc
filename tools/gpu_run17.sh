#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "peer" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --slow-tier peer --no-cpu-baseline > gpurun_out/bench_peer_148.log 2>&1
NOSA_GATHER_VARIANT=1 timeout 900 python bench.py --slow-tier peer --no-cpu-baseline --no-e2e > gpurun_out/bench_peer_148v1.log 2>&1
NOSA_GATHER_CTAS=296 timeout 900 python bench.py --slow-tier peer --no-cpu-baseline --no-e2e > gpurun_out/bench_peer_296.log 2>&1
