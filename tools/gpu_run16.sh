#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --slow-tier peer --no-cpu-baseline --trace-out gpurun_out/tl_peer.txt > gpurun_out/bench_peer_memcpy.log 2>&1
timeout 900 python bench.py --slow-tier peer --gather uva --no-cpu-baseline > gpurun_out/bench_peer_uva.log 2>&1
NOSA_GATHER_CTAS=64 timeout 900 python bench.py --slow-tier peer --gather uva --no-cpu-baseline > gpurun_out/bench_peer_uva64.log 2>&1
