#!/bin/bash
# fp32 warp-group attention kernel: parity (engine / compat / manager tests), cfg 2 and cfg 1 in
# fp32 storage against the one-warp kernel (NOSA_F32_WARP=1)
O=gpurun_out/r2ai; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compat_traces.py tests/test_gpu_kv_manager.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 600 python bench.py --workload cfg2 --dtype fp32 --no-e2e > $O/bench_cfg2_fp32.log 2>&1
NOSA_F32_WARP=1 timeout 600 python bench.py --workload cfg2 --dtype fp32 --no-e2e --no-cpu-baseline > $O/bench_cfg2_fp32_warp.log 2>&1
timeout 600 python bench.py --workload cfg1 --dtype fp32 --no-e2e > $O/bench_cfg1_fp32.log 2>&1
