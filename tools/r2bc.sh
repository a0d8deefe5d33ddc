#!/bin/bash
# gather defaults by block size: fp32 parity subset, cfg 3 fp32 (new defaults, parity + e2e), cfg 3 bf16 (unchanged defaults)
O=gpurun_out/r2bc; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_headline.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 1200 python bench.py --dtype fp32 > $O/bench_cfg3_fp32.log 2> $O/bench_cfg3_fp32.err
timeout 900 python bench.py > $O/bench_cfg3.log 2>&1
