#!/bin/bash
# cfg 3 in fp32 storage: SM-gather grid and load variant (64 KiB blocks)
O=gpurun_out/r2bb; mkdir -p $O
S="python bench.py --dtype fp32 --no-cpu-baseline --no-e2e"
NOSA_GATHER_CTAS=16 timeout 900 $S > $O/ctas16.log 2>&1
NOSA_GATHER_VARIANT=3 timeout 900 $S > $O/var3.log 2>&1
NOSA_GATHER_CTAS=12 NOSA_GATHER_VARIANT=3 timeout 900 $S > $O/ctas12_var3.log 2>&1
