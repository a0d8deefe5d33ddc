#!/bin/bash
# cfg 3 fp32: SM-gather grid / variant around the new default (12 CTAs, variant 3)
O=gpurun_out/r2be; mkdir -p $O
S="python bench.py --dtype fp32 --no-cpu-baseline --no-e2e"
NOSA_GATHER_CTAS=16 NOSA_GATHER_VARIANT=3 timeout 900 $S > $O/c16v3.log 2>&1
NOSA_GATHER_CTAS=12 NOSA_GATHER_VARIANT=1 timeout 900 $S > $O/c12v1.log 2>&1
NOSA_GATHER_CTAS=10 NOSA_GATHER_VARIANT=3 timeout 900 $S > $O/c10v3.log 2>&1
