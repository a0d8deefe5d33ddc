#!/bin/bash
# cfg 3 bf16: SM-gather default (8 CTAs, L2 hint) vs the fp32 setting (12 CTAs, two blocks per iteration)
O=gpurun_out/r2bd; mkdir -p $O
S="python bench.py --no-cpu-baseline"
for rep in 1 2; do
  timeout 900 $S > $O/default_$rep.log 2>&1
  NOSA_GATHER_CTAS=12 NOSA_GATHER_VARIANT=3 timeout 900 $S > $O/c12v3_$rep.log 2>&1
done
