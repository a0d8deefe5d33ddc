#!/bin/bash
# A/B at cfg 3 (20 timed steps, burn-in 32, two alternations): SM gather load variant and grid
# (the host share of the hybrid as one copy-engine copy per block was also measured here:
# 10.5K tok/s at a 10% share, 6.8K at 20%; removed)
O=gpurun_out/r2u; mkdir -p $O
S="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 600 $S > $O/uva_v0_g8_$rep.log 2>&1
  NOSA_GATHER_VARIANT=2 timeout 600 $S > $O/uva_v2_g8_$rep.log 2>&1
  NOSA_GATHER_VARIANT=2 NOSA_GATHER_CTAS=12 timeout 600 $S > $O/uva_v2_g12_$rep.log 2>&1
done
