#!/bin/bash
# e2e input staging at cfg 3: SM zero-copy staging vs copy-engine copies per selection group (the
# copy engine is idle now that the SM gather moves the misses); eager steps, two alternations
O=gpurun_out/r2ab; mkdir -p $O
S="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eager"
for rep in 1 2; do
  timeout 900 $S > $O/sm_$rep.log 2>&1
  NOSA_STAGE_COPIES=1 timeout 900 $S > $O/ce_$rep.log 2>&1
done
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/graph.log 2>&1
