#!/bin/bash
# cfg 2: shorter last attention batches (the step's tail is the last batch's attention + merge)
O=gpurun_out/r2ag; mkdir -p $O
S="python bench.py --workload cfg2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 600 $S > $O/default_$rep.log 2>&1
  NOSA_ATTEND_PLAN=8,8,8,2,2 timeout 600 $S > $O/ap88822_$rep.log 2>&1
  NOSA_ATTEND_PLAN=8,8,8,3,1 timeout 600 $S > $O/ap88831_$rep.log 2>&1
  NOSA_ATTEND_PLAN=8,8,10,2 timeout 600 $S > $O/ap88102_$rep.log 2>&1
done
