#!/bin/bash
# cfg 2 value and e2e by selection-group plan: the first attention batch's group staged and
# selected in smaller pieces (the host step stages inputs per group)
O=gpurun_out/r2az; mkdir -p $O
S="python bench.py --workload cfg2 --no-cpu-baseline"
for rep in 1 2; do
  timeout 600 $S > $O/default_$rep.log 2>&1
  NOSA_SELECT_PLAN=2,2,4,16,4 timeout 600 $S > $O/p22416_$rep.log 2>&1
  NOSA_SELECT_PLAN=1,3,4,16,4 timeout 600 $S > $O/p13416_$rep.log 2>&1
done
