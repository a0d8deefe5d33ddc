#!/bin/bash
# cfg 2: selection group plans (layers per selection launch) and attention batch sizes, 2 alternations
O=gpurun_out/r2ac; mkdir -p $O
S="python bench.py --workload cfg2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 600 $S > $O/default_$rep.log 2>&1
  NOSA_SELECT_PLAN=8,20 timeout 600 $S > $O/sp8_20_$rep.log 2>&1
  NOSA_SELECT_PLAN=8,16,4 timeout 600 $S > $O/sp8_16_4_$rep.log 2>&1
  NOSA_SELECT_PLAN=8,4,4,12 timeout 600 $S > $O/sp8_4_4_12_$rep.log 2>&1
  NOSA_ATTEND_PLAN=8,8,6,6 timeout 600 $S > $O/ap8866_$rep.log 2>&1
  NOSA_ATTEND_PLAN=6,8,8,6 timeout 600 $S > $O/ap6886_$rep.log 2>&1
done
