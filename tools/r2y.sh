#!/bin/bash
# split vs fused screen scan (A/B, two alternations) at cfg 2 and cfg 3; selection phase cycles
# (run when split was the default; with fused the default now, the split arm is NOSA_SPLIT_SCAN=1)
O=gpurun_out/r2y; mkdir -p $O
S="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  NOSA_SPLIT_SCAN=1 timeout 600 $S --workload cfg2 > $O/cfg2_split_$rep.log 2>&1
  timeout 600 $S --workload cfg2 > $O/cfg2_fused_$rep.log 2>&1
done
NOSA_SPLIT_SCAN=1 timeout 600 $S > $O/cfg3_split.log 2>&1
timeout 600 $S > $O/cfg3_fused.log 2>&1
NOSA_SPLIT_SCAN=1 timeout 300 python tools/profile_step.py --batch 32 --layers 8 --context 16384 --cache 1 --steps 4 --sel-prof > $O/selprof_cfg2_split.txt 2>&1
timeout 300 python tools/profile_step.py --batch 32 --layers 8 --context 16384 --cache 1 --steps 4 --sel-prof > $O/selprof_cfg2_fused.txt 2>&1
NOSA_SPLIT_SCAN=1 timeout 300 python tools/profile_step.py --batch 128 --layers 4 --context 32768 --cache 0.25 --steps 4 --sel-prof > $O/selprof_cfg3_split.txt 2>&1
