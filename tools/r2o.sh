#!/bin/bash
# gather: one grid walks the batch's layers (8 CTAs total); sweep grid / variant / staging grid
O=gpurun_out/r2o; mkdir -p $O
timeout 900 python bench.py --per-step --trace-out $O/trace_cfg3.txt > $O/bench_cfg3.log 2> $O/bench_cfg3.err
S="python bench.py --steps 10 --warmup 3 --burn-in 16 --no-cpu-baseline"
for g in 4 6 8 12; do for v in 0 2; do
  NOSA_GATHER_CTAS=$g NOSA_GATHER_VARIANT=$v timeout 600 $S --no-e2e > $O/sweep_g${g}_v${v}.log 2>&1
done; done
for sg in 4 8 16; do NOSA_STAGE_CTAS=$sg timeout 600 $S > $O/sweep_stage${sg}.log 2>&1; done
timeout 600 $S --no-e2e --gather tma > $O/sweep_tma.log 2>&1
NOSA_GATHER_CTAS=4 timeout 600 $S --no-e2e --gather tma > $O/sweep_tma4.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k "gather or mover or headline or engine" > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
