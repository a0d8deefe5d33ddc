#!/bin/bash
# fused selection with the pool rows prefetched to L2 (+ unrolled q_sum) vs without (A/B, two
# alternations at cfg 2 and cfg 3), phase cycles, parity suite
O=gpurun_out/r2aa; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
S="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 600 $S --workload cfg2 > $O/cfg2_pf_$rep.log 2>&1
  NOSA_B200_LIB=$PWD/tools/bin/libnosa_nopf.so timeout 600 $S --workload cfg2 > $O/cfg2_nopf_$rep.log 2>&1
done
timeout 600 $S > $O/cfg3_pf.log 2>&1
NOSA_B200_LIB=$PWD/tools/bin/libnosa_nopf.so timeout 600 $S > $O/cfg3_nopf.log 2>&1
timeout 300 python tools/profile_step.py --batch 32 --layers 8 --context 16384 --cache 1 --steps 4 --sel-prof > $O/selprof_cfg2_pf.txt 2>&1
NOSA_B200_LIB=$PWD/tools/bin/libnosa_nopf.so timeout 300 python tools/profile_step.py --batch 32 --layers 8 --context 16384 --cache 1 --steps 4 --sel-prof > $O/selprof_cfg2_nopf.txt 2>&1
