#!/bin/bash
# hybrid mover (host-packed DMAs + SM gather): parity, share / thread / grid sweep at cfg 3
O=gpurun_out/r2r; mkdir -p $O
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "gather_paths or other_gather" > $O/hp_tests.log 2>&1; echo rc=$? >> $O/hp_tests.log
S="python bench.py --steps 10 --warmup 3 --burn-in 16 --no-cpu-baseline --no-e2e --gather hybrid"
for sh in 0.3 0.4 0.5 0.6; do NOSA_HOST_SHARE=$sh timeout 600 $S > $O/sweep_s${sh}.log 2>&1; done
NOSA_HOST_SHARE=0.4 NOSA_PACK_THREADS=12 timeout 600 $S > $O/sweep_s0.4_t12.log 2>&1
NOSA_HOST_SHARE=0.5 NOSA_PACK_THREADS=12 timeout 600 $S > $O/sweep_s0.5_t12.log 2>&1
NOSA_HOST_SHARE=0.4 NOSA_GATHER_CTAS=6 timeout 600 $S > $O/sweep_s0.4_g6.log 2>&1
NOSA_HOST_SHARE=0.4 NOSA_GATHER_CTAS=12 timeout 600 $S > $O/sweep_s0.4_g12.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --burn-in 16 --no-cpu-baseline --no-e2e > $O/sweep_uva.log 2>&1
