#!/bin/bash
# host-pack mover: parity, cfg 3 bench vs the SM gather, thread / chunk sweep; full GPU suite
O=gpurun_out/r2q; mkdir -p $O
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k "gather_paths or other_gather" > $O/hp_tests.log 2>&1; echo rc=$? >> $O/hp_tests.log
timeout 900 python bench.py --gather hostpack --per-step --trace-out $O/trace_cfg3_hp.txt > $O/bench_cfg3_hp.log 2>&1
S="python bench.py --steps 10 --warmup 3 --burn-in 16 --no-cpu-baseline --no-e2e --gather hostpack"
for t in 4 6 12; do NOSA_PACK_THREADS=$t timeout 600 $S > $O/sweep_t$t.log 2>&1; done
for c in 32 128; do NOSA_PACK_CHUNK=$c timeout 600 $S > $O/sweep_c$c.log 2>&1; done
timeout 900 python bench.py > $O/bench_cfg3_uva.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
