#!/bin/bash
O=gpurun_out/r2s; mkdir -p $O
S="python bench.py --steps 6 --warmup 3 --burn-in 16 --no-cpu-baseline --no-e2e"
NOSA_HOST_SHARE=0.4 timeout 600 $S --gather hybrid --trace-out $O/trace_hybrid.txt > $O/hybrid.log 2>&1
NOSA_HOST_SHARE=1.0 timeout 600 $S --gather hybrid --trace-out $O/trace_hybrid1.txt > $O/hybrid1.log 2>&1
NOSA_HOST_SHARE=0.0 timeout 600 $S --gather hybrid --trace-out $O/trace_hybrid0.txt > $O/hybrid0.log 2>&1
