#!/bin/bash
# cfg 3 in fp32 storage (offloaded; host RAM bounds the batch), with parity and e2e
O=gpurun_out/r2ba; mkdir -p $O
free -g > $O/free.txt
timeout 1200 python bench.py --dtype fp32 > $O/bench_cfg3_fp32.log 2> $O/bench_cfg3_fp32.err
