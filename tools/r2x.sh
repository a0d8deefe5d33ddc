#!/bin/bash
# screen scan with the row bounds prefetched: parity suite, cfg 2 / cfg 3, ncu of the scan
O=gpurun_out/r2x; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
S="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $S --workload cfg2 > $O/cfg2.log 2>&1
timeout 600 $S > $O/cfg3.log 2>&1
A3="python tools/profile_step.py --batch 128 --layers 2 --context 32768 --cache 0.25 --steps 5"
A2="python tools/profile_step.py --batch 32 --layers 28 --context 16384 --cache 1 --steps 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:screen_scan -s 4 -c 1 -o $O/prof3_screen_scan -f $A3 > $O/ncu3_scan.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:screen_scan -s 6 -c 1 -o $O/prof2_screen_scan -f $A2 > $O/ncu2_scan.log 2>&1
