#!/bin/bash
# mover alternatives (graph memcpy nodes, threaded memcpy, interference) + ncu of the hot kernels at
# the cfg 3 shape (2 layers: the 28-layer pinned pool is too large for ncu's replay)
O=gpurun_out/r2n; mkdir -p $O
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/mover_probe.cu -o $O/mover_probe -lpthread && timeout 600 $O/mover_probe > $O/mover_probe.txt 2>&1
A3="python tools/profile_step.py --batch 128 --layers 2 --context 32768 --cache 0.25 --steps 5"
for K in screen_scan select_plan attend_bf16 finalize gather_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 -o $O/prof3_$K -f $A3 > $O/ncu3_$K.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_cfg3_2l.csv $A3 > $O/launches_cfg3_2l.log 2>&1
