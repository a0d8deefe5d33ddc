#!/bin/bash
# ncu of the fp32 warp-group attention kernel at the cfg 2 shape (resident, 2 layers)
O=gpurun_out/r2aj; mkdir -p $O
A="python tools/profile_step.py --batch 32 --layers 2 --context 16384 --cache 1 --steps 4 --dtype fp32"
timeout 300 $A > $O/run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_f32w -s 2 -c 1 -o $O/prof_f32w -f $A > $O/ncu.log 2>&1
