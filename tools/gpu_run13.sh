#!/bin/bash
mkdir -p gpurun_out
ARGS="--batch 32 --layers 4 --context 16384 --cache 1 --steps 6"
for K in select_plan attend_bf16; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 6 -c 1 \
  -o gpurun_out/prof_cfg2_$K -f python tools/profile_step.py $ARGS > gpurun_out/ncu_${K}_stdout.txt 2>&1
done
ARGS3="--batch 128 --layers 2 --context 32768 --cache 0.25 --steps 6 --gather memcpy"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_plan -s 4 -c 1 \
  -o gpurun_out/prof_cfg3_select -f python tools/profile_step.py $ARGS3 > gpurun_out/ncu_sel3_stdout.txt 2>&1
