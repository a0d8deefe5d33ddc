#!/bin/bash
# ncu evidence for the hot kernels (one GPU, short command).  Outputs under gpurun_out/.
mkdir -p gpurun_out
ARGS="--batch 128 --layers 2 --context 32768 --cache 0.25 --steps 5"
# plain timing, offload shape and all-resident shape (no concurrent gathers)
python tools/profile_step.py $ARGS > gpurun_out/prof_offload.txt 2>&1
python tools/profile_step.py --batch 128 --layers 2 --context 32768 --cache 1 --steps 5 > gpurun_out/prof_resident.txt 2>&1
# launch list with device times
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python tools/profile_step.py $ARGS > gpurun_out/ncu_launches_stdout.txt 2>&1
# full set on one launch of the attention kernel and of the select kernel (after warm-up)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_bf16 -s 4 -c 1 \
  -o gpurun_out/prof_attend -f python tools/profile_step.py $ARGS > gpurun_out/ncu_attend_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_plan -s 4 -c 1 \
  -o gpurun_out/prof_select -f python tools/profile_step.py $ARGS > gpurun_out/ncu_select_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 4 -c 1 \
  -o gpurun_out/prof_gather -f python tools/profile_step.py $ARGS > gpurun_out/ncu_gather_stdout.txt 2>&1
ls -la gpurun_out
