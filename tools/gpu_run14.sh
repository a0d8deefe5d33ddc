#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e --trace-out gpurun_out/tl_cfg2.txt > gpurun_out/bench_cfg2.log 2>&1
NOSA_ONE_ATT_STREAM=1 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_one.log 2>&1
NOSA_NO_STREAM_PRIORITY=1 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_noprio.log 2>&1
NOSA_ATTEND_LAYERS=7 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_l7.log 2>&1
ARGS="--batch 32 --layers 4 --context 16384 --cache 1 --steps 6"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_plan -s 3 -c 1 \
  -o gpurun_out/prof_cfg2_select_plan -f python tools/profile_step.py $ARGS > gpurun_out/ncu_sel_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_bf16 -s 3 -c 1 \
  -o gpurun_out/prof_cfg2_attend_bf16 -f python tools/profile_step.py $ARGS > gpurun_out/ncu_att_stdout.txt 2>&1
