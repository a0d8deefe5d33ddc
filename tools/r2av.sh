#!/bin/bash
# evidence after the fp32 latency work: GPU suite, smoke, cfg 2 / cfg 1 fp32 lines (parity + e2e),
# cfg 3 default line, ncu of the fp32 kernel, fp32 launch list
O=gpurun_out/r2av; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py --workload cfg2 --dtype fp32 --trace-out $O/trace_cfg2_fp32.txt > $O/bench_cfg2_fp32.log 2>&1
timeout 900 python bench.py --workload cfg1 --dtype fp32 > $O/bench_cfg1_fp32.log 2>&1
timeout 900 python bench.py > $O/bench_cfg3.log 2>&1
A="python tools/profile_step.py --batch 32 --layers 2 --context 16384 --cache 1 --steps 4 --dtype fp32"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_f32w -s 2 -c 1 -o $O/prof_f32w -f $A > $O/ncu.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_cfg2_fp32.csv python bench.py --workload cfg2 --dtype fp32 --eager --steps 3 --warmup 3 --burn-in 2 --no-cpu-baseline --no-e2e > $O/launches_cfg2_fp32.log 2>&1
