#!/bin/bash
# final round-2 evidence on the final code: GPU suite, smoke, every BASELINE config (bf16), cfg 2 /
# cfg 1 in fp32 storage, hidden-state lines, peer tier, reference arm, launch list of the default bench
O=gpurun_out/r2ar; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py --per-step --trace-out $O/trace_cfg3.txt --report-dir $O/report_cfg3 > $O/bench_cfg3.log 2> $O/bench_cfg3.err
timeout 900 python bench.py --workload cfg2 --trace-out $O/trace_cfg2.txt --report-dir $O/report_cfg2 > $O/bench_cfg2.log 2>&1
timeout 900 python bench.py --workload cfg2 --dtype fp32 > $O/bench_cfg2_fp32.log 2>&1
timeout 900 python bench.py --workload cfg1 --dtype fp32 > $O/bench_cfg1_fp32.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
for W in cfg1 cfg4; do timeout 900 python bench.py --workload $W --report-dir $O/report_$W > $O/bench_$W.log 2>&1; done
timeout 900 python bench.py --workload cfg4 --selector infllmv2 --no-cpu-baseline --report-dir $O/report_cfg4_infllmv2 > $O/bench_cfg4_infllmv2.log 2>&1
timeout 1200 python bench.py --workload cfg5 --no-cpu-baseline > $O/bench_cfg5.log 2>&1
timeout 900 python bench.py --inputs hidden --no-cpu-baseline > $O/bench_cfg3_hidden.log 2>&1
timeout 900 python bench.py --workload cfg2 --inputs hidden --no-cpu-baseline > $O/bench_cfg2_hidden.log 2>&1
timeout 900 python bench.py --slow-tier peer --no-cpu-baseline > $O/bench_cfg3_peer.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_cfg2_fp32.csv python bench.py --workload cfg2 --dtype fp32 --eager --steps 3 --warmup 3 --burn-in 2 --no-cpu-baseline --no-e2e > $O/launches_cfg2_fp32.log 2>&1
