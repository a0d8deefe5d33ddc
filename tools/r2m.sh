#!/bin/bash
# round-2 evidence (split screen scan): parity suite, smoke, BASELINE configs, reference arm, ncu
# launch list and --set full captures of the hot kernels at the bench shape (one GPU)
O=gpurun_out/r2m; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 900 python bench.py --per-step --trace-out $O/trace_cfg3.txt --report-dir $O/report_cfg3 > $O/bench_cfg3.log 2> $O/bench_cfg3.err
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/link_probe.cu -o $O/link_probe && timeout 300 $O/link_probe > $O/link_probe.txt 2>&1
S="python bench.py --steps 10 --warmup 3 --burn-in 16 --no-cpu-baseline --no-e2e"
for g in 4 8 16 32; do for v in 0 1 2 3; do
  NOSA_GATHER_CTAS=$g NOSA_GATHER_VARIANT=$v timeout 600 $S > $O/sweep_g${g}_v${v}.log 2>&1
done; done
NOSA_ATTEND_LAYERS=1 timeout 600 $S > $O/sweep_att1.log 2>&1
timeout 600 $S --gather tma > $O/sweep_tma.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py --workload cfg2 --report-dir $O/report_cfg2 > $O/bench_cfg2.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
B="python bench.py --steps 3 --warmup 3 --burn-in 2 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_cfg3.csv $B > $O/launches_cfg3.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_cfg2.csv $B --workload cfg2 --eager > $O/launches_cfg2.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:screen_scan -s 3 -c 1 -o $O/prof3_scan -f $B > $O/ncu3_scan.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:select_plan -s 3 -c 1 -o $O/prof3_select -f $B > $O/ncu3_select.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:attend_bf16 -s 1 -c 1 -o $O/prof3_attend -f $B > $O/ncu3_attend.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:finalize -s 1 -c 1 -o $O/prof3_finalize -f $B > $O/ncu3_finalize.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:select_plan -s 3 -c 1 -o $O/prof2_select -f $B --workload cfg2 --eager > $O/ncu2_select.log 2>&1
for W in cfg1 cfg4; do timeout 900 python bench.py --workload $W --report-dir $O/report_$W > $O/bench_$W.log 2>&1; done
timeout 900 python bench.py --workload cfg4 --selector infllmv2 --no-cpu-baseline --report-dir $O/report_cfg4_infllmv2 > $O/bench_cfg4_infllmv2.log 2>&1
timeout 1200 python bench.py --workload cfg5 --no-cpu-baseline > $O/bench_cfg5.log 2>&1
timeout 900 python bench.py --inputs hidden --no-cpu-baseline > $O/bench_cfg3_hidden.log 2>&1
