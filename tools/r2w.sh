#!/bin/bash
# fp32 projection + compat tests; staging grid A/B (e2e, cfg 3); refreshed evidence on the final
# movers (gather L2::256B loads): parity suite, smoke, every BASELINE config, reference arm
O=gpurun_out/r2w; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
S="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
for sg in 8 16; do NOSA_STAGE_CTAS=$sg timeout 900 $S > $O/stage$sg.log 2>&1; done
timeout 900 python bench.py --per-step --trace-out $O/trace_cfg3.txt --report-dir $O/report_cfg3 > $O/bench_cfg3.log 2> $O/bench_cfg3.err
timeout 900 python bench.py --workload cfg2 --trace-out $O/trace_cfg2.txt --report-dir $O/report_cfg2 > $O/bench_cfg2.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
for W in cfg1 cfg4; do timeout 900 python bench.py --workload $W --report-dir $O/report_$W > $O/bench_$W.log 2>&1; done
timeout 900 python bench.py --workload cfg4 --selector infllmv2 --no-cpu-baseline --report-dir $O/report_cfg4_infllmv2 > $O/bench_cfg4_infllmv2.log 2>&1
timeout 1200 python bench.py --workload cfg5 --no-cpu-baseline > $O/bench_cfg5.log 2>&1
timeout 900 python bench.py --inputs hidden --no-cpu-baseline > $O/bench_cfg3_hidden.log 2>&1
timeout 900 python bench.py --slow-tier peer --no-cpu-baseline > $O/bench_cfg3_peer.log 2>&1
A3="python tools/profile_step.py --batch 128 --layers 2 --context 32768 --cache 0.25 --steps 5"
for K in screen_scan gather_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 -o $O/prof3_$K -f $A3 > $O/ncu3_$K.log 2>&1
done
