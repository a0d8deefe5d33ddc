#!/bin/bash
# re-entry verification of HEAD (selection-group doubling, finalize record-count load): parity suite,
# smoke, cfg 3 / cfg 2 / cfg 2 hidden bench lines, reference arm
O=gpurun_out/r2ah; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py --per-step --report-dir $O/report_cfg3 > $O/bench_cfg3.log 2> $O/bench_cfg3.err
timeout 900 python bench.py --workload cfg2 --trace-out $O/trace_cfg2.txt --report-dir $O/report_cfg2 > $O/bench_cfg2.log 2>&1
timeout 900 python bench.py --workload cfg2 --inputs hidden --no-cpu-baseline > $O/bench_cfg2_hidden.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
