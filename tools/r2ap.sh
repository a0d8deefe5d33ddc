#!/bin/bash
# fp32 kernel, next chunk metadata prefetched link by link: parity subset, cfg 2 fp32 x2, ncu
O=gpurun_out/r2ap; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compat_traces.py tests/test_gpu_headline.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
S="python bench.py --workload cfg2 --dtype fp32 --no-e2e"
timeout 600 $S > $O/bench_cfg2_fp32_1.log 2>&1
timeout 600 $S --no-cpu-baseline > $O/bench_cfg2_fp32_2.log 2>&1
A="python tools/profile_step.py --batch 32 --layers 2 --context 16384 --cache 1 --steps 4 --dtype fp32"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_f32w -s 2 -c 1 -o $O/prof_f32w -f $A > $O/ncu.log 2>&1
