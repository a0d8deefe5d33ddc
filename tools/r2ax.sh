#!/bin/bash
# bf16 kernel A/B on one box: QK MMA chain split over two accumulators (default build) vs one
# (tools/bin/libnosa_bfbase.so), cfg 2 (HBM-bound); bf16 parity subset on the new build
O=gpurun_out/r2ax; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compat_traces.py -q -x -p no:cacheprovider -k "bf16 or bitwise" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
S="python bench.py --workload cfg2 --no-e2e --no-cpu-baseline"
for rep in 1 2 3; do
  NOSA_B200_LIB=tools/bin/libnosa_bfbase.so timeout 600 $S > $O/base_$rep.log 2>&1
  timeout 600 $S > $O/new_$rep.log 2>&1
done
