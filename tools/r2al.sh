#!/bin/bash
# fp32 kernel A/B: 8 consumer warps (8 dims per lane) vs 16 (4 dims per lane), cfg 2 fp32
O=gpurun_out/r2al; mkdir -p $O
NOSA_F32_WARPS16=1 timeout 600 python -m pytest tests/test_gpu_engine.py -q -x -p no:cacheprovider -k fp32 > $O/tests16.log 2>&1; echo rc=$? >> $O/tests16.log
S="python bench.py --workload cfg2 --dtype fp32 --no-e2e --no-cpu-baseline"
for rep in 1 2; do
  timeout 600 $S > $O/w8_$rep.log 2>&1
  NOSA_F32_WARPS16=1 timeout 600 $S > $O/w16_$rep.log 2>&1
done
