#!/bin/bash
# fp32 kernel A/B on one box: r2an's kernel (59f2f0c), r2an + the metadata prefetch, HEAD
O=gpurun_out/r2aq; mkdir -p $O
S="python bench.py --workload cfg2 --dtype fp32 --no-e2e --no-cpu-baseline"
for rep in 1 2; do
  NOSA_B200_LIB=tools/bin/libnosa_an.so timeout 600 $S > $O/an_$rep.log 2>&1
  NOSA_B200_LIB=tools/bin/libnosa_apx.so timeout 600 $S > $O/apx_$rep.log 2>&1
  timeout 600 $S > $O/head_$rep.log 2>&1
done
