#!/bin/bash
# fp32 kernel A/B on one box: one barrier per block (every warp forms all running maxima, probabilities of its own keys; default build) vs two barriers (lanep)

O=gpurun_out/r2aw; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compat_traces.py -q -x -p no:cacheprovider -k fp32 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
S="python bench.py --workload cfg2 --dtype fp32 --no-e2e --no-cpu-baseline"
for rep in 1 2; do
  NOSA_B200_LIB=tools/bin/libnosa_lanep.so timeout 600 $S > $O/lanep_$rep.log 2>&1
  timeout 600 $S > $O/new_$rep.log 2>&1
done
