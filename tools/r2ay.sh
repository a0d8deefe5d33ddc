#!/bin/bash
# closing check of the final tree: GPU suite, smoke, the default bench line and the reference arm
O=gpurun_out/r2ay; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg3.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
