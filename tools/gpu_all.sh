#!/bin/bash
# every BASELINE config through bench.py + the reference arm + parity tests + smoke
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg3.log 2>&1
for W in cfg1 cfg2 cfg4; do timeout 900 python bench.py --workload $W > gpurun_out/bench_$W.log 2>&1; done
timeout 900 python bench.py --workload cfg4 --selector infllmv2 --no-cpu-baseline > gpurun_out/bench_cfg4_infllmv2.log 2>&1
timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1
