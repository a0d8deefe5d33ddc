mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --per-step --trace-out gpurun_out/trace_cfg3.txt > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo rc=$? >> gpurun_out/bench_default.log
NOSA_MEMCPY_READBACK=1 timeout 900 python bench.py --per-step --no-cpu-baseline > gpurun_out/bench_readback.log 2> gpurun_out/bench_readback.err; echo rc=$? >> gpurun_out/bench_readback.log
