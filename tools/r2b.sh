mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_headline.py -x -q -s > gpurun_out/headline.log 2>&1; echo rc=$? >> gpurun_out/headline.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo rc=$? >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
