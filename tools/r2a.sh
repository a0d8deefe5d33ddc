mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; lscpu > gpurun_out/lscpu.txt; free -g > gpurun_out/free.txt; numactl -H > gpurun_out/numa.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo rc=$? >> gpurun_out/bench_default.log
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1
