#!/bin/bash
O=gpurun_out/r2p; mkdir -p $O
nproc > $O/host.txt; lscpu | head -30 >> $O/host.txt; numactl -H >> $O/host.txt 2>&1; nvidia-smi topo -m >> $O/host.txt 2>&1
nvcc -O3 -std=c++17 -Xcompiler -fopenmp -gencode arch=compute_100a,code=sm_100a tools/mover_probe.cu -o $O/mover_probe -lpthread -lgomp
timeout 300 $O/mover_probe 4 > $O/mover_probe4.txt 2>&1
GPU_NODE=$(cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | tr 'A-F' 'a-f' | sed 's/^0000//; s/^/0000/' | cut -c1-12)/numa_node 2>/dev/null)
echo "gpu numa node: $GPU_NODE" >> $O/host.txt
if [ -n "$GPU_NODE" ] && [ "$GPU_NODE" -ge 0 ]; then timeout 300 numactl --cpunodebind=$GPU_NODE --membind=$GPU_NODE $O/mover_probe 4 > $O/mover_probe4_numa.txt 2>&1; fi
timeout 900 python bench.py --workload cfg2 --per-step --trace-out $O/trace_cfg2.txt --no-cpu-baseline > $O/bench_cfg2.log 2>&1
