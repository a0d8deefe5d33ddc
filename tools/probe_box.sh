#!/bin/bash
# One-off hardware probe of the GPU box: host RAM, cores, NUMA, PCIe link, H2D bandwidth.
set -x
mkdir -p gpurun_out
{
nvidia-smi
nvidia-smi topo -m
nvidia-smi -q | grep -i -A3 -E "pcie gen|link width" | head -40
free -g
nproc
lscpu | head -30
cat /sys/fs/cgroup/memory.max 2>/dev/null
ulimit -l
numactl -H 2>/dev/null
python - <<'PY'
import torch, time
torch.cuda.init()
x = torch.empty(1<<30, dtype=torch.uint8, pin_memory=True)
y = torch.empty(1<<30, dtype=torch.uint8, device='cuda')
for i in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
best = 0
for i in range(10):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); y.copy_(x, non_blocking=True); e.record(); e.synchronize()
    best=max(best,(1<<30)/s.elapsed_time(e)/1e6)
print("H2D pinned 1GiB best GB/s", best)
best=0
for i in range(10):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); x.copy_(y, non_blocking=True); e.record(); e.synchronize()
    best=max(best,(1<<30)/s.elapsed_time(e)/1e6)
print("D2H pinned 1GiB best GB/s", best)
# pin time for big buffers
for gb in (8, 32):
    t=time.time(); z = torch.empty(gb<<30, dtype=torch.uint8, pin_memory=True); print("pin", gb, "GB s", time.time()-t); del z
PY
} > gpurun_out/probe.txt 2>&1
