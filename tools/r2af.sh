#!/bin/bash
# ncu PCIe counters of the miss gather (cfg 3 shape, 2 layers): bytes read over PCIe per launch and
# the link throughput, next to the kernel time; the attention launches alongside for HBM
O=gpurun_out/r2af; mkdir -p $O
A3="python tools/profile_step.py --batch 128 --layers 2 --context 32768 --cache 0.25 --steps 8"
M=gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,syslts__t_sector_throughput_aperture_sysmem.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -k regex:"gather_kernel|attend_bf16" --csv --log-file $O/pcie_cfg3.csv $A3 > $O/pcie_cfg3.log 2>&1
