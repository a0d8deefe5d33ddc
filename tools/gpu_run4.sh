#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "bitwise" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python tools/profile_step.py --batch 32 --layers 28 --context 16384 --cache 1 --steps 4 --trace > gpurun_out/trace_cfg2.txt 2>&1
timeout 600 python tools/profile_step.py --batch 128 --layers 28 --context 32768 --cache 0.25 --steps 4 --gather memcpy --trace > gpurun_out/trace_cfg3.txt 2>&1
