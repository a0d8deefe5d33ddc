#!/bin/bash
# compute-sanitizer over the fp32 warp-group attention kernel (both QK forms: golden engine_small,
# the 1B-shaped multi-layer test) and the custom-eviction-policy manager path
O=gpurun_out/san_f32; mkdir -p $O
SUB='(test_engine_vs_reference_golden and fp32 and engine_small and not infllmv2) or test_fp32_multilayer_batched_attention'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_engine.py -q -x -p no:cacheprovider -k "$SUB" > $O/f32_$tool.txt 2>&1
  echo "rc=$?" >> $O/f32_$tool.txt
done
for tool in memcheck racecheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_kv_manager.py -q -x -p no:cacheprovider -k "policy" > $O/mgr_$tool.txt 2>&1
  echo "rc=$?" >> $O/mgr_$tool.txt
done
