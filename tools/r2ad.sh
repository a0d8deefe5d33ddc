#!/bin/bash
# compute-sanitizer over the parity subset with this round's final code: SM gather (one grid per
# attention batch, L2::256B), host-pack and hybrid movers, fused selection, fp32 projection
O=gpurun_out/san2; mkdir -p $O
SUB='test_engine_vs_reference_golden and engine_small and not infllmv2 or test_ragged_batch_and_partial_tails or test_host_step_graph_replay_matches_eager or test_other_gather_paths_vs_oracle or test_peer_slow_tier_loopback or test_resident_multilayer_batched_attention'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1800 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_engine.py -q -x -p no:cacheprovider -k "$SUB" > $O/engine_$tool.txt 2>&1
  echo "rc=$?" >> $O/engine_$tool.txt
done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_projection.py tests/test_gpu_kv_manager.py -q -x -p no:cacheprovider -k "not fuzz" > $O/proj_mgr_$tool.txt 2>&1
  echo "rc=$?" >> $O/proj_mgr_$tool.txt
done
