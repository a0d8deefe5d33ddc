#!/bin/bash
# compute-sanitizer over a reduced parity subset (SMALL configs, the three movers, graph and
# host-step replays, the tcgen05 projection, the device-resident block manager)
mkdir -p gpurun_out/san
SUB='test_engine_vs_reference_golden and engine_small and not infllmv2 or test_gather_paths_and_schedules_bitwise_identical or test_host_step_graph_replay_matches_eager or test_graph_replay_matches_eager or test_ragged_batch_and_partial_tails or test_peer_slow_tier_loopback'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_engine.py -q -x -p no:cacheprovider -k "$SUB" > gpurun_out/san/engine_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san/engine_$tool.txt
done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_projection.py tests/test_gpu_kv_manager.py -q -x -p no:cacheprovider -k "not fuzz" > gpurun_out/san/proj_mgr_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san/proj_mgr_$tool.txt
done
