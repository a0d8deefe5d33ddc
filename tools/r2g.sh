mkdir -p gpurun_out/san
for tool in synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_projection.py -q -x -p no:cacheprovider > gpurun_out/san/proj_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san/proj_$tool.txt
done
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_kv_manager.py -q -x -p no:cacheprovider -k "not fuzz" > gpurun_out/san/mgr_synccheck.txt 2>&1
echo "rc=$?" >> gpurun_out/san/mgr_synccheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_kv_manager.py -q -x -p no:cacheprovider -k "not fuzz" > gpurun_out/san/mgr_racecheck.txt 2>&1
echo "rc=$?" >> gpurun_out/san/mgr_racecheck.txt
timeout 900 python tools/make_gpu_traces.py gpurun_out/traces > gpurun_out/traces.log 2>&1; echo rc=$? >> gpurun_out/traces.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -k "shard or headline or full_head or compat or engine_vs_reference or shared_pool" > gpurun_out/gpu_subset.log 2>&1; echo rc=$? >> gpurun_out/gpu_subset.log
for n in 1 2 4; do
  NOSA_ATTEND_LAYERS=$n timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg3_al$n.log 2>&1
done
for n in 4 7 14; do
  NOSA_ATTEND_LAYERS=$n timeout 600 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 > gpurun_out/bench_cfg2_al$n.log 2>&1
done
