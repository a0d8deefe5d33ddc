mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/gpu_tests_h.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_h.log
timeout 300 python tools/profile_step.py --batch 128 --layers 4 --context 32768 --cache 0.25 --steps 4 --sel-prof > gpurun_out/selprof_cfg3.txt 2>&1
timeout 300 python tools/profile_step.py --batch 32 --layers 4 --context 16384 --cache 1 --steps 4 --sel-prof > gpurun_out/selprof_cfg2.txt 2>&1
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2_h.log 2>&1
timeout 900 python bench.py --per-step > gpurun_out/bench_cfg3_h.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_kv_manager.py -q -x -p no:cacheprovider -k "not fuzz" > gpurun_out/san/mgr_racecheck_h.txt 2>&1
echo "rc=$?" >> gpurun_out/san/mgr_racecheck_h.txt
for t in memcheck racecheck; do
timeout 900 compute-sanitizer --tool $t --print-limit 30 --error-exitcode 99 \
    python -m pytest tests/test_gpu_engine.py -q -x -p no:cacheprovider -k "engine_vs_reference_golden and engine_small or capacity or full_head or shared_pool" > gpurun_out/san/sel_${t}_h.txt 2>&1
echo "rc=$?" >> gpurun_out/san/sel_${t}_h.txt
done
