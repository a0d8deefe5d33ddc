mkdir -p gpurun_out/ab
for v in v1 v3_256 v3_128; do
  export NOSA_B200_LIB=$PWD/tools/bin/libnosa_$v.so
  timeout 300 python tools/profile_step.py --batch 128 --layers 4 --context 32768 --cache 0.25 --steps 4 --sel-prof > gpurun_out/ab/selprof_cfg3_$v.txt 2>&1
  timeout 300 python tools/profile_step.py --batch 32 --layers 4 --context 16384 --cache 1 --steps 4 --sel-prof > gpurun_out/ab/selprof_cfg2_$v.txt 2>&1
  timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/ab/bench_cfg2_$v.log 2>&1
done
export NOSA_B200_LIB=$PWD/tools/bin/libnosa_v3_128.so
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_headline.py tests/test_gpu_select_manager.py -q -x -p no:cacheprovider > gpurun_out/ab/tests_v3_128.log 2>&1; echo rc=$? >> gpurun_out/ab/tests_v3_128.log
unset NOSA_B200_LIB
for p in "1,7,8,8,4" "2,6,8,8,3,1" "1,3,8,8,7,1" "4,8,8,8"; do
  NOSA_ATTEND_PLAN=$p timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/ab/bench_cfg2_plan_${p//,/_}.log 2>&1
done
