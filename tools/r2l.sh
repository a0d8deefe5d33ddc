O=gpurun_out/ab3; mkdir -p $O
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
for m in split fused split4 split6; do
  unset NOSA_FUSED_SCAN NOSA_B200_LIB
  if [ $m == fused ]; then export NOSA_FUSED_SCAN=1; fi
  if [ $m == split4 ] || [ $m == split6 ]; then export NOSA_B200_LIB=$PWD/tools/bin/libnosa_$m.so; fi
  timeout 300 python tools/profile_step.py --batch 128 --layers 4 --context 32768 --cache 0.25 --steps 4 --sel-prof > $O/selprof_cfg3_$m.txt 2>&1
  timeout 300 python tools/profile_step.py --batch 32 --layers 4 --context 16384 --cache 1 --steps 4 --sel-prof > $O/selprof_cfg2_$m.txt 2>&1
  timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2_$m.log 2>&1
  NOSA_SELECT_PLAN=28 timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2_s28_$m.log 2>&1
  timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg3_$m.log 2>&1
done
unset NOSA_FUSED_SCAN NOSA_B200_LIB
timeout 900 ncu --set full --clock-control none --import-source on -k regex:screen_scan -s 6 -c 1 -o $O/prof_scan -f python tools/profile_step.py --batch 128 --layers 4 --context 32768 --cache 0.25 --steps 4 > $O/ncu_scan.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_plan -s 6 -c 1 -o $O/prof_selplan -f python tools/profile_step.py --batch 128 --layers 4 --context 32768 --cache 0.25 --steps 4 > $O/ncu_selplan.log 2>&1
