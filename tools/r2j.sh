mkdir -p gpurun_out/ab2
run() { name=$1; shift; env "$@" timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/ab2/cfg2_$name.log 2>&1; }
run base
run s28 NOSA_SELECT_PLAN=28
run s8_20 NOSA_SELECT_PLAN=8,20
run s4_24_a4 NOSA_SELECT_PLAN=4,24 NOSA_ATTEND_PLAN=4,8,8,8
run s8_20_plo NOSA_SELECT_PLAN=8,20 NOSA_PRIO=1,0,0,0
run s8_8_12_plo NOSA_PRIO=1,0,0,0
run s14_14_a14 NOSA_SELECT_PLAN=14,14 NOSA_ATTEND_PLAN=14,14
run base2
