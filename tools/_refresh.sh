timeout 900 python bench.py --workload cfg5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r_cfg5.json
timeout 900 python bench.py --slow-tier peer --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r_peer.json
timeout 900 python bench.py --workload cfg2 --inputs hidden --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r_cfg2_hidden.json
timeout 900 python bench.py --inputs hidden --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r_cfg3_hidden.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_cfg2.csv python bench.py --workload cfg2 --eager --steps 3 --warmup 3 --burn-in 2 \
  --no-cpu-baseline --no-e2e > gpurun_out/launches_cfg2.log 2>&1
