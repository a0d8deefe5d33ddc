mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -p no:cacheprovider -k "capacity or full" > gpurun_out/cap_tests.log 2>&1; echo rc=$? >> gpurun_out/cap_tests.log
bash tools/sanitize.sh
