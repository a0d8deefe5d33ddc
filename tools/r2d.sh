mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kv_manager.py -x -q > gpurun_out/mgr_tests.log 2>&1; echo rc=$? >> gpurun_out/mgr_tests.log
bash tools/sanitize.sh
