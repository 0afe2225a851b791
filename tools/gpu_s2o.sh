mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout=200 -x -k "sync_free" > gpurun_out/pytest_sf.log 2>&1; echo sf rc=$?; grep -E "^E |passed|failed" gpurun_out/pytest_sf.log | head -10
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -3 gpurun_out/pytest_gpu.log
