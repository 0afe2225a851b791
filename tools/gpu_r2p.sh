mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -k "h3" -q -p no:cacheprovider --timeout=60 > gpurun_out/pytest_h3.log 2>&1; echo h3 rc=$?; tail -2 gpurun_out/pytest_h3.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider --timeout=900 > gpurun_out/pytest_multi.log 2>&1; echo multi rc=$?; tail -2 gpurun_out/pytest_multi.log
