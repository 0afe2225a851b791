mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_configs.py -v -s -p no:cacheprovider --timeout=600 > gpurun_out/pytest_configs.log 2>&1; echo configs rc=$?
grep -E "PASS|FAIL|passed|failed|dloss|scaled|auc|Error" gpurun_out/pytest_configs.log | tail -50
timeout 1800 python -m pytest tests/test_gpu_multi.py -v -s -p no:cacheprovider --timeout=900 > gpurun_out/pytest_multi.log 2>&1; echo multi rc=$?
grep -E "PASS|FAIL|passed|failed|Error" gpurun_out/pytest_multi.log | tail -30
