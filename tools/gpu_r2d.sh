mkdir -p gpurun_out
timeout 60 python -m pytest tests/test_gpu_parity.py -k "h3_gemm_nt_accuracy and 128-128-32" -x -s -p no:cacheprovider > gpurun_out/pytest_h3a.log 2>&1; echo h3a rc=$?
tail -5 gpurun_out/pytest_h3a.log
timeout 240 python -m pytest tests/test_gpu_parity.py -k "h3" -v -s -p no:cacheprovider --timeout=60 > gpurun_out/pytest_h3.log 2>&1; echo h3 rc=$?
grep -E "PASS|FAIL|passed|failed|err=|Error|error|Timeout" gpurun_out/pytest_h3.log | tail -30
