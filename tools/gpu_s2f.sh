mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "fused_pool" > gpurun_out/pytest_ga.log 2>&1; echo ga rc=$?; grep -E "^E |passed|failed|Error" gpurun_out/pytest_ga.log | head -20
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu_ab2.sh KP_FUSED_POOL
