mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "fused_pool" > gpurun_out/pytest_ga.log 2>&1; echo ga rc=$?; grep -E "^E |passed|failed|Error" gpurun_out/pytest_ga.log | head -20
