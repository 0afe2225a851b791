mkdir -p gpurun_out
KP_POOL_PP=1 timeout 300 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout=200 -x -k "c2 or pooling or fused" > gpurun_out/pytest_pp.log 2>&1; echo pp rc=$?; tail -2 gpurun_out/pytest_pp.log
bash tools/gpu_ab2.sh KP_POOL_PP
