mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -v -s -p no:cacheprovider --timeout=600 > gpurun_out/pytest_configs.log 2>&1; echo configs rc=$?
grep -E "PASS|FAIL|passed|failed|dloss|scaled|auc" gpurun_out/pytest_configs.log | tail -40
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=300 --deselect tests/test_gpu_configs.py > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?; grep -E "FAIL|passed|failed" gpurun_out/pytest_gpu.log | tail -6
timeout 800 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()}, d['loss'], d['clocks'], d['roofline']['frac'])"
