mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_configs.py -v -s -p no:cacheprovider --timeout=300 > gpurun_out/pytest_configs.log 2>&1; echo configs rc=$?
grep -E "PASS|FAIL|passed|failed|dloss|scaled|Error|Timeout" gpurun_out/pytest_configs.log | tail -30
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()}, d['loss'], d['roofline']['frac'])"
tail -3 gpurun_out/bench.log | cut -c1-2000
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=300 --deselect tests/test_gpu_configs.py > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?; grep -E "FAIL|passed|failed|Timeout" gpurun_out/pytest_gpu.log | tail -10
