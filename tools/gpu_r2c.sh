mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -k "h3" -v -s -p no:cacheprovider > gpurun_out/pytest_h3.log 2>&1; echo h3 rc=$?
grep -E "PASS|FAIL|passed|failed|err=|Error|error" gpurun_out/pytest_h3.log | tail -30
timeout 600 python -m pytest tests/test_gpu_configs.py -v -s -p no:cacheprovider -x > gpurun_out/pytest_configs.log 2>&1; echo configs rc=$?
grep -E "PASS|FAIL|passed|failed|dloss|scaled|Error" gpurun_out/pytest_configs.log | tail -30
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()}, d['loss'], d['roofline']['frac'])"
tail -5 gpurun_out/bench.log
