mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_parity.py -k "h3" -q -s -p no:cacheprovider --timeout=60 > gpurun_out/pytest_h3.log 2>&1; echo h3 rc=$?
grep -E "FAIL|passed|failed|Timeout|err=" gpurun_out/pytest_h3.log | tail -20
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()}, d['loss'], d['roofline']['frac'])"
timeout 600 bash tools/gpu_launches.sh r02c
