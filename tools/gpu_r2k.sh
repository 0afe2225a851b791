mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -p no:cacheprovider --timeout=300 -x > gpurun_out/pytest_pp.log 2>&1; echo parity rc=$?
grep -E "FAIL|passed|failed|Timeout|Error" gpurun_out/pytest_pp.log | tail -5
for v in 0 1; do
KP_SEG_PRE=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_pre$v.log 2>&1; echo bench $v rc=$?
tail -1 gpurun_out/bench_pre$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
