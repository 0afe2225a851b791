mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout=300 -k "trainer or store" > gpurun_out/pytest_p.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/pytest_p.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
