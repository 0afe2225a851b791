mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
