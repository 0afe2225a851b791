mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -3 gpurun_out/pytest_gpu.log
C1="--batch 4096 --slots 26 --dim 8 --vocab 1000000 --hidden 64,32"
timeout 300 python bench.py $C1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c1.log 2>&1; tail -1 gpurun_out/c1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], {k:round(v['ms_per_step'],4) for k,v in d['stages'].items()})"
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/c1_launches.csv python bench.py $C1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-stage-profile > /dev/null 2>&1; echo ncu rc=$?
