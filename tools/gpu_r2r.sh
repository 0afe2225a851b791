mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --vocab 1000000 --dim 8 --slots 26 --batch 4096 --hidden 64,32 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo c1 rc=$?
tail -1 gpurun_out/bench_c1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],3), d['gpu_launches'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo default rc=$?
tail -1 gpurun_out/bench_default.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['cpu_baseline'], d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-1500
