mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -k "h3 or tcgen05 or trainer" -q -p no:cacheprovider --timeout=100 > gpurun_out/pytest_h3.log 2>&1; echo h3 rc=$?; tail -1 gpurun_out/pytest_h3.log
timeout 300 python bench.py --vocab 1000000 --dim 8 --slots 26 --batch 4096 --hidden 64,32 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo c1 rc=$?
tail -1 gpurun_out/bench_c1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],3), d['gpu_launches'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
