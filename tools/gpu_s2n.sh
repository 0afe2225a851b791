mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout=200 -x -k "sync_free" > gpurun_out/pytest_sf.log 2>&1; echo sf rc=$?; grep -E "^E |passed|failed" gpurun_out/pytest_sf.log | head -10
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu_ab2.sh KP_SYNC_FREE
C1="--batch 4096 --slots 26 --dim 8 --vocab 1000000 --hidden 64,32"
timeout 300 python bench.py $C1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c1.log 2>&1; tail -1 gpurun_out/c1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1', round(d['value']), d['ms_per_step'], {k:round(v['ms_per_step'],4) for k,v in d['stages'].items()})"
