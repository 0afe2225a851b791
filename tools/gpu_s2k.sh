mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -2 gpurun_out/pytest_gpu.log
C1="--batch 4096 --slots 26 --dim 8 --vocab 1000000 --hidden 64,32"
timeout 300 python bench.py $C1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c1.log 2>&1; tail -1 gpurun_out/c1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], {k:round(v['ms_per_step'],4) for k,v in d['stages'].items()})"
bash tools/gpu_ncu_one.sh s2k k_downsweep
