mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_fuse.log 2>&1; echo t rc=$?; tail -3 gpurun_out/pytest_fuse.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fuse$i.log 2>&1; echo b rc=$?
grep '^{' gpurun_out/bench_fuse$i.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['gpu_launches'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
KP_SPLIT_FUSE=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nofuse.log 2>&1; echo b rc=$?
grep '^{' gpurun_out/bench_nofuse.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nofuse', round(d['value']), round(d['e2e']['value']), d['gpu_launches'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
C1="--batch 4096 --slots 26 --dim 8 --vocab 1000000 --hidden 64,32"
timeout 600 python bench.py --steps 10 --warmup 3 $C1 --no-cpu-baseline > gpurun_out/c1f.log 2>&1; echo c1 rc=$?
grep '^{' gpurun_out/c1f.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1', round(d['value']), round(d['e2e']['value']), d['gpu_launches'])"
