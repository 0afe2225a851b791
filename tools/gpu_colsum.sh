mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_cs.log 2>&1; echo t rc=$?; tail -3 gpurun_out/pytest_cs.log
C1="--batch 4096 --slots 26 --dim 8 --vocab 1000000 --hidden 64,32"
for i in 1 2; do
for f in 1 0; do
KP_COLSUM_FUSE=$f timeout 600 python bench.py --steps 30 --warmup 3 $C1 --no-cpu-baseline > gpurun_out/c1c$f.log 2>&1
grep '^{' gpurun_out/c1c$f.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 cf=$f', round(d['value']), round(d['e2e']['value']), d['gpu_launches'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
done
