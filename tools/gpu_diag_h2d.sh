mkdir -p gpurun_out
for i in 1 2; do
for f in "" "--diag-h2d"; do
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $f > gpurun_out/dh.log 2>&1
grep '^{' gpurun_out/dh.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$f]', round(d['value']), round(d['e2e']['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
done
