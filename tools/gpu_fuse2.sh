mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout=300 -x -k "split_rows_colmax or graph_replay or staged" > gpurun_out/pytest_fuse2.log 2>&1; echo t rc=$?; tail -2 gpurun_out/pytest_fuse2.log
for i in 1 2; do
for f in 1 0; do
KP_SPLIT_FUSE=$f timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_f$f.log 2>&1
grep '^{' gpurun_out/bench_f$f.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fuse=$f', round(d['value']), round(d['e2e']['value']), d['gpu_launches'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
done
