# multi-GPU round-2 check: sharded parity tests, bench at G = 1,2,4 (+ NVLink counters), k sweep at G=4
mkdir -p gpurun_out
N=$(python -c "import torch; print(torch.cuda.device_count())")
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider --timeout=900 > gpurun_out/pytest_multi.log 2>&1; echo multi rc=$?; tail -1 gpurun_out/pytest_multi.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g1.log 2>&1; echo bench g1 rc=$?
for n in 2 4; do
  [ $n -gt $N ] && continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/bench_g$n.log 2>&1; echo bench g$n rc=$?
  grep '^{' gpurun_out/bench_g$n.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()}, round((d.get('e2e') or {}).get('value') or 0), d['nvlink'])"
done
if [ $N -ge 4 ]; then
for k in 1 4 16 64; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 8 --warmup 3 --k $k --no-e2e > gpurun_out/sweep_k$k.log 2>&1; echo sweep k$k rc=$?
  grep '^{' gpurun_out/sweep_k$k.log | tail -1 > gpurun_out/sweep_k$k.json
done
fi
