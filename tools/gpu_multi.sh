# multi-GPU check: sharded parity tests + bench at N = number of visible GPUs
mkdir -p gpurun_out
N=$(python -c "import torch; print(torch.cuda.device_count())")
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo multi rc=$?; tail -1 gpurun_out/pytest_multi.log
for n in $(seq 2 $N); do
  [ $n -eq 3 ] && continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench_g$n.log 2>&1; echo bench g$n rc=$?
  grep '^{' gpurun_out/bench_g$n.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()}, round((d.get('e2e') or {}).get('value') or 0))"
done
