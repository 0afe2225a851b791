# configs C5-like on the visible GPUs: 500M keys, global batch 262144, Zipf 1.1 and 1.3
N=$(python -c "import torch; print(torch.cuda.device_count())")
B=$((262144 / N))
for z in 1.1 1.3; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus $N --steps 8 --warmup 3 --no-e2e --vocab 500000000 --batch $B --zipf $z > gpurun_out/c5_z$z.log 2>&1; echo c5 z$z rc=$?
  grep '^{' gpurun_out/c5_z$z.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 z', $z, d['n_gpus'], round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()}, round(d['unique_keys_per_step']))"
done
