# configs C4 (k sweep, 4 GPUs here) and C1 (small model) measurements
mkdir -p gpurun_out
N=$(python -c "import torch; print(torch.cuda.device_count())")
for k in 1 4 16 64; do
  st=$(( k > 8 ? k : 8 )); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus $N --steps $st --warmup 3 --no-e2e --k $k > gpurun_out/sweep_k$k.log 2>&1; echo k $k rc=$?
  grep '^{' gpurun_out/sweep_k$k.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('k', $k, d['n_gpus'], round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
timeout 600 python bench.py --steps 10 --warmup 3 --vocab 1000000 --dim 8 --slots 26 --batch 4096 --hidden 64,32 --no-cpu-baseline > gpurun_out/c1.log 2>&1; echo c1 rc=$?
grep '^{' gpurun_out/c1.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --vocab 1000000 --dim 8 --slots 26 --batch 4096 --hidden 64,32 > gpurun_out/c1_ref.log 2>&1; echo c1ref rc=$?
grep '^{' gpurun_out/c1_ref.log | tail -1 | cut -c1-300
