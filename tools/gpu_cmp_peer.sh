# multi-GPU: parity (peer windows) + bench peer vs NCCL exchange
bash tools/gpu_multi.sh
for pm in 0; do
KP_PEER=$pm timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_peer$pm.log 2>&1; echo peer $pm rc=$?
grep '^{' gpurun_out/bench_peer$pm.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
