for ce in 0 1; do
KP_PEER_CE=$ce timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_ce$ce.log 2>&1; echo ce $ce rc=$?
grep '^{' gpurun_out/bench_ce$ce.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
KP_PEER_CE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29577 tools/mgpu_parity.py /tmp/r.json 1 1 2>&1 | grep "^{" | tail -1 | cut -c1-200
