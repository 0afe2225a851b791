mkdir -p gpurun_out
for st in 5 20 5; do
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $n --steps $st --warmup 3 > gpurun_out/bench_g${n}_s$st.log 2>&1
grep '^{' gpurun_out/bench_g${n}_s$st.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, $st, round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
done
