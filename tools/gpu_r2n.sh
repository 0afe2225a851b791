mkdir -p gpurun_out
python tools/nvml_probe.py > gpurun_out/nvml_probe.log 2>&1; cat gpurun_out/nvml_probe.log | head -12
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3"
for opt in "" "--no-stage-profile" "--no-e2e" ; do
timeout 600 $R $opt > gpurun_out/bench_g2x.log 2>&1; echo "g2 [$opt] rc=$?"
grep '^{' gpurun_out/bench_g2x.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['wall_ms_per_step'],3), round((d.get('e2e') or {}).get('value') or 0), d['gpu_launches'])"
done
