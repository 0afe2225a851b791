# A/B of an env toggle on the 1-GPU bench: bash tools/gpu_ab.sh VAR val_a val_b
mkdir -p gpurun_out
V=$1; shift
for x in "$@"; do
  env $V=$x timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$x.log 2>&1; echo "$V=$x rc=$?"
  tail -1 gpurun_out/ab_$x.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['loss'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
done
