mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -k "h3" -q -p no:cacheprovider --timeout=60 > gpurun_out/pytest_h3.log 2>&1; echo h3 rc=$?; tail -1 gpurun_out/pytest_h3.log
B="python bench.py --steps 1 --warmup 1 --pool 1 --no-e2e --no-cpu-baseline"
for bn in 0 256; do
KP_H3_BN=$bn timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:"^k_h3" --clock-control none -c 20 --csv --log-file gpurun_out/bn_$bn.csv $B > /dev/null 2>&1; echo bn $bn rc=$?
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/bn_$bn.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows[-8:]: print(r[4][:40], r[-3][:30], r[-1])
PY
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
