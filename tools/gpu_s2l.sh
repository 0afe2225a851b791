mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout=200 -x -k "dedup or shard or trainer_det or c2" > gpurun_out/pytest_ds.log 2>&1; echo ds rc=$?; tail -2 gpurun_out/pytest_ds.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum -k regex:"^k_downsweep|^k_upsweep|^k_dedup|^k_scan|^k_head_count|^k_minmax|^k_prepare" --clock-control none -c 14 --csv --log-file gpurun_out/ds.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/ds.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows[-14:]: print('   ', r[4][:50], r[-1])
PY
