mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout=200 -x -k "store or dedup or trainer_det or c2 or sync_free" > gpurun_out/pytest_pr.log 2>&1; echo pr rc=$?; tail -2 gpurun_out/pytest_pr.log
for r in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"; done
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum -k regex:"^k_probe" --clock-control none -c 3 --csv --log-file gpurun_out/probe.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/probe.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows[-3:]: print('   ', r[4][:40], r[-1])
PY
