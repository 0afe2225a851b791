mkdir -p gpurun_out
PYTHONPATH=.:tests timeout 100 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -s -k "fused_pool and 96" 2>&1 | grep -E "map_rows|passed|failed|^E " | head
for d in 0 3 4; do
KP_H3_DBG=$d PYTHONPATH=.:tests timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum -k regex:"^k_h3" --clock-control none -c 4 --csv --log-file gpurun_out/ga$d.csv python tools/ga_time.py > /dev/null 2>&1; echo "dbg=$d rc=$?"
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/ga$d.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows[-4:]: print('   ', r[4][:40], r[-1])
PY
done
