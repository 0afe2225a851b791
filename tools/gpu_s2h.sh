mkdir -p gpurun_out
for v in "KP_GA_NOSTORE=1 KP_H3_DBG=0" "KP_GA_NOSTORE=1 KP_H3_DBG=4" "KP_GA_NOSTORE=1 KP_H3_DBG=3"; do
env $v PYTHONPATH=.:tests timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum -k regex:"^k_h3" --clock-control none -c 4 --csv --log-file gpurun_out/gax.csv python tools/ga_time.py > /dev/null 2>&1; echo "$v rc=$?"
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/gax.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows[-4:-3]: print('   ', r[4][:40], r[-1])
PY
done
