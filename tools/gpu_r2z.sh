mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --pool 1 --no-e2e --no-cpu-baseline"
for cfg in "KP_GEMM_CG=2" "KP_GEMM_CG=1" "KP_GEMM_PRE=0" "KP_GEMM_F16=0"; do
env $cfg timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum -k regex:"^k_tc_gemm|^k_split|^k_reduce|^k_transpose|^k_head|^k_loss|^k_colsum" --clock-control none -c 40 --csv --log-file gpurun_out/l2.csv $B > /dev/null 2>&1; echo "$cfg rc=$?"
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/l2.csv')) if len(r)>10 and r[0].isdigit()]
tot=0
for r in rows[-20:]:
    print('   ', r[4][:50], r[-1]); tot+=float(r[-1])
print('   total', tot)
PY
done
