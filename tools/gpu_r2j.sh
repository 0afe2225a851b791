mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --pool 1 --no-e2e --no-cpu-baseline"
for d in 0 1 2; do
KP_H3_DBG=$d timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:"^k_h3" --clock-control none -c 20 --csv --log-file gpurun_out/dbg_$d.csv $B > /dev/null 2>&1; echo dbg $d rc=$?
grep k_h3 gpurun_out/dbg_$d.csv | grep duration | tail -3 | cut -c1-40,200-400
done
