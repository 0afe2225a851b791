# One GPU: bench (both arms) + ncu launch list   (bash tools/profile_round.sh <tag>)
# then per-kernel ncu --set full captures with   (bash tools/profile_round.sh <tag> full)
T=${1:-r01}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 1 --pool 1 --no-e2e --no-cpu-baseline"
if [ "$2" != "full" ]; then
  timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1; echo bench rc=$?
  timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$T.log 2>&1; echo ref rc=$?
  $B > gpurun_out/plain_$T.log 2>&1; echo plain rc=$?
  timeout 900 $NCU --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$T.csv $B > /dev/null 2>&1; echo launches rc=$?
else
  # one launch of each top kernel (the timed step's), full section set
  for k in k_tc_gemm k_seg_chunks k_pool k_downsweep k_probe k_dedup_emit; do
    n=1; [ $k = k_tc_gemm ] && n=6
    timeout 900 $NCU --set full --import-source on --clock-control none -k regex:"^$k" -s 0 -c $n -o gpurun_out/full_${T}_$k $B > gpurun_out/ncu_full_${T}_$k.log 2>&1; echo $k rc=$?
  done
  du -sh gpurun_out
fi
