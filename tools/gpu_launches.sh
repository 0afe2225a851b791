# ncu launch list of one bench step (bash tools/gpu_launches.sh <tag>)
T=${1:-r01}
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --pool 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_$T.log 2>&1; echo plain rc=$?
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$T.csv $B > /dev/null 2>&1; echo launches rc=$?
