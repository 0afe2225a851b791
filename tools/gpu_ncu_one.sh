# ncu --set full of the first launch of each named kernel in one bench step
# (bash tools/gpu_ncu_one.sh <tag> <kernel regex> [<kernel regex> ...])
T=$1; shift
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --pool 1 --no-e2e --no-cpu-baseline"
for k in "$@"; do
  timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"^$k" -s 0 -c 1 -o gpurun_out/full_${T}_$k $B > gpurun_out/ncu_full_${T}_$k.log 2>&1; echo $k rc=$?
done
