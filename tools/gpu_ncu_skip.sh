# ncu --set full of ONE launch of a kernel, skipping earlier launches of it
# (bash tools/gpu_ncu_skip.sh <tag> <kernel regex> <skip>); e.g. k_probe with
# skip 6 passes the six 16.7M-key prefill chunks of the 100M-key table
T=$1; K=$2; S=${3:-0}
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --pool 1 --no-e2e --no-cpu-baseline"
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"^$K" -s $S -c 1 -o gpurun_out/full_${T}_$K $B > gpurun_out/ncu_full_${T}_$K.log 2>&1; echo $K rc=$?
