mkdir -p gpurun_out
B="python bench.py --vocab 1000000 --dim 8 --slots 26 --batch 4096 --hidden 64,32 --steps 1 --warmup 2 --pool 1 --no-e2e --no-cpu-baseline"
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv $B > /dev/null 2>&1; echo c1 launches rc=$?
