mkdir -p gpurun_out
C1="--batch 4096 --slots 26 --dim 8 --vocab 1000000 --hidden 64,32"
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/c1_launches.csv python bench.py $C1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc=$?
