mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
B="python bench.py --steps 1 --warmup 1 --pool 1 --no-e2e --no-cpu-baseline"
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:"^k_probe" --clock-control none -c 20 --csv --log-file gpurun_out/probe.csv $B > /dev/null 2>&1; echo probe rc=$?
grep -E "duration|bytes_read" gpurun_out/probe.csv | tail -2 | awk -F'","' '{print $(NF-2), $NF}'
