mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1; echo ref rc=$?
bash tools/gpu_launches.sh r02f
