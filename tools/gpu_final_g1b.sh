mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1; echo ref rc=$?
C1="--batch 4096 --slots 26 --dim 8 --vocab 1000000 --hidden 64,32"
timeout 600 python bench.py --steps 30 --warmup 3 $C1 --no-cpu-baseline > gpurun_out/c1.log 2>&1; echo c1 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 $C1 > gpurun_out/c1_ref.log 2>&1; echo c1ref rc=$?
bash tools/gpu_launches.sh r02g
