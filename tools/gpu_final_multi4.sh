# 4-GPU check of the final tree: sharded parity suite + bench (e2e on)
O=gpurun_out/fm4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -v -x > $O/pytest_multi_g4.log 2>&1; echo EXIT $? >> $O/pytest_multi_g4.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 \
  bench.py --gpus 4 --steps 20 --warmup 3 --no-cpu-baseline > $O/b4.log 2>&1
