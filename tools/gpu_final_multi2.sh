# 2-GPU check of the final tree: sharded parity suite + bench (e2e on)
O=gpurun_out/fm2; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_multi.py -v -x > $O/pytest_multi_g2.log 2>&1; echo EXIT $? >> $O/pytest_multi_g2.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > $O/b2.log 2>&1
