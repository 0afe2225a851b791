# 4-GPU: sharded parity suite + KP_MERGE_RW A/B at G = 4 (k = 1), then G = 2
O=gpurun_out/mrw4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -v -x > $O/pytest_multi_g4.log 2>&1; echo EXIT $? >> $O/pytest_multi_g4.log
for r in 1 2; do for m in 0 1; do
KP_MERGE_RW=$m timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$m \
  bench.py --gpus 4 --steps 20 --warmup 3 --no-cpu-baseline > $O/b4_m${m}_$r.log 2>&1
done; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > $O/b2_final.log 2>&1
