# 2-GPU: sharded parity suite with the hoisted-load merge kernel, then A/B of
# KP_MERGE_RW (k = 1: a merge every step)
O=gpurun_out/mrw; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_multi.py -v -x > $O/pytest_multi_g2.log 2>&1; echo EXIT $? >> $O/pytest_multi_g2.log
for r in 1 2; do for m in 0 1; do
KP_MERGE_RW=$m timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$m \
  bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_m${m}_$r.log 2>&1
done; done
