# NVLink traffic counters around 2-GPU bench runs of two lengths: the
# difference isolates the per-step exchange bytes (setup, prefill and the
# e2e leg cancel). Run with: gpurun --gpus 2 -- bash tools/gpu_nvlink_ctr.sh
O=gpurun_out/nvl
mkdir -p $O
nvidia-smi nvlink -s -i 0 > $O/status.txt 2>&1
nvidia-smi nvlink -gt d > $O/gt_d_0.txt 2>&1
nvidia-smi nvlink -gt r > $O/gt_r_0.txt 2>&1
for S in 20 220; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --steps $S --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$S.log 2>&1
  nvidia-smi nvlink -gt d > $O/gt_d_$S.txt 2>&1
  nvidia-smi nvlink -gt r > $O/gt_r_$S.txt 2>&1
done
python tools/nvml_probe.py > $O/nvml.txt 2>&1
