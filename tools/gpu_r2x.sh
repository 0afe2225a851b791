mkdir -p gpurun_out
bash tools/gpu_c5.sh
# ncu --set full of the step's top kernels on one GPU (after the multi-GPU runs)
export CUDA_VISIBLE_DEVICES=0
timeout 900 bash tools/gpu_ncu_skip.sh r02f k_h3 0
timeout 900 bash tools/gpu_ncu_skip.sh r02f k_pool_planes_ident 0
timeout 900 bash tools/gpu_ncu_skip.sh r02f k_seg_chunks 0
timeout 900 bash tools/gpu_ncu_skip.sh r02f k_probe 6
timeout 900 bash tools/gpu_ncu_skip.sh r02f k_downsweep 0
ls gpurun_out/*.ncu-rep
