mkdir -p gpurun_out
export KP_H3_AR=0
timeout 600 bash tools/gpu_ncu_skip.sh r02dx k_h3 1
unset KP_H3_AR
timeout 600 bash tools/gpu_ncu_skip.sh r02 k_pool_planes_ident 0
timeout 600 bash tools/gpu_ncu_skip.sh r02 k_seg_chunks 0
