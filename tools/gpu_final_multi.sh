# round-end multi-GPU evidence: sharded parity tests, weak scaling, k sweep, C1, C5-like
bash tools/gpu_multi.sh
bash tools/gpu_sweep.sh
bash tools/gpu_c5.sh
