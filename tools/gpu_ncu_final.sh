# round-end ncu --set full captures of the step's top kernels (one GPU)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --pool 1 --no-e2e --no-cpu-baseline"
NCU=/usr/local/cuda/bin/ncu
$B > gpurun_out/plain_final.log 2>&1; echo plain rc=$?
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:"^k_h3$" -s 0 -c 3 -o gpurun_out/full_r02z_k_h3 $B > gpurun_out/ncu_full_r02z_k_h3.log 2>&1; echo k_h3 rc=$?
for k in k_seg_chunks k_pool_planes_ident k_downsweep k_dedup_emit; do
  timeout 600 $NCU --set full --import-source on --clock-control none -k regex:"^$k" -s 0 -c 1 -o gpurun_out/full_r02z_$k $B > gpurun_out/ncu_full_r02z_$k.log 2>&1; echo $k rc=$?
done
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:"^k_probe" -s 6 -c 1 -o gpurun_out/full_r02z_k_probe $B > gpurun_out/ncu_full_r02z_k_probe.log 2>&1; echo k_probe rc=$?
du -sh gpurun_out
