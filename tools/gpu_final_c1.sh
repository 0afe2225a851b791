# final tree, 1 GPU: configs[0] with e2e, and configs[1] default bench
O=gpurun_out/fc1; mkdir -p $O
C1="--batch 4096 --slots 26 --dim 8 --vocab 1000000 --hidden 64,32"
timeout 300 python bench.py $C1 --steps 30 --warmup 5 > $O/c1.log 2>&1
timeout 300 python bench.py $C1 --steps 30 --warmup 5 --impl reference > $O/c1_ref.log 2>&1
timeout 600 python bench.py > $O/c2.log 2>&1
