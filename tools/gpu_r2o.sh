mkdir -p gpurun_out
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29630 tools/mgpu_parity.py gpurun_out/dbg.json 1 4 base 24 > gpurun_out/dbg_$1.log 2>&1; echo "$1 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/dbg.json')); import numpy as np
dl=[abs(a-b) for a,b in zip(d['loss'],d['oracle_loss'])]
print('w', d['w_max_abs'], 'x', d['x_max_abs'], 'dloss', ['%.1e'%v for v in dl])"; }
KP_PEER=1 run peer_grow
KP_PEER=0 run nccl_grow
MGPU_CONST_BATCH=1 KP_PEER=1 run peer_const
KP_GEMM_H3=0 KP_PEER=1 run peer_grow_noh3
