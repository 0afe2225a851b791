"""Per-step wall/device times of the sync-free step with CUDA graphs (capture
on the second sight of a batch shape, replay after)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05500_b200 as kp
from paper_2201_05500_b200.data import make_batch
B, S, E, V = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (65536, 100, 64, 100_000_000)))
hid = [256, 128] if E == 64 else [64, 32]
tr = kp.Trainer(table_capacity=V + 1_000_000, n_workers=1, minibatch_size=B, embedding_dim=E,
                n_slots=S, hidden=hid, k=1, alpha=0.01, sparse_lr=0.05, seed=42)
tr.prefill(0, 1, V)
bts = [make_batch(B, V=V, zipf_s=1.1, n_slots=S, seed=1000 + b) for b in range(3)]
dev = [{"offs": torch.from_numpy(bt.offs.view(np.int32)).cuda(), "keys": torch.from_numpy(bt.keys.view(np.int64)).cuda(),
        "slots": torch.from_numpy(bt.slots.view(np.int16)).cuda(), "labels": torch.from_numpy(bt.labels).cuda()} for bt in bts]
stream = torch.cuda.ExternalStream(tr.stream())
for i in range(12):
    bt, d = bts[i % 3], dev[i % 3]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(stream)
    tr.train_batch_device(bt.offs, d["offs"].data_ptr(), d["keys"].data_ptr(), d["slots"].data_ptr(),
                          d["labels"].data_ptr(), bt.n)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"step {i}: wall {(time.perf_counter() - w0) * 1e3:.3f} ms  dev {e0.elapsed_time(e1):.3f} ms  launches {kp.launch_count()}")
