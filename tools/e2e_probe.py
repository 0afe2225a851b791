"""Where does the e2e (staged, pinned host buffers) step lose time vs the
device-resident step?  python tools/e2e_probe.py  (one GPU, configs[1])"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2201_05500_b200 as kp
from paper_2201_05500_b200.data import make_batch

B, S, E, V = 65536, 100, 64, 100_000_000
tr = kp.Trainer(table_capacity=V + 1_000_000, n_workers=1, minibatch_size=B, embedding_dim=E,
                n_slots=S, hidden=[256, 128], k=1, alpha=0.01, sparse_lr=0.05, seed=42)
tr.prefill(0, 1, V)
bts = [make_batch(B, V=V, zipf_s=1.1, n_slots=S, seed=1000 + b) for b in range(3)]
pin = []
for bt in bts:
    p = {k: torch.from_numpy(v).pin_memory() for k, v in
         (("offs", bt.offs.view(np.int32)), ("keys", bt.keys.view(np.int64)),
          ("slots", bt.slots.view(np.int16)), ("labels", bt.labels))}
    pin.append({"offs": p["offs"].numpy().view(np.uint32), "keys": p["keys"].numpy().view(np.uint64),
                "slots": p["slots"].numpy().view(np.uint16), "labels": p["labels"].numpy(), "_t": p})
dev = [{"offs": torch.from_numpy(bt.offs.view(np.int32)).cuda(), "keys": torch.from_numpy(bt.keys.view(np.int64)).cuda(),
        "slots": torch.from_numpy(bt.slots.view(np.int16)).cuda(), "labels": torch.from_numpy(bt.labels).cuda()} for bt in bts]
stream = torch.cuda.ExternalStream(tr.stream())


def stage(i):
    p = pin[i % 3]
    tr.stage_batch(i % 2, p["offs"], p["keys"], p["labels"], slots=p["slots"])


def timed(fn, n=8, label=""):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    w0 = time.perf_counter()
    for i in range(3, 3 + n):
        fn(i)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{label:40s} dev {e0.elapsed_time(e1) / n:.3f} ms/step  wall {(time.perf_counter() - w0) * 1e3 / n:.3f}")


def step_dev(i):
    bt, d = bts[i % 3], dev[i % 3]
    tr.train_batch_device(bt.offs, d["offs"].data_ptr(), d["keys"].data_ptr(), d["slots"].data_ptr(),
                          d["labels"].data_ptr(), bt.n)


def step_staged_overlap(i):
    stage(i + 1)
    tr.train_staged(i % 2, n_local=B)


def step_staged_serial(i):
    stage(i)
    tr.train_staged(i % 2, n_local=B)


def stage_only(i):
    stage(i)
    torch.cuda.synchronize()


stage(0)
timed(step_dev, label="device-resident")
stage(3)
timed(step_staged_overlap, label="staged, next batch's H2D overlapped")
timed(step_staged_serial, label="staged, H2D then step")
tr.profile(True)
for i in range(4):
    step_dev(i)
pd = tr.profile(False)
tr.profile(True)
stage(0)
for i in range(4):
    step_staged_overlap(i)
ps = tr.profile(False)
ks = ("dedup", "pull", "pool", "mlp", "push", "dense")
print("stages dev   ", {k: round(pd[k] / max(pd["steps"], 1), 3) for k in ks})
print("stages staged", {k: round(ps[k] / max(ps["steps"], 1), 3) for k in ks})
