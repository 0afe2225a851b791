"""Multi-GPU parity worker (launched by tests/test_gpu_multi.py under torchrun).

Each rank trains its shard_batch slice of the same global batches with the
table hash-sharded key % G over NCCL; rank 0 gathers every shard and compares
with the f64 oracle running the same N=G workers in one process.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2201_05500_b200.data import make_batch
    from paper_2201_05500_b200.dist import DistributedTrainer

    out_path = sys.argv[1]
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    S = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    variant = sys.argv[4] if len(sys.argv) > 4 else "base"
    extra = (dict(pooling="mean", sparse_rule="adam", activation="tanh", sparse_eps=1e-6)
             if variant == "mean_adam" else {})
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    cfg = dict(n_workers=world, k=k, minibatch_size=96, embedding_dim=8, n_slots=S, hidden=[16, 8],
               alpha=0.05, beta1=0.9, beta2=0.99, sparse_lr=0.5, seed=5, **extra)
    if variant == "mean_adam":
        cfg["sparse_lr"] = 0.05
    tr = DistributedTrainer(device=local, table_capacity=1 << 16, **cfg)
    res = {"loss": [], "auc": []}
    batches = []
    for b in range(4):
        if S > 1:
            bt = make_batch(600 + 17 * b, V=4000, zipf_s=1.1, n_slots=S, seed=b)
        else:
            bt = make_batch(600 + 17 * b, V=4000, zipf_s=1.1, nnz=7, poisson=True, seed=b)
        batches.append(bt)
        r = tr.train_batch(bt, predict_first=True)
        res["loss"].append(r["loss"])
        res["auc"].append(r.get("auc"))
    keys, w, s1, _ = tr.tr.table()
    x = tr.tr.worker_state(0)["x"]
    parts = [None] * world
    dist.all_gather_object(parts, (keys.tolist(), w.tolist(), s1.tolist(), x.tolist()))
    if rank == 0:
        ocfg = O.TrainerCfg(n_workers=world, k=k, minibatch_size=96, embedding_dim=8, n_slots=S,
                            hidden=(16, 8), alpha=0.05, beta1=0.9, beta2=0.99,
                            sparse_lr=cfg["sparse_lr"], seed=5, **extra)
        orc = O.Orc(ocfg, 64)
        oloss, oauc = [], []
        for bt in batches:
            r = orc.batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=True)
            oloss.append(r["loss"])
            oauc.append(r["auc"])
        ok, ow, oa, _ = orc.table()
        allk = np.concatenate([np.array(p[0], np.uint64) for p in parts])
        allw = np.concatenate([np.array(p[1], np.float64).reshape(-1, 8) for p in parts])
        alla = np.concatenate([np.array(p[2], np.float64).reshape(-1, 8) for p in parts])
        order = np.argsort(allk)
        allk, allw, alla = allk[order], allw[order], alla[order]
        owners_ok = all(all(int(kk) % world == g for kk in p[0]) for g, p in enumerate(parts))
        xs = [np.array(p[3]) for p in parts]
        ox = [orc.worker_state(i)["x"] for i in range(world)]
        summary = {
            "world": world, "k": k, "S": S,
            "keyset_equal": bool(np.array_equal(allk, ok)),
            "owners_ok": bool(owners_ok),
            "w_max_abs": float(np.max(np.abs(allw - ow))) if np.array_equal(allk, ok) else None,
            "acc_max_rel": (float(np.max(np.abs(alla - oa) / oa)) if variant == "base" else
                            float(np.max(np.abs(alla - oa)))) if np.array_equal(allk, ok) else None,
            "variant": variant,
            "x_max_abs": float(max(np.max(np.abs(a - b)) for a, b in zip(xs, ox))),
            "loss": res["loss"], "oracle_loss": oloss,
            "auc": res["auc"], "oracle_auc": oauc,
            "table_rows_per_rank": [len(p[0]) for p in parts],
        }
        with open(out_path, "w") as f:
            json.dump(summary, f)
        print(json.dumps(summary))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
