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
    n_batches = int(sys.argv[5]) if len(sys.argv) > 5 else 4
    if variant == "ledger":
        return ledger_main(out_path, S)
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
    grow = 0 if os.environ.get("MGPU_CONST_BATCH") == "1" else 17
    # variant "span": the key space jumps 4e3 -> 1e12 -> 1e5 between batches,
    # so the sync-free dedup's pass plan (from the previous batch) misses on
    # some rank and every rank redoes its sort and the counts exchange
    spans = [4000, 4000, 10**12, 10**12, 10**5, 4000]
    for b in range(n_batches):
        V = spans[b % len(spans)] if variant == "span" else 4000
        if S > 1:
            bt = make_batch(600 + grow * b, V=V, zipf_s=1.1, n_slots=S, seed=b)
        else:
            bt = make_batch(600 + grow * b, V=V, zipf_s=1.1, nnz=7, poisson=True, seed=b)
        batches.append(bt)
        r = tr.train_batch(bt, predict_first=True)
        res["loss"].append(r["loss"])
        res["auc"].append(r.get("auc"))
        tr_cum = r.get("cumulative_auc")
    keys, w, s1, _ = tr.tr.table()
    x = tr.tr.worker_state(0)["x"]
    parts = [None] * world
    dist.all_gather_object(parts, (keys.tolist(), w.tolist(), s1.tolist(), x.tolist()))
    if rank == 0:
        ocfg = O.TrainerCfg(n_workers=world, k=k, minibatch_size=96, embedding_dim=8, n_slots=S,
                            hidden=(16, 8), alpha=0.05, beta1=0.9, beta2=0.99,
                            sparse_lr=cfg["sparse_lr"], seed=5, **extra)
        orc = O.Orc(ocfg, 64)
        o32 = O.Orc(ocfg, 32)  # the fp32 restatement: the drift envelope of fp32 arithmetic
        oloss, oauc, env_loss = [], [], 0.0
        for bt in batches:
            r = orc.batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=True)
            r32 = o32.batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=True)
            oloss.append(r["loss"])
            oauc.append(r["auc"])
            orc_cum = r["cumulative_auc"]
            env_loss = max(env_loss, abs(r32["loss"] - r["loss"]))
        ok, ow, oa, _ = orc.table()
        k32, w32, a32, _ = o32.table()
        x32 = [o32.worker_state(i)["x"] for i in range(world)]
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
            "batches": n_batches, "steps": tr.tr.completed_steps, "merges": tr.tr.merges,
            "oracle_steps": orc.steps(), "oracle_merges": orc.merges(),
            "cum_auc": tr_cum, "oracle_cum_auc": orc_cum,
            "env_w_max_abs": float(np.max(np.abs(w32 - ow))) if np.array_equal(k32, ok) else None,
            "env_x_max_abs": float(max(np.max(np.abs(a - b)) for a, b in zip(x32, [orc.worker_state(i)["x"] for i in range(world)]))),
            "env_loss": env_loss,
        }
        with open(out_path, "w") as f:
            json.dump(summary, f)
        print(json.dumps(summary))
    dist.barrier()
    dist.destroy_process_group()


def ledger_main(out_path, S):
    """Measured-traffic ledger (Trainer::ledger, trainer.hpp:81) for the same
    batches at k = 1/4/16/64: each rank's gpu_pull / gpu_push bytes against the
    counts implied by the batches (remote unique keys x (8 + 4e) and x 4e),
    merge events against floor(T/k), and kstep_ratio (ledger.cpp:132-145)
    of every k over k = 1 next to the paper's Figure-9 ratios."""
    import torch
    import torch.distributed as dist

    import paper_2201_05500_b200 as kp
    from paper_2201_05500_b200.data import make_batch
    from paper_2201_05500_b200.dist import DistributedTrainer, rank_slice

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    e, mb = 16, 128
    batches = [make_batch(world * mb, V=50000, zipf_s=1.1, n_slots=S, seed=900 + b) for b in range(16)]
    ledgers, merges = {}, {}
    for k in (1, 4, 16, 64):
        tr = DistributedTrainer(device=local, table_capacity=1 << 18, n_workers=world, k=k,
                                minibatch_size=mb, embedding_dim=e, n_slots=S, hidden=[64, 32],
                                alpha=0.02, beta1=0.9, beta2=0.99, sparse_lr=0.1)
        for bt in batches:
            tr.train_batch(bt)
        ledgers[k] = tr.tr.ledger()
        merges[k] = tr.tr.merges
        D = tr.tr.dense_dim
        del tr
    # expected sparse bytes from the batches (one minibatch step per batch)
    remote = 0
    for bt in batches:
        first, n = rank_slice(bt.n, world, 1, mb, rank)
        u = np.unique(bt.keys[bt.offs[first]:bt.offs[first + n]])
        remote += int(np.count_nonzero(u % np.uint64(world) != np.uint64(rank)))
    got = {k: ledgers[k] for k in ledgers}
    parts = [None] * world
    dist.all_gather_object(parts, (got, remote, merges, D))
    if rank == 0:
        res = {"world": world, "e": e, "D": D, "per_rank": []}
        for g, (led, rem, mg, _) in enumerate(parts):
            res["per_rank"].append({
                "pull_ok": all(led[k]["gpu_pull"]["bytes"] == rem * (8 + 4 * e) for k in led),
                "push_ok": all(led[k]["gpu_push"]["bytes"] == rem * 4 * e for k in led),
                "merges": mg, "ledger": {str(k): v for k, v in led.items()}})
        led0 = parts[0][0]
        res["kstep_ratio"] = {str(k): kp.kstep_ratio(led0[k], led0[1]) for k in (4, 16, 64)}
        res["paper_fig9_model_transmission_ratio"] = {"10": 0.181, "20": 0.108, "50": 0.064,
                                                      "100": 0.028, "200": 0.012}
        res["merges_ok"] = all(p[2][k] == 16 // k for p in parts for k in (1, 4, 16, 64))
        with open(out_path, "w") as f:
            json.dump(res, f)
        print(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
