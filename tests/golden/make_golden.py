"""Regenerates tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref/
libkpsim_ref.so, built by oracle/Makefile from /root/reference/proj/src).

Each fixture holds the exact inputs (CSR batches) and the reference's f64
outputs after every batch: per-batch loss/AUC, the dense worker states and the
full embedding table. Tests compare the f64 restatement bit-exactly and the
B200 path within the fp32 tolerance against these.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref, TrainerCfg, ref_dedup, ref_kstep  # noqa: E402
from paper_2201_05500_b200.data import make_batch  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CONFIGS = {
    # single worker, k=1: the monolithic-loop configuration (test_trainer.cpp:116-187)
    "n1_k1": dict(cfg=dict(n_workers=1, k=1, minibatch_size=256, embedding_dim=8, hidden=(16, 8),
                           activation="relu", pooling="sum", alpha=0.01, sparse_lr=0.05),
                  data=dict(B=512, V=2000, zipf_s=1.1, nnz=10, poisson=True), batches=3),
    # 4 workers, k=4, tanh, mean pooling, 16-instance minibatches
    "n4_k4_mean": dict(cfg=dict(n_workers=4, k=4, minibatch_size=16, embedding_dim=4, hidden=(8,),
                                activation="tanh", pooling="mean", alpha=0.02, beta1=0.9,
                                beta2=0.99, sparse_lr=0.3),
                       data=dict(B=300, V=500, zipf_s=1.1, nnz=6, poisson=True), batches=3),
    # the desk benchmark defaults (proj/data/desk.json, config.cpp:32-40)
    "desk": dict(cfg=dict(n_workers=4, k=8, minibatch_size=16, embedding_dim=8, hidden=(),
                          activation="relu", pooling="sum", alpha=0.11, beta1=0.0, beta2=0.999,
                          epsilon=0.01, sparse_lr=0.7),
                 data=dict(B=1024, V=10000, zipf_s=None, nnz=10, poisson=True), batches=2),
}


def run(name, spec):
    cfg = TrainerCfg(**spec["cfg"])
    ref = Ref(cfg, tempfile.mkdtemp(prefix="kpsim_golden_"))
    out = {}
    for b in range(spec["batches"]):
        bt = make_batch(spec["data"]["B"], V=spec["data"]["V"], zipf_s=spec["data"]["zipf_s"],
                        nnz=spec["data"]["nnz"], poisson=spec["data"]["poisson"], seed=100 + b)
        r = ref.batch(bt.offs, bt.keys, bt.labels, predict_first=True)
        out[f"b{b}_offs"] = bt.offs
        out[f"b{b}_keys"] = bt.keys
        out[f"b{b}_labels"] = bt.labels
        out[f"b{b}_loss"] = np.float64(r["loss"])
        out[f"b{b}_auc"] = np.float64(r["auc"])
        out[f"b{b}_cum_auc"] = np.float64(r["cumulative_auc"])
        out[f"b{b}_unique"] = ref_dedup(bt.keys)
    for i in range(cfg.n_workers):
        ws = ref.worker_state(i)
        for f, v in ws.items():
            out[f"w{i}_{f}"] = v
    k, w, acc = ref.table()
    out["table_keys"], out["table_w"], out["table_acc"] = k, w, acc
    out["steps"], out["merges"] = np.int64(ref.steps()), np.int64(ref.merges())
    meta = dict(spec["cfg"])
    meta["hidden"] = list(meta.get("hidden", ()))
    out["meta"] = np.array(repr(dict(cfg=meta, batches=spec["batches"])))
    np.savez_compressed(os.path.join(HERE, f"trainer_{name}.npz"), **out)


def kstep_golden():
    """Engine trajectories (N, k) under fixed pseudo-random gradients."""
    rng = np.random.default_rng(5)
    out = {}
    for N, k in [(1, 1), (2, 2), (3, 5), (8, 4)]:
        D, T = 6, 40
        x0 = rng.uniform(-1, 1, D)
        g = rng.normal(size=(T, N, D))
        r = ref_kstep(0.05, 0.9, 0.99, 0.01, k, N, x0, g)
        out[f"n{N}_k{k}_x0"] = x0
        out[f"n{N}_k{k}_g"] = g
        for f in ("x", "m", "v", "v_bar", "merged"):
            out[f"n{N}_k{k}_{f}"] = r[f]
    np.savez_compressed(os.path.join(HERE, "kstep.npz"), **out)


if __name__ == "__main__":
    for n, s in CONFIGS.items():
        run(n, s)
        print("wrote", n)
    kstep_golden()
    print("wrote kstep")
