"""CPU: the oracle is pinned before it is trusted.

1. the f64 C restatement (oracle/kpsim_oracle.c) is BIT-EXACT against the
   compiled reference -- live (oracle/_ref/libkpsim_ref.so) and against the
   committed reference fixtures (tests/golden/, made by make_golden.py);
2. the reference's own known-answer tests, restated with their tolerances
   (proj/tests/test_optimizer.cpp, test_store.cpp, test_eval.cpp, acceptance.cpp);
3. the f32 restatement's drift from f64 -- the envelope the GPU tolerance is
   derived from.
"""
from __future__ import annotations

import tempfile

import numpy as np
import pytest

from helpers import golden_batches, load_golden
from oracle import oracle as O
from paper_2201_05500_b200.data import make_batch

ref_only = pytest.mark.skipif(not O.ref_available(), reason="reference not compiled here")


# ---------------------------------------------------------------- fixtures --
@pytest.mark.parametrize("name", ["n1_k1", "n4_k4_mean", "desk"])
def test_orc64_bit_exact_vs_reference_fixture(name):
    d, meta = load_golden("trainer_" + name)
    cfg = O.TrainerCfg(**meta["cfg"])
    o = O.Orc(cfg, 64)
    for b, (offs, keys, labels) in enumerate(golden_batches(d, meta["batches"])):
        r = o.batch(offs, keys, labels, predict_first=True)
        assert r["loss"] == d[f"b{b}_loss"]
        assert r["auc"] == d[f"b{b}_auc"] or (np.isnan(r["auc"]) and np.isnan(d[f"b{b}_auc"]))
        assert r["cumulative_auc"] == d[f"b{b}_cum_auc"]
        u, _ = O.orc_dedup(keys)
        assert np.array_equal(u, d[f"b{b}_unique"])
    for i in range(cfg.n_workers):
        ws = o.worker_state(i)
        for f in ("x", "m", "v", "v_bar"):
            assert np.array_equal(ws[f], d[f"w{i}_{f}"]), (i, f)
    k, w, acc, _ = o.table()
    assert np.array_equal(k, d["table_keys"])
    assert np.array_equal(w, d["table_w"])
    assert np.array_equal(acc, d["table_acc"])
    assert o.steps() == d["steps"] and o.merges() == d["merges"]


@ref_only
@pytest.mark.parametrize("N,k,mb,pool,act,hidden", [
    (1, 1, 64, "sum", "relu", (16, 8)),
    (2, 3, 32, "mean", "relu", (4,)),
    (3, 2, 16, "sum", "tanh", ()),
    (8, 16, 8, "mean", "tanh", (6, 3)),
])
def test_orc64_bit_exact_vs_live_reference(N, k, mb, pool, act, hidden):
    cfg = O.TrainerCfg(n_workers=N, k=k, minibatch_size=mb, embedding_dim=5, hidden=hidden,
                       pooling=pool, activation=act, alpha=0.03, beta1=0.5, beta2=0.95, sparse_lr=0.2)
    r = O.Ref(cfg, tempfile.mkdtemp())
    o = O.Orc(cfg, 64)
    for b in range(3):
        bt = make_batch(200 + 37 * b, V=700, zipf_s=1.2, nnz=7, poisson=True, seed=b + 11)
        a = r.batch(bt.offs, bt.keys, bt.labels, predict_first=b % 2 == 0)
        c = o.batch(bt.offs, bt.keys, bt.labels, predict_first=b % 2 == 0)
        assert a["loss"] == c["loss"]
    for i in range(N):
        wr, wo = r.worker_state(i), o.worker_state(i)
        for f in wr:
            assert np.array_equal(wr[f], wo[f])
    kr, wr, ar = r.table()
    ko, wo, ao, _ = o.table()
    assert np.array_equal(kr, ko) and np.array_equal(wr, wo) and np.array_equal(ar, ao)


@ref_only
def test_init_dense_matches_reference():
    for e, hidden, seed in [(8, (16,), 42), (3, (), 7), (64, (256, 128), 1)]:
        x = O.ref_init_dense(e, hidden, seed)
        assert np.array_equal(x, O.orc_init_dense(seed, len(x)))


@ref_only
def test_dedup_matches_std_set():
    rng = np.random.default_rng(3)
    for n in [0, 1, 17, 5000]:
        keys = rng.integers(0, 50, n).astype(np.uint64)
        if n:
            keys[0] = np.uint64(0xFFFFFFFFFFFFFFFF)  # legitimate reference key
        u, inv = O.orc_dedup(keys)
        assert np.array_equal(u, O.ref_dedup(keys))
        if n:
            assert np.array_equal(u[inv], keys)


def test_shard_is_stable_bucket():
    u = np.unique(np.random.default_rng(0).integers(0, 10**9, 1000).astype(np.uint64))
    for G in (1, 2, 3, 8):
        perm, counts = O.orc_shard(u, G)
        assert counts.sum() == len(u)
        owners = u[perm] % np.uint64(G)
        assert np.all(np.diff(owners.astype(np.int64)) >= 0)
        start = 0
        for g in range(G):
            blk = u[perm[start:start + counts[g]]]
            assert np.all(np.diff(blk.astype(np.float64)) > 0)  # ascending inside a bucket
            start += counts[g]


# ---------------------------------------------------------- restated KATs --
def test_kat_local_adam_step():
    # test_optimizer.cpp:47-64 (tolerance 1e-12)
    r = O.orc_kstep(64, 0.1, 0.0, 0.999, 0.01, 4, 1, [1.0], np.array([[[0.5]]]))
    assert abs(r["m"][0, 0, 0] - 0.5) <= 1e-12
    assert abs(r["v"][0, 0, 0] - 0.01024) <= 1e-12
    assert abs(r["x"][0, 0, 0] - 0.5) <= 1e-12
    assert r["v_bar"][0, 0, 0] == 0.01
    r = O.orc_kstep(64, 0.1, 0.9, 0.999, 0.01, 4, 1, [1.0], np.array([[[0.5]]]))
    assert abs(r["m"][0, 0, 0] - 0.04999999999999999) <= 1e-12
    assert abs(r["x"][0, 0, 0] - 0.95) <= 1e-12


# N=2, k=2, T=4 frozen replay table (test_optimizer.cpp:144-195, acceptance.cpp:132-178)
REPLAY_G0 = [0.5, -0.25, 0.125, 1.0]
REPLAY_G1 = [-1.0, 0.75, 0.3, -0.5]
REPLAY_WANT = [  # x0 m0 v0 x1 m1 v1 vbar
    (0.95, 0.04999999999999999, 0.012400000000000003, 1.1, -0.09999999999999998,
     0.019900000000000008, 0.01),
    (1.0231917024319275, 0.019999999999999997, 0.019113500000000005, 1.0231917024319275, -0.015,
     0.019113500000000005, 0.019113500000000005),
    (1.0011304721014411, 0.030499999999999996, 0.019078615000000007, 1.011256938482648,
     0.016499999999999994, 0.01982236500000001, 0.019113500000000005),
    (0.9772968452476795, 0.12744999999999998, 0.025505985100000014, 0.9772968452476795,
     -0.035149999999999994, 0.025505985100000014, 0.025505985100000014),
]


@pytest.mark.parametrize("bits,tol", [(64, 1e-12), (32, 2e-6)])
def test_kat_replay_table(bits, tol):
    g = np.array([[[a], [b]] for a, b in zip(REPLAY_G0, REPLAY_G1)])
    r = O.orc_kstep(bits, 0.1, 0.9, 0.99, 0.01, 2, 2, [1.0], g)
    assert list(r["merged"]) == [0, 1, 0, 1]
    for t, w in enumerate(REPLAY_WANT):
        got = (r["x"][t, 0, 0], r["m"][t, 0, 0], r["v"][t, 0, 0], r["x"][t, 1, 0], r["m"][t, 1, 0],
               r["v"][t, 1, 0], r["v_bar"][t, 0, 0])
        for a, b in zip(got, w):
            assert abs(a - b) <= tol * max(1.0, abs(b)), (t, a, b)


def test_kat_textbook_adam_k1_n1():
    # acceptance.cpp:72-102: k=1 N=1 == Adam without bias correction, v0=eps, T=1000
    d, T = 10, 1000
    center = 0.3 * np.arange(d) - 1.0
    x = np.zeros(d)
    m, v = np.zeros(d), np.full(d, 0.01)
    xs, gs = [], []
    for _ in range(T):
        g = x - center
        gs.append(g.copy())
        m = 0.9 * m + (1 - 0.9) * g
        v = 0.999 * v + (1 - 0.999) * g * g
        x = x - 0.01 * m / np.sqrt(v)
        xs.append(x.copy())
    r = O.orc_kstep(64, 0.01, 0.9, 0.999, 0.01, 1, 1, np.zeros(d), np.array(gs)[:, None, :])
    assert np.max(np.abs(r["x"][:, 0, :] - np.array(xs))) <= 1e-12


@pytest.mark.parametrize("bits", [64, 32])
@pytest.mark.parametrize("k", [1, 5, 16])
def test_kat_replica_invariance(bits, k):
    # acceptance.cpp:106-128: N identical workers == N=1, bitwise (centered mean)
    rng = np.random.default_rng(k)
    T, d = 200, 7
    g = rng.normal(size=(T, 1, d))
    x0 = rng.uniform(-1, 1, d)
    solo = O.orc_kstep(bits, 0.01, 0.9, 0.999, 0.01, k, 1, x0, g)
    octo = O.orc_kstep(bits, 0.01, 0.9, 0.999, 0.01, k, 8, x0, np.repeat(g, 8, axis=1))
    for i in range(8):
        assert np.array_equal(octo["x"][:, i, :], solo["x"][:, 0, :])


@pytest.mark.parametrize("k", [1, 3, 7, 32])
def test_kat_merge_cadence(k):
    # test_optimizer.cpp:262-275: exactly floor(T/k) merges
    g = np.random.default_rng(0).normal(size=(100, 3, 3))
    r = O.orc_kstep(64, 0.01, 0.0, 0.999, 0.01, k, 3, [1.0, -1.0, 0.5], g)
    assert r["merged"].sum() == 100 // k


def test_kat_adagrad():
    # test_optimizer.cpp:295-320 and test_smoke.py:86-97
    f = O.orc_fn(64, "adagrad")
    import ctypes as C
    f.argtypes = [O._f64p, O._f64p, O._f64p, C.c_uint64, C.c_double]
    w, acc = np.array([1.0]), np.array([1.0])
    f(w, acc, np.array([3.0]), 1, 0.1)
    assert abs(acc[0] - 10.0) <= 1e-12 and abs(w[0] - 0.9051316701949486) <= 1e-12
    w, acc = np.array([1.0, -2.0]), np.array([0.5, 0.25])
    f(w, acc, np.zeros(2), 2, 0.1)
    assert list(w) == [1.0, -2.0] and list(acc) == [0.5, 0.25]
    w, acc = np.zeros(2), np.full(2, 1e-6)
    f(w, acc, np.array([1.0, -1.0]), 2, 0.1)
    assert list(acc) == [1.0 + 1e-6, 1.0 + 1e-6]
    assert abs(w[0] + 0.1 * 1.0 / np.sqrt(1.0 + 1e-6)) < 1e-12


def test_kat_auc():
    # test_smoke.py:11-15, test_eval.cpp pair-count oracle
    assert O.orc_auc([0.1, 0.9], [0, 1]) == 1.0
    assert O.orc_auc([0.9, 0.1], [0, 1]) == 0.0
    assert O.orc_auc([0.5, 0.5], [0, 1]) == 0.5
    assert np.isnan(O.orc_auc([0.5, 0.6], [1, 1]))
    rng = np.random.default_rng(67)
    for trial in range(10):
        n = int(rng.integers(10, 300))
        s = rng.integers(1, 25, n) / 25.0 if trial % 3 == 0 else rng.random(n)
        y = rng.integers(0, 2, n)
        y[0], y[-1] = 0, 1
        pos, neg = s[y == 1], s[y == 0]
        won = (pos[:, None] > neg[None, :]).sum() + 0.5 * (pos[:, None] == neg[None, :]).sum()
        assert abs(O.orc_auc(s, y) - won / (len(pos) * len(neg))) <= 1e-12


def test_kstep_fixture_bit_exact():
    z = np.load(__import__("os").path.join(__import__("helpers").GOLDEN, "kstep.npz"))
    for key in [k[:-3] for k in z.files if k.endswith("_x0")]:
        N, k = (int(p[1:]) for p in key.split("_"))
        r = O.orc_kstep(64, 0.05, 0.9, 0.99, 0.01, k, N, z[key + "_x0"], z[key + "_g"])
        for f in ("x", "m", "v", "v_bar", "merged"):
            assert np.array_equal(r[f], z[f"{key}_{f}"]), (key, f)


def test_f32_envelope_is_small():
    """The fp32 restatement stays within the envelope the GPU tests use."""
    d, meta = load_golden("trainer_n1_k1")
    cfg = O.TrainerCfg(**meta["cfg"])
    o = O.Orc(cfg, 32)
    for b, (offs, keys, labels) in enumerate(golden_batches(d, meta["batches"])):
        r = o.batch(offs, keys, labels, predict_first=True)
        assert abs(r["loss"] - d[f"b{b}_loss"]) <= 1e-5
        assert abs(r["auc"] - d[f"b{b}_auc"]) <= 1e-3
    _, w, acc, _ = o.table()
    assert np.max(np.abs(w - d["table_w"])) <= 1e-5
    ws = o.worker_state(0)
    assert np.max(np.abs(ws["x"] - d["w0_x"])) <= 1e-5


@pytest.mark.parametrize("pool,act,k", [("sum", "relu", 1), ("mean", "tanh", 2)])
def test_torch64_pinned_to_orc64(pool, act, k):
    """oracle/torch64.py (the f64 checker the full-size GPU tests use) agrees
    with the pinned C oracle to f64 rounding on the same batches."""
    torch = pytest.importorskip("torch")
    from oracle.torch64 import Torch64Trainer
    from paper_2201_05500_b200.data import make_batch as mk
    cfg = O.TrainerCfg(n_workers=1, k=k, minibatch_size=512, embedding_dim=16, n_slots=8,
                       hidden=(32, 16), pooling=pool, activation=act, alpha=0.02, beta1=0.9,
                       beta2=0.99, sparse_lr=0.1)
    o64 = O.Orc(cfg, 64)
    t64 = Torch64Trainer(cfg, "cpu")
    assert np.array_equal(t64.worker_state()["x"], o64.worker_state(0)["x"])
    for b in range(3):
        bt = mk(512, V=3000, zipf_s=1.1, n_slots=8, seed=70 + b)
        keys, slots, offs = bt.keys, bt.slots, bt.offs
        if b == 1:  # multi-hot slots
            keys, slots = np.repeat(bt.keys, 2), np.repeat(bt.slots, 2)
            offs = (bt.offs.astype(np.int64) * 2).astype(np.uint32)
        ro = o64.batch(offs, keys, bt.labels, slots=slots, predict_first=True, want_preds=True)
        rt = t64.batch(offs, keys, bt.labels, slots=slots, predict_first=True)
        assert abs(ro["loss"] - rt["loss"]) < 1e-12
        assert np.max(np.abs(ro["preds"] - rt["preds"])) < 1e-12
    ko, wo, ao, _ = o64.table()
    kt, wt, at = t64.table()
    assert np.array_equal(ko, kt)
    assert np.max(np.abs(wo - wt)) <= 1e-12 * max(1.0, np.abs(wo).max())
    assert np.max(np.abs(ao - at) / ao) <= 1e-12
    xo, xt = o64.worker_state(0)["x"], t64.worker_state()["x"]
    assert np.max(np.abs(xo - xt)) <= 1e-12
