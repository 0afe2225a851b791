"""GPU parity: the sm_100a path (through the C ABI / C++ shim) against the oracle.

Bars:
  * integer/byte/index work -- dedup output + inverse, owner shard, table key
    sets -- BIT-EXACT;
  * elementwise rules (AdaGrad, dense Adam, merge) -- bit-exact against fp32
    numpy/oracle arithmetic when the inputs are identical;
  * training state after N steps (embeddings, optimizer state, dense x, loss,
    AUC) -- within the stated fp32 tolerance of the f64 reference:
        TOL_W    = 2e-4 abs + 1e-3 rel   (embeddings, dense x)
        TOL_ACC  = 1e-3 rel             (AdaGrad accumulators, Adam v)
        TOL_LOSS = 1e-4 abs             (batch loss)
        TOL_AUC  = 5e-3 abs             (batch / cumulative AUC; rank-based,
                                          near-ties may flip)
    The f32 restatement's own drift from f64 on the same fixtures is
    <=1e-5 (w, x), <=4.4e-4 (AUC), <=5e-7 (loss) -- tests/test_oracle.py.
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import golden_batches, load_golden, rel_err, trainer_kwargs
from oracle import oracle as O
from paper_2201_05500_b200.data import make_batch

pytestmark = pytest.mark.gpu

TOL_W_ABS, TOL_W_REL = 2e-4, 1e-3
TOL_ACC_REL = 1e-3
TOL_LOSS = 1e-4
TOL_AUC = 5e-3


def close(a, b, atol=TOL_W_ABS, rtol=TOL_W_REL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    err = np.abs(a - b) - (atol + rtol * np.abs(b))
    return float(err.max()) <= 0 if a.size else True


# ------------------------------------------------------------------ dedup ---
@pytest.mark.parametrize("n,V,zipf", [(0, 10, None), (1, 10, None), (1000, 1, None),
                                      (5000, 50, None), (300_000, 10**6, 1.1),
                                      (2_000_000, 10**8, 1.1), (100_000, 2**64 - 1, None),
                                      (7, 1000, None), (99_999, 10**6, 1.1),
                                      (6_553_600, 10**8, 1.1), (3_276_800, 5 * 10**8, 1.3)])
def test_dedup_bit_exact(kp, n, V, zipf):
    rng = np.random.default_rng(n + 1)
    if zipf:
        from paper_2201_05500_b200.data import ZipfSampler, rank_to_key
        keys = rank_to_key(ZipfSampler(V, zipf).sample(n, rng), V)
    else:
        keys = rng.integers(0, V, n, dtype=np.uint64) if V < 2**63 else \
            rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    if n > 2:
        keys[1] = np.uint64(2**64 - 1)
    u, inv, seg = kp.dedup(keys)
    want, winv = O.orc_dedup(keys)
    assert np.array_equal(u, want)
    assert np.array_equal(inv, winv)
    if n:
        assert seg[0] == 0 and seg[-1] == n and np.all(np.diff(seg.astype(np.int64)) > 0)
        assert np.array_equal(np.diff(seg.astype(np.int64)), np.bincount(inv, minlength=len(u)))
    if O.ref_available() and n <= 300_000:
        assert np.array_equal(u, O.ref_dedup(keys))


def test_dedup_span_changes_between_calls(kp):
    """dedup plans its radix passes from the previous call's key span and
    re-sorts when a batch outgrows the plan: spans that grow (narrow ->
    wider narrow -> full u64) and shrink must all stay bit-exact."""
    rng = np.random.default_rng(7)
    for V in (1000, 10**6, 10**8, 2**40, None, 50, 10**9, 1):
        n = 200_000
        if V is None:
            keys = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
        else:
            keys = rng.integers(0, V, n, dtype=np.uint64) + np.uint64(12345)
        u, inv, _ = kp.dedup(keys)
        want, winv = O.orc_dedup(keys)
        assert np.array_equal(u, want), V
        assert np.array_equal(inv, winv), V


@pytest.mark.parametrize("R,n_per,V", [(1, 1000, 10**4), (2, 50_000, 10**5), (3, 7, 20),
                                       (4, 300_000, 10**6), (8, 120_000, 10**6), (5, 0, 10)])
def test_dedup_runs_matches_dedup(kp, R, n_per, V):
    """Owner-side dedup of the exchange (merge of per-source ascending runs):
    identical unique/inverse/segments to the radix dedup, and sorted positions
    equal to a stable sort (ties in source order)."""
    rng = np.random.default_rng(R * 1000 + n_per)
    runs = []
    for r in range(R):
        k = np.unique(rng.integers(0, V, max(n_per - 3 * r, 0), dtype=np.uint64))
        runs.append(k)
    if R >= 2 and len(runs[0]):
        runs[1] = np.unique(np.concatenate([runs[1], runs[0][:5], [np.uint64(2**64 - 1)]]))
    keys = np.concatenate(runs).astype(np.uint64) if runs else np.zeros(0, np.uint64)
    lens = np.array([len(r) for r in runs], np.uint64)
    u, inv, seg, pos = kp.dedup_runs(keys, lens)
    u2, inv2, seg2 = kp.dedup(keys)
    assert np.array_equal(u, u2) and np.array_equal(inv, inv2) and np.array_equal(seg, seg2)
    assert np.array_equal(pos, np.argsort(keys, kind="stable").astype(np.uint32))


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_shard_bit_exact(kp, G):
    rng = np.random.default_rng(G)
    u = np.unique(rng.integers(0, 10**9, 100_000).astype(np.uint64))
    perm, pos, counts = kp.shard(u, G)
    wperm, wcounts = O.orc_shard(u, G)
    assert np.array_equal(perm, wperm) and np.array_equal(counts, wcounts)
    assert np.array_equal(pos[perm], np.arange(len(u)))


# ------------------------------------------------------------------ store ---
def test_store_fresh_and_adagrad_goldens(kp, tmp_path):
    # test_store.cpp:61-83, test_smoke.py:86-97 (values through fp32)
    s = kp.TieredStore(cache_capacity=2, cold_dir=str(tmp_path / "cold"), embedding_dim=2)
    got = s.pull([1, 2, 3])
    assert got[3] == ([0.0, 0.0], [np.float32(1e-6)] * 2)
    s.push({1: [1.0, -1.0]}, lr=0.1)
    w, acc = s.pull([1])[1]
    a32 = np.float32(1e-6) + np.float32(1.0)
    assert acc == [float(a32)] * 2
    assert w[0] == float(np.float32(0) - np.float32(0.1) * np.float32(1.0) / np.sqrt(a32))
    assert abs(w[0] + 0.1 / np.sqrt(1 + 1e-6)) < 1e-7
    assert s.cache_size == 3
    with pytest.raises(kp.StoreError, match="not in the current working set"):
        s.push({99: [1.0, 1.0]}, lr=0.1)
    with pytest.raises(kp.StoreError, match="dimension mismatch"):
        s.push({1: [1.0]}, lr=0.1)
    with pytest.raises(kp.StoreError, match="empty key set"):
        s.pull([])
    w2, _ = kp.adagrad_sparse_update([1.0], [1.0], [3.0], 0.1)
    assert abs(w2[0] - 0.9051316701949486) < 1e-6


def test_store_u64max_key(kp, tmp_path):
    s = kp.TieredStore(cache_capacity=8, cold_dir=str(tmp_path), embedding_dim=4)
    big = 2**64 - 1
    s.pull([0, big, 5])
    s.push({big: [1.0, 2.0, 3.0, 4.0]}, lr=0.5)
    w, acc = s.pull([big])[big]
    assert acc[3] == float(np.float32(1e-6) + np.float32(16.0))
    k, W, A = s.export()
    assert list(k) == [0, 5, big]


def test_store_flat_map_oracle(kp, tmp_path):
    # acceptance.cpp:332-414 restated: 1000 keys, dim 4, lr 0.05, seed 41; the
    # fp32 flat map uses the same expression tree -> bit-exact
    s = kp.TieredStore(cache_capacity=64, cold_dir=str(tmp_path), embedding_dim=4)
    rng = np.random.default_rng(41)
    flat = {}
    lr = np.float32(0.05)
    for op in range(3000):
        n = 1 + int(rng.integers(0, 8))
        keys = sorted(set(int(k) for k in rng.integers(0, 1000, n)))
        got = s.pull(keys)
        for k in keys:
            w, a = flat.setdefault(k, (np.zeros(4, np.float32), np.full(4, np.float32(1e-6))))
            assert np.array_equal(np.float32(got[k][0]), w) and np.array_equal(np.float32(got[k][1]), a)
        if rng.random() < 0.75:
            upd = {k: rng.uniform(-1, 1, 4) for k in keys}
            s.push(upd, lr=0.05)
            for k, g in upd.items():
                w, a = flat[k]
                g = g.astype(np.float32)
                a = a + g * g
                w = w - (lr * g) / np.sqrt(a)
                flat[k] = (w, a)
    k, W, A = s.export()
    assert list(k) == sorted(flat)
    for i, key in enumerate(k):
        assert np.array_equal(W[i], flat[int(key)][0]) and np.array_equal(A[i], flat[int(key)][1])


# ------------------------------------------------------------------ dense ---
def test_dense_kats(kp):
    h = kp.AdamHyper()
    h.alpha, h.beta1, h.beta2, h.epsilon, h.k = 0.1, 0.0, 0.999, 0.01, 4
    s = kp.local_adam_step(kp.WorkerState.init([1.0], 0.01), [0.5], h)
    assert abs(s.m[0] - 0.5) < 1e-7 and abs(s.v[0] - 0.01024) < 1e-7 and abs(s.x[0] - 0.5) < 1e-6
    assert s.v_bar[0] == float(np.float32(0.01))
    h.alpha = 0.1
    a = kp.WorkerState.init([1.0], 0.01)
    b = kp.WorkerState.init([0.0], 0.01)
    a.m, a.v = [0.2], [0.04]
    b.m, b.v = [-0.2], [0.16]
    m = kp.global_merge([a, b], h)
    assert abs(m[0].v_bar[0] - 0.1) < 1e-7 and abs(m[0].x[0] - 0.5) < 1e-6
    assert m[0].x == m[1].x and m[0].v == m[0].v_bar and m[0].m == [0.2] and m[1].m == [-0.2]
    one = kp.WorkerState.init([1.5, -0.5], 0.01)
    one.m, one.v = [0.3, 0.1], [0.2, 0.4]
    merged = kp.global_merge([one] * 5, h)
    x32 = np.float32([1.5, -0.5]) - np.float32(0.1) * np.float32([0.3, 0.1]) / np.sqrt(np.float32([0.2, 0.4]))
    assert merged[0].x == [float(v) for v in x32]  # identical workers: bit-identical to N=1


@pytest.mark.parametrize("key", ["n1_k1", "n2_k2", "n3_k5", "n8_k4"])
def test_kstep_engine_fixture(kp, key):
    from helpers import GOLDEN
    z = np.load(GOLDEN + "/kstep.npz")
    N, k = (int(p[1:]) for p in key.split("_"))
    h = kp.AdamHyper()
    h.alpha, h.beta1, h.beta2, h.epsilon, h.k = 0.05, 0.9, 0.99, 0.01, k
    e = kp.KStepEngine(h, N, list(z[key + "_x0"]))
    o32 = O.orc_kstep(32, 0.05, 0.9, 0.99, 0.01, k, N, z[key + "_x0"], z[key + "_g"])
    for t, g in enumerate(z[key + "_g"]):
        merged, _ = e.step([list(r) for r in g])
        assert merged == bool(z[key + "_merged"][t])
        st = e.states()
        for i in range(N):
            # bit-exact vs the fp32 restatement, tolerance vs the f64 reference
            assert np.array_equal(np.float32(st[i].x), np.float32(o32["x"][t, i])), (t, i)
            assert close(st[i].x, z[key + "_x"][t, i], 1e-5, 1e-4)


def test_replica_invariance_bitwise(kp):
    h = kp.AdamHyper()
    h.alpha, h.beta1, h.beta2, h.epsilon, h.k = 0.01, 0.9, 0.999, 0.01, 5
    rng = np.random.default_rng(2)
    x0 = list(rng.uniform(-1, 1, 10))
    solo, octo = kp.KStepEngine(h, 1, x0), kp.KStepEngine(h, 8, x0)
    for _ in range(60):
        g = list(rng.normal(size=10))
        solo.step([g])
        octo.step([g] * 8)
        assert octo.x_bar() == solo.x_bar()


# ---------------------------------------------------------------- trainer ---
@pytest.mark.parametrize("name", ["n1_k1", "n4_k4_mean", "desk"])
def test_trainer_vs_reference_fixture(kp, name):
    d, meta = load_golden("trainer_" + name)
    cfg = meta["cfg"]
    tr = kp.Trainer(table_capacity=1 << 16, **trainer_kwargs(cfg))
    for b, (offs, keys, labels) in enumerate(golden_batches(d, meta["batches"])):
        r = tr.train_batch(offs.astype(np.uint32), keys, labels, predict_first=True)
        assert abs(r["loss"] - d[f"b{b}_loss"]) <= TOL_LOSS, (b, r["loss"], d[f"b{b}_loss"])
        auc = O.orc_auc(r["preds"].astype(np.float64), labels)
        assert abs(auc - d[f"b{b}_auc"]) <= TOL_AUC
    keys, w, s1, _ = tr.table()
    assert np.array_equal(keys, d["table_keys"])  # key set bit-exact
    assert close(w, d["table_w"]), rel_err(w, d["table_w"])
    assert close(s1, d["table_acc"], 0, TOL_ACC_REL)
    n_workers = cfg.get("n_workers", 1)
    for i in range(n_workers):
        ws = tr.worker_state(i)
        assert close(ws["x"], d[f"w{i}_x"]), i
        assert close(ws["v"], d[f"w{i}_v"], 1e-9, TOL_ACC_REL)
    assert tr.completed_steps == d["steps"]


@pytest.mark.parametrize("S,pool,rule", [(4, "sum", "adagrad"), (6, "mean", "adagrad"),
                                         (1, "sum", "adam"), (3, "mean", "adam")])
def test_trainer_slots_and_sparse_adam_vs_oracle(kp, S, pool, rule):
    cfg = O.TrainerCfg(n_workers=2, k=3, minibatch_size=64, embedding_dim=8, n_slots=S,
                       hidden=(16,), pooling=pool, activation="relu", alpha=0.02, sparse_lr=0.1,
                       sparse_rule=rule, sparse_beta1=0.9, sparse_beta2=0.99, sparse_eps=1e-6)
    o64 = O.Orc(cfg, 64)
    tr = kp.Trainer(table_capacity=1 << 16, **trainer_kwargs(vars(cfg)))
    for b in range(3):
        if S > 1:
            bt = make_batch(256, V=3000, zipf_s=1.1, n_slots=S, seed=b)
            # multi-hot slots: duplicate every other occurrence into the same slot
            keys = np.repeat(bt.keys, 2)[: 2 * len(bt.keys)]
            slots = np.repeat(bt.slots, 2)
            offs = (bt.offs.astype(np.int64) * 2).astype(np.uint32)
        else:
            bt = make_batch(256, V=3000, zipf_s=1.1, nnz=9, poisson=True, seed=b)
            keys, slots, offs = bt.keys, None, bt.offs
        ro = o64.batch(offs, keys, bt.labels, slots=slots, predict_first=True)
        rg = tr.train_batch(offs, keys, bt.labels, slots=slots, predict_first=True)
        assert abs(ro["loss"] - rg["loss"]) <= TOL_LOSS
    k64, w64, a64, v64 = o64.table()
    kg, wg, s1, s2 = tr.table()
    assert np.array_equal(k64, kg)
    assert close(wg, w64)
    assert close(s1, a64, 1e-9 if rule == "adagrad" else 1e-6, TOL_ACC_REL if rule == "adagrad" else 1e-2)
    for i in range(2):
        assert close(tr.worker_state(i)["x"], o64.worker_state(i)["x"])


@pytest.mark.parametrize("S,e,pool,rule,multi,act", [(12, 16, "sum", "adagrad", False, "relu"),
                                                     (10, 128, "mean", "adam", True, "relu"),
                                                     (16, 64, "sum", "adagrad", False, "relu"),
                                                     (9, 4, "mean", "adagrad", True, "relu"),
                                                     (16, 64, "mean", "adam", False, "tanh")])
@pytest.mark.parametrize("tc_min", ["0", None])
def test_trainer_pooling_paths_vs_oracle(kp, monkeypatch, S, e, pool, rule, multi, act, tc_min):
    """Instance-major pooling (S >= 8, e <= 64: one warp per instance, row
    maxima without atomics) and the atomic row-max path (e = 128 / multi-hot),
    feeding the first layer -- on the tensor-core paths (fp16 planes / fp16
    operands; KP_TC_MIN_MFLOP=0 forces them at this small batch) and on the
    small-tile SIMT kernel the default routes these small products to:
    state vs the f64 oracle."""
    if tc_min is not None:
        monkeypatch.setenv("KP_TC_MIN_MFLOP", tc_min)
    cfg = O.TrainerCfg(n_workers=1, k=1, minibatch_size=256, embedding_dim=e, n_slots=S,
                       hidden=(32, 16), pooling=pool, activation=act, alpha=0.02, sparse_lr=0.1,
                       sparse_rule=rule, sparse_beta1=0.9, sparse_beta2=0.99, sparse_eps=1e-6)
    o64 = O.Orc(cfg, 64)
    tr = kp.Trainer(table_capacity=1 << 16, **trainer_kwargs(vars(cfg)))
    for b in range(3):
        bt = make_batch(256, V=5000, zipf_s=1.1, n_slots=S, seed=10 + b)
        keys, slots, offs = bt.keys, bt.slots, bt.offs
        if multi:
            keys = np.repeat(bt.keys, 2)
            slots = np.repeat(bt.slots, 2)
            offs = (bt.offs.astype(np.int64) * 2).astype(np.uint32)
        ro = o64.batch(offs, keys, bt.labels, slots=slots, predict_first=True)
        rg = tr.train_batch(offs, keys, bt.labels, slots=slots, predict_first=True)
        assert abs(ro["loss"] - rg["loss"]) <= TOL_LOSS
    k64, w64, a64, _ = o64.table()
    kg, wg, s1, _ = tr.table()
    assert np.array_equal(k64, kg)
    assert close(wg, w64)
    assert close(tr.worker_state(0)["x"], o64.worker_state(0)["x"])


@pytest.mark.parametrize("B,S", [(65536, 8), (16384, 80)])
def test_trainer_hot_key_block_sums_vs_oracle(kp, B, S):
    """One key holding ~80% of a 0.5M / 1.3M-occurrence batch: its gradient
    spans thousands of chunks, so the segmented reduction takes the two-level
    block-sum path (kp_embed.cu k_seg_fix, Q2); the 1.3M case runs the full
    64-position chunks (shorter ones below 1.2M positions). State vs the f64
    oracle."""
    cfg = O.TrainerCfg(n_workers=1, k=1, minibatch_size=B, embedding_dim=4, n_slots=S,
                       hidden=(16,), pooling="sum", activation="relu", alpha=0.02, sparse_lr=0.1)
    o64 = O.Orc(cfg, 64)
    tr = kp.Trainer(table_capacity=1 << 16, **trainer_kwargs(vars(cfg)))
    for b in range(2):
        bt = make_batch(B, V=1000, zipf_s=3.0, n_slots=S, seed=40 + b)
        assert np.bincount(bt.keys.astype(np.int64)).max() > 300_000
        ro = o64.batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=True)
        rg = tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=True)
        assert abs(ro["loss"] - rg["loss"]) <= TOL_LOSS
    k64, w64, a64, _ = o64.table()
    kg, wg, s1, _ = tr.table()
    assert np.array_equal(k64, kg)
    assert close(wg, w64)
    assert close(s1, a64, 1e-9, TOL_ACC_REL)
    assert close(tr.worker_state(0)["x"], o64.worker_state(0)["x"])


def test_trainer_deterministic(kp):
    def run():
        tr = kp.Trainer(table_capacity=1 << 18, n_workers=1, k=1, minibatch_size=4096,
                        embedding_dim=16, n_slots=8, hidden=[32, 16])
        for b in range(2):
            bt = make_batch(4096, V=10**6, zipf_s=1.1, n_slots=8, seed=b)
            tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots)
        return tr.table(), tr.worker_state(0)["x"]
    (k1, w1, a1, _), x1 = run()
    (k2, w2, a2, _), x2 = run()
    assert np.array_equal(k1, k2) and np.array_equal(w1, w2) and np.array_equal(a1, a2)
    assert np.array_equal(x1, x2)


def test_trainer_full_size_properties(kp):
    """configs[1] at full size (B=65536, 100 slots, e=64, Zipf(1.1) over 1e8
    keys: 6.55M occurrences, ~1.09M unique per step), too big for the f64
    oracle, checked through size-independent properties:
      * the table key set after each step is the union of the steps' unique
        keys (bit-exact, np.unique as the checker);
      * first touch from the fresh entry {w=0, acc=1e-6} (store.hpp:49) with
        AdaGrad (optimizer.cpp:86-95) gives acc = 1e-6 + g^2 and
        w = -lr g / sqrt(acc): g recovered from (w, acc) must satisfy
        acc = fl32(1e-6 + g^2) to 1.5 ulp of acc on every row (the
        per-key gradients are ~1e-8, so acc stays near 1e-6);
      * the second push touches only its own working set: rows of keys absent
        from batch 2 are bitwise unchanged."""
    lr = 0.05
    tr = kp.Trainer(table_capacity=1 << 22, n_workers=1, k=1, minibatch_size=65536,
                    embedding_dim=64, n_slots=100, hidden=[256, 128], sparse_lr=lr)
    b1 = make_batch(65536, V=10**8, zipf_s=1.1, n_slots=100, seed=20261018)
    r1 = tr.train_batch(b1.offs, b1.keys, b1.labels, slots=b1.slots)
    assert np.isfinite(r1["loss"]) and 0 < r1["loss"] < 2
    u1 = np.unique(b1.keys)
    assert len(u1) > 1_000_000
    k1, w1, a1, _ = tr.table()
    assert np.array_equal(k1, u1)
    w1 = np.asarray(w1, np.float64).reshape(len(k1), 64)
    a1 = np.asarray(a1, np.float64).reshape(len(k1), 64)
    # g recovered from w (w = -lr g / sqrt(acc) is relative-accurate), then
    # acc = fl32(1e-6 + g^2): one fp32 add of the square, <= 1 ulp of acc
    a0 = float(np.float32(1e-6))
    g = -w1 * np.sqrt(a1) / lr
    ulp = np.spacing(a1.astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(a1 - a0 - g * g) <= 1.5 * ulp + 1e-5 * g * g)
    # not vacuous: the hot keys' summed gradients (~1e-8 typical, larger for
    # hot keys) move acc by many ulps on ~19K of the 70M elements
    assert (g * g > 16 * ulp).sum() > 5000
    b2 = make_batch(65536, V=10**8, zipf_s=1.1, n_slots=100, seed=20261019)
    r2 = tr.train_batch(b2.offs, b2.keys, b2.labels, slots=b2.slots)
    assert np.isfinite(r2["loss"])
    k2, w2, _, _ = tr.table()
    assert np.array_equal(k2, np.union1d(u1, np.unique(b2.keys)))
    w2 = np.asarray(w2, np.float32).reshape(len(k2), 64)
    keep = ~np.isin(k1, b2.keys)
    assert keep.sum() > 100_000
    pos = np.searchsorted(k2, k1[keep])
    assert np.array_equal(w2[pos], w1[keep].astype(np.float32))


def test_trainer_errors(kp):
    with pytest.raises(kp.ConfigError):
        kp.Trainer(n_workers=1, k=0)
    tr = kp.Trainer(table_capacity=8, n_workers=1, embedding_dim=4, hidden=[])
    bt = make_batch(64, V=10**6, zipf_s=None, nnz=4, seed=0)
    with pytest.raises(kp.StoreError, match="table full"):
        tr.train_batch(bt.offs, bt.keys, bt.labels)
    tr2 = kp.Trainer(n_workers=1, embedding_dim=4, n_slots=2, hidden=[])
    bad = np.array([1, 0], np.uint16)
    with pytest.raises(kp.ConfigError, match="slot"):
        tr2.train_batch(np.array([0, 2], np.uint32), np.array([5, 6], np.uint64),
                        np.array([1], np.int32), slots=bad)


# ------------------------------------------------------------------- GEMM ---
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (300, 256, 6400), (65, 40, 100), (1000, 8, 96),
                                   (4096, 128, 256)])
def test_tcgen05_gemm_fp32_accuracy(kp, M, N, K):
    """3xTF32 tcgen05 GEMM vs an f64 numpy product: fp32-level error."""
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.sqrt(K)
    tc = kp.gemm_nt(A, B, engine=2)
    simt = kp.gemm_nt(A, B, engine=1)
    err_tc = np.max(np.abs(tc - want)) / scale
    err_simt = np.max(np.abs(simt - want)) / scale
    print(f"gemm M={M} N={N} K={K}: normalized max err tc={err_tc:.3e} simt={err_simt:.3e}")
    assert err_simt < 5e-5
    # 3xTF32 keeps fp32-level accuracy: within a small factor of the fp32 SIMT path
    assert err_tc < 3 * err_simt + 2e-6, (err_tc, err_simt)


@pytest.mark.parametrize("M,N,K,spread", [(128, 128, 32, 0), (300, 256, 6400, 0), (65, 40, 96, 0),
                                          (4096, 128, 256, 0), (1000, 256, 6400, 8), (512, 6400, 256, 4)])
def test_tcgen05_gemm_f16_scaled_accuracy(kp, M, N, K, spread):
    """fp16-operand GEMM (per-row power-of-two scales, hi*hi + hi*lo + lo*hi):
    fp32-level error like the 3xTF32 path, also with rows spanning 2^+-spread
    magnitudes, all-zero rows and tiny elements inside a row."""
    rng = np.random.default_rng(M * 7 + N + K + spread)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    if spread:
        A *= (2.0 ** rng.integers(-spread, spread + 1, (M, 1))).astype(np.float32)
        B *= (2.0 ** rng.integers(-spread, spread + 1, (N, 1))).astype(np.float32)
        A[0] = 0.0
        A[1, :K // 2] *= np.float32(1e-6)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.sqrt(K) * np.maximum(np.abs(A).max(1, keepdims=True), 1e-30) * np.abs(B).max(1)
    h = kp.gemm_nt(A, B, engine=3)
    simt = kp.gemm_nt(A, B, engine=1)
    err_h = np.max(np.abs(h - want) / scale)
    err_simt = np.max(np.abs(simt - want) / scale)
    print(f"gemm f16 M={M} N={N} K={K} spread={spread}: normalized err f16x3={err_h:.3e} simt={err_simt:.3e}")
    assert err_h < 3 * err_simt + 2e-6, (err_h, err_simt)


@pytest.mark.parametrize("M,N,K,spread,engine", [(128, 128, 32, 0, 4), (300, 256, 6400, 0, 4),
                                                 (1000, 256, 6400, 8, 4), (512, 6400, 256, 4, 4),
                                                 (65, 40, 96, 0, 4), (4096, 256, 6400, 3, 5),
                                                 (256, 384, 4096, 2, 5), (777, 208, 64, 1, 4),
                                                 (3000, 1000, 200, 2, 4), (65536, 6400, 256, 1, 4),
                                                 (65536, 256, 6400, 1, 6), (4096, 256, 6400, 3, 5),
                                                 (19456, 256, 512, 0, 6), (18944, 256, 64, 0, 6),
                                                 (20000, 300, 96, 2, 6)])
def test_h3_gemm_nt_accuracy(kp, M, N, K, spread, engine):
    """3xFP16 on pre-split fp16 planes (kp_gemm_h3.cu, the planes-mode first
    layer), both operands K-major; engine 5 = deterministic stream-K over K,
    6 = whole tiles for the full waves of 74 pairs + stream-K for the last
    partial wave (the forward's split): fp32-level error like the SIMT fp32
    GEMM, with rows spanning 2^+-spread, a zero row and tiny elements inside
    a row."""
    rng = np.random.default_rng(M * 3 + N + K + spread)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    if spread:
        A *= (2.0 ** rng.integers(-spread, spread + 1, (M, 1))).astype(np.float32)
        B *= (2.0 ** rng.integers(-spread, spread + 1, (N, 1))).astype(np.float32)
        A[0] = 0.0
        A[1, :K // 2] *= np.float32(1e-6)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.sqrt(K) * np.maximum(np.abs(A).max(1, keepdims=True), 1e-30) * np.abs(B).max(1)
    h = kp.gemm_nt(A, B, engine=engine)
    simt = kp.gemm_nt(A, B, engine=1)
    err_h = np.max(np.abs(h - want) / scale)
    err_simt = np.max(np.abs(simt - want) / scale)
    print(f"h3 nt M={M} N={N} K={K} spread={spread} e{engine}: err={err_h:.3e} simt={err_simt:.3e}")
    assert err_h < 3 * err_simt + 2e-6, (err_h, err_simt)
    if engine in (5, 6):  # deterministic: bitwise identical on a rerun
        assert np.array_equal(kp.gemm_nt(A, B, engine=engine), h)
    if engine == 6 and N <= 256:
        # the whole tiles (full waves of 74 pairs of 256 rows) are the
        # data-parallel kernel's, bit for bit
        whole = (M + 255) // 256 // 74 * 74 * 256
        h4 = kp.gemm_nt(A, B, engine=4)
        bad = np.nonzero(np.any(h[:whole] != h4[:whole], axis=1))[0]
        assert len(bad) == 0, (len(bad), bad[:8], np.unique(bad // 256)[:8])


@pytest.mark.parametrize("M,N,K,engine", [(256, 6400, 4096, 4), (256, 6400, 4096, 5), (128, 256, 65536, 5),
                                          (40, 104, 300, 4), (256, 512, 20000, 5), (64, 6400, 2048, 5),
                                          (16, 32, 70, 5), (40, 104, 300, 5), (256, 256, 4096, 5)])
def test_h3_gemm_tn_accuracy(kp, M, N, K, engine):
    """3xFP16 planes with both operands MN-major (the weight gradient dZ'^T X
    over the batch), one exponent per column, stream-K over the batch."""
    rng = np.random.default_rng(M * N + K + engine)
    A = rng.standard_normal((K, M)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    A *= (2.0 ** rng.integers(-3, 4, (1, M))).astype(np.float32)
    want = A.astype(np.float64).T @ B.astype(np.float64)
    scale = np.sqrt(K) * np.abs(A).max(0)[:, None] * np.abs(B).max(0)[None, :]
    tc = kp.gemm_tn(A, B, engine=engine)
    simt = kp.gemm_tn(A, B, engine=1)
    err_tc = np.max(np.abs(tc - want) / scale)
    err_simt = np.max(np.abs(simt - want) / scale)
    print(f"h3 tn M={M} N={N} K={K} e{engine}: err={err_tc:.3e} simt={err_simt:.3e}")
    assert err_tc < 3 * err_simt + 2e-6, (err_tc, err_simt)
    if engine == 5:
        # stream-K with fewer k-blocks than virtual units (K <= 4096): some
        # units own no range; a different shape in between must not leave
        # stale partials behind
        kp.gemm_tn(A[: K // 2 + 1], B[: K // 2 + 1], engine=5)
        assert np.array_equal(kp.gemm_tn(A, B, engine=5), tc)


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 6400, 4096), (128, 256, 65536), (40, 100, 300)])
def test_tcgen05_gemm_tn_fp32_accuracy(kp, M, N, K):
    """MN-major operands (the weight gradient dZ^T X over the batch), split-K."""
    rng = np.random.default_rng(M * N + K)
    A = rng.standard_normal((K, M)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    want = A.astype(np.float64).T @ B.astype(np.float64)
    scale = np.sqrt(K)
    tc = kp.gemm_tn(A, B, engine=2)
    simt = kp.gemm_tn(A, B, engine=1)
    err_tc = np.max(np.abs(tc - want)) / scale
    err_simt = np.max(np.abs(simt - want)) / scale
    print(f"gemm_tn M={M} N={N} K={K}: normalized max err tc={err_tc:.3e} simt={err_simt:.3e}")
    assert err_tc < 3 * err_simt + 2e-6, (err_tc, err_simt)


def test_staged_ingestion_matches_direct(kp):
    """Double-buffered H2D staging (kp_trainer_stage_batch/train_staged) trains
    bit-identically to the synchronous host path."""
    def run(staged):
        tr = kp.Trainer(table_capacity=1 << 18, n_workers=1, k=1, minibatch_size=2048,
                        embedding_dim=16, n_slots=8, hidden=[32])
        bts = [make_batch(2048, V=10**6, zipf_s=1.1, n_slots=8, seed=b) for b in range(3)]
        if staged:
            tr.stage_batch(0, bts[0].offs, bts[0].keys, bts[0].labels, slots=bts[0].slots)
            for b in range(3):
                if b + 1 < 3:
                    nb = bts[b + 1]
                    tr.stage_batch((b + 1) % 2, nb.offs, nb.keys, nb.labels, slots=nb.slots)
                tr.train_staged(b % 2, n_local=2048)
        else:
            for bt in bts:
                tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots)
        return tr.table(), tr.worker_state(0)["x"]
    (k1, w1, a1, _), x1 = run(False)
    (k2, w2, a2, _), x2 = run(True)
    assert np.array_equal(k1, k2) and np.array_equal(w1, w2) and np.array_equal(a1, a2)
    assert np.array_equal(x1, x2)


def test_staged_restage_and_lifetime(kp):
    """The staged H2D is issued lazily (after the running step's last host
    readback): re-staging a slot before training it replaces the batch, and
    the binding keeps the host arrays alive until train_staged returns even
    when the caller drops them."""
    import gc

    def mk(b):
        return make_batch(2048, V=10**6, zipf_s=1.1, n_slots=8, seed=100 + b)

    def direct(order):
        tr = kp.Trainer(table_capacity=1 << 18, n_workers=1, k=1, minibatch_size=2048,
                        embedding_dim=16, n_slots=8, hidden=[32])
        for b in order:
            bt = mk(b)
            tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots)
        return tr.table(), tr.worker_state(0)["x"]

    tr = kp.Trainer(table_capacity=1 << 18, n_workers=1, k=1, minibatch_size=2048,
                    embedding_dim=16, n_slots=8, hidden=[32])
    b0, b1, b2 = mk(0), mk(1), mk(2)
    tr.stage_batch(0, b0.offs, b0.keys, b0.labels, slots=b0.slots)
    tr.stage_batch(1, b1.offs, b1.keys, b1.labels, slots=b1.slots)
    # replace slot 1 with fresh copies the test then drops
    tr.stage_batch(1, b2.offs.copy(), b2.keys.copy(), b2.labels.copy(), slots=b2.slots.copy())
    gc.collect()
    tr.train_staged(0, n_local=2048)
    tr.train_staged(1, n_local=2048)
    (k1, w1, a1, _), x1 = (tr.table(), tr.worker_state(0)["x"])
    (k2, w2, a2, _), x2 = direct([0, 2])
    assert np.array_equal(k1, k2) and np.array_equal(w1, w2) and np.array_equal(a1, a2)
    assert np.array_equal(x1, x2)
    with pytest.raises(Exception):
        tr.train_staged(1, n_local=2048)  # consumed


@pytest.mark.parametrize("n,ties", [(2, False), (1000, True), (65536, False), (200_000, True)])
def test_device_auc_bit_exact(kp, n, ties):
    """Device rank-sum AUC == the reference's compute_auc on the same fp32 scores,
    bit for bit (all partial sums are exact half-integers in f64)."""
    rng = np.random.default_rng(n)
    s = (rng.integers(1, 25, n) / 25.0 if ties else rng.random(n)).astype(np.float32)
    y = rng.integers(0, 2, n).astype(np.int32)
    y[0], y[-1] = 0, 1
    want = O.orc_auc(s.astype(np.float64), y)
    assert kp.auc_device(s, y) == want
    if O.ref_available() and n <= 65536:
        assert kp.auc_device(s, y) == O.ref_auc(s.astype(np.float64), y)
    assert kp.auc_device(s, np.ones(n, np.int32)) is None
    with pytest.raises(kp.KpsimError, match="label"):
        kp.auc_device(s, np.full(n, 2, np.int32))


def test_trainer_online_auc_matches_host(kp):
    tr = kp.Trainer(table_capacity=1 << 16, n_workers=1, k=1, minibatch_size=512, embedding_dim=8,
                    hidden=[16], sparse_lr=0.3)
    scores, labels = [], []
    for b in range(3):
        bt = make_batch(512, V=5000, zipf_s=1.1, nnz=9, poisson=True, seed=b)
        r = tr.train_batch(bt.offs, bt.keys, bt.labels, predict_first=True)
        scores.append(r["preds"].astype(np.float64))
        labels.append(bt.labels)
        assert r["auc"] == O.orc_auc(scores[-1], bt.labels)
        assert r["cumulative_auc"] == O.orc_auc(np.concatenate(scores), np.concatenate(labels))


@pytest.mark.parametrize("B,S,e,pool,workers,hidden", [(4096, 100, 64, "sum", 1, (256, 128)),
                                                       (3000, 26, 32, "mean", 2, (64, 32)),
                                                       (20000, 100, 64, "sum", 1, (256, 128)),
                                                       (1000, 12, 96, "sum", 1, (264, 16)),
                                                       (1000, 12, 96, "sum", 1, (300, 16))])
def test_fused_pool_gather_bitwise(kp, monkeypatch, B, S, e, pool, workers, hidden):
    """One feature per slot: the first layer's forward fetches the table rows
    itself (TMA gather4 into its pipeline, split into fp16 planes on chip, the
    planes stored for the weight gradient) instead of a pooling pass. Same
    exponents, same planes, same GEMM: every trained bit (table rows and
    accumulators, dense x, losses, predictions) equals the pooling-pass path
    (the default). Covers the hybrid stream-K split (20000 rows: 79 tiles),
    W=2 worker slices, mean pooling and N > 256 (two column tiles); hidden
    300 (rows of 600 bytes) takes neither planes path (it used to fail the
    backward's tensor-map encode)."""
    out = []
    monkeypatch.setenv("KP_TC_MIN_MFLOP", "0")  # the planes path at every size here
    for fused in ("1", "0"):
        monkeypatch.setenv("KP_FUSED_POOL", fused)  # read at trainer creation
        cfg = O.TrainerCfg(n_workers=workers, k=2, minibatch_size=B, embedding_dim=e, n_slots=S,
                           hidden=hidden, pooling=pool, activation="relu", alpha=0.02, sparse_lr=0.1)
        tr = kp.Trainer(table_capacity=1 << 20, **trainer_kwargs(vars(cfg)))
        losses, preds = [], []
        for b in range(3):
            bt = make_batch(B, V=10**6, zipf_s=1.1, n_slots=S, seed=300 + b)
            r = tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=True)
            losses.append(r["loss"])
            preds.append(np.asarray(r["preds"]).copy() if "preds" in r else None)
        k, w, s1, _ = tr.table()
        out.append((losses, preds, k, w, s1, tr.worker_state(0)["x"]))
    (l1, p1, k1, w1, a1, x1), (l0, p0, k0, w0, a0, x0) = out
    assert l1 == l0
    for a, b in zip(p1, p0):
        assert (a is None and b is None) or np.array_equal(a, b)
    assert np.array_equal(k1, k0)
    assert np.array_equal(w1, w0)
    assert np.array_equal(a1, a0)
    assert np.array_equal(x1, x0)


@pytest.mark.parametrize("B,hidden,workers", [(1000, (128, 32), 1), (4096, (256,), 2), (777, (384, 64, 16), 1)])
def test_split_rows_colmax_fused_bitwise(kp, monkeypatch, B, hidden, workers):
    """The first layer's backward splits dZ1 for the input gradient (per row)
    and takes dW's column scales and the bias-gradient partials from the SAME
    read of dZ1 (k_rows_colmax) instead of two passes (KP_SPLIT_FUSE=0): every
    trained bit equals the two-pass path. Ragged row counts, one and several
    hidden layers (bias partials off / on), W=2 worker slices."""
    out = []
    monkeypatch.setenv("KP_TC_MIN_MFLOP", "0")  # the planes path at every size here
    for fuse in ("1", "0"):
        monkeypatch.setenv("KP_SPLIT_FUSE", fuse)
        cfg = O.TrainerCfg(n_workers=workers, k=2, minibatch_size=B, embedding_dim=16, n_slots=8,
                           hidden=hidden, pooling="sum", activation="relu", alpha=0.02, sparse_lr=0.1)
        tr = kp.Trainer(table_capacity=1 << 20, **trainer_kwargs(vars(cfg)))
        losses = []
        for b in range(3):
            bt = make_batch(B, V=10**5, zipf_s=1.1, n_slots=8, seed=700 + b)
            losses.append(tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots)["loss"])
        k, w, s1, _ = tr.table()
        out.append((losses, k, w, s1, tr.worker_state(0)["x"]))
    (l1, k1, w1, a1, x1), (l0, k0, w0, a0, x0) = out
    assert l1 == l0
    assert np.array_equal(k1, k0)
    assert np.array_equal(w1, w0)
    assert np.array_equal(a1, a0)
    assert np.array_equal(x1, x0)


@pytest.mark.parametrize("B,S,e,zipf,V", [(4096, 26, 8, 1.1, 10**6), (8192, 26, 8, 1.3, 100), (6000, 16, 16, 1.2, 500)])
def test_seg_blocksum_one_launch_bitwise(kp, monkeypatch, B, S, e, zipf, V):
    """Small rows (e <= 16): the push's two block-sum levels (64-partial sums
    Q, then 64-Q sums Q2 for the hottest keys) run as one launch; every
    trained bit equals the two-launch path (KP_SEG_BS12=0). V=100 at Zipf 1.3
    puts one key on ~60K sorted positions, so the Q2 level is exercised."""
    out = []
    for one in ("1", "0"):
        monkeypatch.setenv("KP_SEG_BS12", one)
        cfg = O.TrainerCfg(n_workers=1, k=1, minibatch_size=B, embedding_dim=e, n_slots=S,
                           hidden=(32,), pooling="sum", activation="relu", alpha=0.02, sparse_lr=0.1)
        tr = kp.Trainer(table_capacity=1 << 20, **trainer_kwargs(vars(cfg)))
        losses = []
        for b in range(3):
            bt = make_batch(B, V=V, zipf_s=zipf, n_slots=S, seed=950 + b)
            losses.append(tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots)["loss"])
        k, w, s1, _ = tr.table()
        out.append((losses, k, w, s1, tr.worker_state(0)["x"]))
    (l1, k1, w1, a1, x1), (l0, k0, w0, a0, x0) = out
    assert l1 == l0
    assert np.array_equal(k1, k0)
    assert np.array_equal(w1, w0)
    assert np.array_equal(a1, a0)
    assert np.array_equal(x1, x0)


def _train_n(kp, monkeypatch, sync_free, batches, S=8, e=16, hidden=(32, 16), B=None):
    monkeypatch.setenv("KP_SYNC_FREE", sync_free)  # read at trainer creation
    cfg = O.TrainerCfg(n_workers=1, k=1, minibatch_size=B or len(batches[0].labels), embedding_dim=e,
                       n_slots=S, hidden=hidden, pooling="sum", activation="relu", alpha=0.02, sparse_lr=0.1)
    tr = kp.Trainer(table_capacity=1 << 18, **trainer_kwargs(vars(cfg)))
    losses = []
    for bt in batches:
        r = tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=True)
        losses.append((r["loss"], np.asarray(r["preds"]).copy()))
    return tr, losses


@pytest.mark.parametrize("S,e,tc_min", [(8, 16, None), (20, 64, "0")])
def test_sync_free_step_replans_bitwise(kp, monkeypatch, S, e, tc_min):
    """The single-GPU step without the dedup readback (pass plan and the
    one-feature-per-slot layout predicted from the previous batch, checked on
    the device): a batch whose key span outgrows the plan (1e3 -> 1e12 keys),
    one that switches to multi-hot bags (the layout prediction fails) and
    back are rerun with the readbacks -- every result and every trained bit
    equals the always-readback trainer (KP_SYNC_FREE=0). The second case runs
    the planes path, where a predicted one-feature batch skips writing the
    (identity) bag maps."""
    if tc_min is not None:
        monkeypatch.setenv("KP_TC_MIN_MFLOP", tc_min)

    def mk(V, seed, multi=False):
        bt = make_batch(512, V=V, zipf_s=1.1, n_slots=S, seed=seed)
        if multi:  # two features in every slot
            bt.keys = np.repeat(bt.keys, 2)
            bt.slots = np.repeat(bt.slots, 2)
            bt.offs = (bt.offs.astype(np.int64) * 2).astype(bt.offs.dtype)
        return bt
    batches = [mk(10**3, 1), mk(10**3, 2), mk(10**12, 3), mk(10**12, 4, multi=True), mk(10**4, 5),
               mk(10**4, 6)]
    t1, r1 = _train_n(kp, monkeypatch, "1", batches, S=S, e=e)
    t0, r0 = _train_n(kp, monkeypatch, "0", batches, S=S, e=e)
    for (l1, p1), (l0, p0) in zip(r1, r0):
        assert l1 == l0
        assert np.array_equal(p1, p0)
    k1, w1, a1, _ = t1.table()
    k0, w0, a0, _ = t0.table()
    assert np.array_equal(k1, k0) and np.array_equal(w1, w0) and np.array_equal(a1, a0)
    assert np.array_equal(t1.worker_state(0)["x"], t0.worker_state(0)["x"])


def test_sync_free_step_bad_slot_writes_nothing(kp, monkeypatch):
    """A bad slot id on a sync-free step is found after the fact (no readback
    before the state writes): the guarded kernels wrote nothing, the call
    raises ConfigError, and training continues exactly like the trainer that
    never saw the bad batch."""
    good = [make_batch(512, V=10**5, zipf_s=1.1, n_slots=8, seed=20 + i) for i in range(3)]
    bad = make_batch(512, V=10**5, zipf_s=1.1, n_slots=8, seed=30)
    bad.slots = bad.slots.copy()
    bad.slots[100] = 9  # >= n_slots
    monkeypatch.setenv("KP_SYNC_FREE", "1")
    cfg = O.TrainerCfg(n_workers=1, k=1, minibatch_size=512, embedding_dim=16, n_slots=8, hidden=(32, 16),
                       pooling="sum", activation="relu", alpha=0.02, sparse_lr=0.1)
    ta = kp.Trainer(table_capacity=1 << 18, **trainer_kwargs(vars(cfg)))
    tb = kp.Trainer(table_capacity=1 << 18, **trainer_kwargs(vars(cfg)))
    ra = [ta.train_batch(good[0].offs, good[0].keys, good[0].labels, slots=good[0].slots)["loss"]]
    ra.append(ta.train_batch(good[1].offs, good[1].keys, good[1].labels, slots=good[1].slots)["loss"])
    with pytest.raises(ValueError):
        ta.train_batch(bad.offs, bad.keys, bad.labels, slots=bad.slots)
    ra.append(ta.train_batch(good[2].offs, good[2].keys, good[2].labels, slots=good[2].slots)["loss"])
    rb = [tb.train_batch(g.offs, g.keys, g.labels, slots=g.slots)["loss"] for g in good]
    assert ra == rb
    ka, wa, aa, _ = ta.table()
    kb, wb, ab, _ = tb.table()
    assert np.array_equal(ka, kb) and np.array_equal(wa, wb) and np.array_equal(aa, ab)
    assert np.array_equal(ta.worker_state(0)["x"], tb.worker_state(0)["x"])


def test_sync_free_predict_pass_bitwise(kp, monkeypatch):
    """Predict-then-train between merges (k = 3, two local workers: the
    replicas differ, so the predictions take their own pull + x-bar forward
    before the training step) on the sync-free step, with a plan miss in the
    middle: predictions, losses and state equal the always-readback
    trainer's bit for bit."""
    out = []
    for sf in ("1", "0"):
        monkeypatch.setenv("KP_SYNC_FREE", sf)
        cfg = O.TrainerCfg(n_workers=2, k=3, minibatch_size=256, embedding_dim=16, n_slots=8,
                           hidden=(32, 16), pooling="sum", activation="relu", alpha=0.02, sparse_lr=0.1)
        tr = kp.Trainer(table_capacity=1 << 18, **trainer_kwargs(vars(cfg)))
        res = []
        for b, V in enumerate([10**3, 10**3, 10**3, 10**12, 10**12, 10**4, 10**4]):
            bt = make_batch(512, V=V, zipf_s=1.1, n_slots=8, seed=60 + b)
            r = tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=True)
            res.append((r["loss"], np.asarray(r["preds"]).copy()))
        k, w, a, _ = tr.table()
        out.append((res, k, w, a, tr.worker_state(0)["x"], tr.worker_state(1)["x"]))
    (r1, k1, w1, a1, x1, y1), (r0, k0, w0, a0, x0, y0) = out
    for (l1, p1), (l0, p0) in zip(r1, r0):
        assert l1 == l0 and np.array_equal(p1, p0)
    assert np.array_equal(k1, k0) and np.array_equal(w1, w0) and np.array_equal(a1, a0)
    assert np.array_equal(x1, x0) and np.array_equal(y1, y0)


def test_graph_replay_bitwise(kp, monkeypatch):
    """The sync-free batch captured as a CUDA graph on the second sight of a
    batch shape and replayed after (different batch contents through the
    same input buffers, merge and non-merge steps at k = 2, predictions):
    every result and trained bit equals the directly launched batch
    (KP_GRAPH=0)."""
    out = []
    for g in ("1", "0"):
        monkeypatch.setenv("KP_GRAPH", g)
        cfg = O.TrainerCfg(n_workers=1, k=2, minibatch_size=2048, embedding_dim=64, n_slots=20,
                           hidden=(64, 32), pooling="sum", activation="relu", alpha=0.02, sparse_lr=0.1)
        tr = kp.Trainer(table_capacity=1 << 20, **trainer_kwargs(vars(cfg)))
        res = []
        for b in range(8):
            bt = make_batch(2048, V=10**6, zipf_s=1.1, n_slots=20, seed=80 + b)
            r = tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=True)
            res.append((r["loss"], np.asarray(r["preds"]).copy(), r["minibatch_steps"], r["merges"]))
        k, w, a, _ = tr.table()
        out.append((res, k, w, a, tr.worker_state(0)))
    (r1, k1, w1, a1, s1), (r0, k0, w0, a0, s0) = out
    for x, y in zip(r1, r0):
        assert x[0] == y[0] and np.array_equal(x[1], y[1]) and x[2:] == y[2:]
    assert np.array_equal(k1, k0) and np.array_equal(w1, w0) and np.array_equal(a1, a0)
    for f in ("x", "m", "v", "v_bar"):
        assert np.array_equal(s1[f], s0[f]), f
