"""TEST INFRASTRUCTURE ONLY: ctypes handles on the parity checkers in oracle/_ref.

- ``Ref``: the unmodified reference (``libkpsim_ref.so``: /root/reference/proj/src
  compiled by oracle/Makefile + ``ref_driver.cpp``).
- ``Orc``: the plain-C restatement (``kpsim_oracle.c``) in f64 (``bits=64``,
  pinned bit-exact against ``Ref``) or f32 (``bits=32``, tolerance envelope).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu-baseline leg may import
this module. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import functools
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


def build(quiet: bool = True) -> None:
    """Compile the checkers (the reference part only when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


@functools.lru_cache(maxsize=None)
def _lib(name: str) -> C.CDLL:
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


def ref_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libkpsim_ref.so"))


class TrainerCfg:
    """Field names follow kpsim::TrainerConfig / ModelConfig / AdamHyper."""

    def __init__(self, *, seed=42, n_workers=1, minibatch_size=128, sparse_lr=0.05,
                 alpha=0.01, beta1=0.0, beta2=0.999, epsilon=0.01, k=1, reset_local_v=True,
                 embedding_dim=8, n_slots=1, hidden=(16,), activation="relu", pooling="sum",
                 sparse_rule="adagrad", sparse_beta1=0.9, sparse_beta2=0.999, sparse_eps=1e-8,
                 vocab=1 << 40):
        self.seed, self.n_workers, self.minibatch_size = seed, n_workers, minibatch_size
        self.sparse_lr, self.alpha, self.beta1, self.beta2 = sparse_lr, alpha, beta1, beta2
        self.epsilon, self.k, self.reset_local_v = epsilon, k, reset_local_v
        self.embedding_dim, self.n_slots, self.hidden = embedding_dim, n_slots, tuple(hidden)
        self.activation, self.pooling, self.sparse_rule = activation, pooling, sparse_rule
        self.sparse_beta1, self.sparse_beta2, self.sparse_eps = sparse_beta1, sparse_beta2, sparse_eps
        self.vocab = vocab

    def dense_dim(self) -> int:
        w = [self.embedding_dim * self.n_slots, *self.hidden, 1]
        return sum(w[i] * w[i + 1] + w[i + 1] for i in range(len(w) - 1))


class _OrcConfig(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_workers", C.c_uint64), ("minibatch", C.c_uint64),
                ("sparse_lr", C.c_double), ("alpha", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("k", C.c_uint64),
                ("reset_v", C.c_int32), ("emb_dim", C.c_uint64), ("n_slots", C.c_uint64),
                ("hidden", C.c_uint64 * 8), ("n_hidden", C.c_int32), ("activation", C.c_int32),
                ("pooling", C.c_int32), ("sparse_rule", C.c_int32),
                ("sparse_beta1", C.c_double), ("sparse_beta2", C.c_double),
                ("sparse_eps", C.c_double)]


class Orc:
    """The C restatement's trainer (f64 or f32)."""

    def __init__(self, cfg: TrainerCfg, bits: int = 64):
        self.lib = _lib(f"liborc{bits}.so")
        p = f"orc{bits}_"
        self.p = p
        L = self.lib
        getattr(L, p + "trainer_create").restype = C.c_void_p
        getattr(L, p + "trainer_create").argtypes = [C.POINTER(_OrcConfig)]
        getattr(L, p + "trainer_destroy").argtypes = [C.c_void_p]
        getattr(L, p + "trainer_batch").argtypes = [
            C.c_void_p, _u64p, _u64p, C.c_void_p, _i32p, C.c_uint64, C.c_int,
            C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p]
        getattr(L, p + "trainer_dense_dim").restype = C.c_uint64
        getattr(L, p + "trainer_dense_dim").argtypes = [C.c_void_p]
        getattr(L, p + "trainer_steps").restype = C.c_uint64
        getattr(L, p + "trainer_steps").argtypes = [C.c_void_p]
        getattr(L, p + "trainer_merges").restype = C.c_uint64
        getattr(L, p + "trainer_merges").argtypes = [C.c_void_p]
        getattr(L, p + "trainer_worker_state").argtypes = [C.c_void_p, C.c_uint64, _f64p, _f64p, _f64p, _f64p]
        getattr(L, p + "trainer_table_size").restype = C.c_uint64
        getattr(L, p + "trainer_table_size").argtypes = [C.c_void_p]
        getattr(L, p + "trainer_table").argtypes = [C.c_void_p, _u64p, _f64p, _f64p, C.c_void_p]
        c = _OrcConfig()
        c.seed, c.n_workers, c.minibatch = cfg.seed, cfg.n_workers, cfg.minibatch_size
        c.sparse_lr, c.alpha, c.beta1, c.beta2 = cfg.sparse_lr, cfg.alpha, cfg.beta1, cfg.beta2
        c.eps, c.k, c.reset_v = cfg.epsilon, cfg.k, int(cfg.reset_local_v)
        c.emb_dim, c.n_slots = cfg.embedding_dim, cfg.n_slots
        for i, h in enumerate(cfg.hidden):
            c.hidden[i] = h
        c.n_hidden = len(cfg.hidden)
        c.activation = 1 if cfg.activation == "tanh" else 0
        c.pooling = 1 if cfg.pooling == "mean" else 0
        c.sparse_rule = 1 if cfg.sparse_rule == "adam" else 0
        c.sparse_beta1, c.sparse_beta2, c.sparse_eps = cfg.sparse_beta1, cfg.sparse_beta2, cfg.sparse_eps
        self.cfg = cfg
        self.h = getattr(L, p + "trainer_create")(C.byref(c))

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self.lib, self.p + "trainer_destroy")(self.h)
            self.h = None

    def batch(self, offs, keys, labels, slots=None, predict_first=False, want_preds=False):
        offs = np.ascontiguousarray(offs, np.uint64)
        keys = np.ascontiguousarray(keys, np.uint64)
        labels = np.ascontiguousarray(labels, np.int32)
        n = len(offs) - 1
        sl = None
        if slots is not None:
            slots = np.ascontiguousarray(slots, np.uint16)
            sl = slots.ctypes.data_as(C.c_void_p)
        preds = np.zeros(n, np.float64) if want_preds else None
        loss, auc, cum = C.c_double(), C.c_double(), C.c_double()
        rc = getattr(self.lib, self.p + "trainer_batch")(
            self.h, offs, keys, sl, labels, n, int(predict_first), C.byref(loss), C.byref(auc),
            C.byref(cum), preds.ctypes.data_as(C.c_void_p) if preds is not None else None)
        if rc:
            raise RuntimeError("oracle batch failed")
        out = {"loss": loss.value, "auc": auc.value, "cumulative_auc": cum.value}
        if preds is not None:
            out["preds"] = preds
        return out

    def dense_dim(self):
        return int(getattr(self.lib, self.p + "trainer_dense_dim")(self.h))

    def steps(self):
        return int(getattr(self.lib, self.p + "trainer_steps")(self.h))

    def merges(self):
        return int(getattr(self.lib, self.p + "trainer_merges")(self.h))

    def worker_state(self, i):
        D = self.dense_dim()
        x, m, v, vb = (np.zeros(D) for _ in range(4))
        if getattr(self.lib, self.p + "trainer_worker_state")(self.h, i, x, m, v, vb):
            raise IndexError(i)
        return {"x": x, "m": m, "v": v, "v_bar": vb}

    def table(self):
        n = int(getattr(self.lib, self.p + "trainer_table_size")(self.h))
        e = self.cfg.embedding_dim
        keys = np.zeros(n, np.uint64)
        w, s1, s2 = np.zeros(n * e), np.zeros(n * e), np.zeros(n * e)
        getattr(self.lib, self.p + "trainer_table")(self.h, keys, w, s1, s2.ctypes.data_as(C.c_void_p))
        return keys, w.reshape(n, e), s1.reshape(n, e), s2.reshape(n, e)


def orc_fn(bits: int, name: str):
    return getattr(_lib(f"liborc{bits}.so"), f"orc{bits}_{name}")


def orc_dedup(keys, bits=64):
    keys = np.ascontiguousarray(keys, np.uint64)
    f = orc_fn(bits, "dedup")
    f.restype = C.c_uint64
    f.argtypes = [_u64p, C.c_uint64, _u64p, _u32p]
    uniq = np.zeros(max(len(keys), 1), np.uint64)
    inv = np.zeros(max(len(keys), 1), np.uint32)
    u = f(keys, len(keys), uniq, inv)
    return uniq[:u], inv[:len(keys)]


def orc_shard(unique, G, bits=64):
    unique = np.ascontiguousarray(unique, np.uint64)
    f = orc_fn(bits, "shard")
    f.argtypes = [_u64p, C.c_uint64, C.c_uint32, _u32p, _u64p]
    perm = np.zeros(max(len(unique), 1), np.uint32)
    counts = np.zeros(G, np.uint64)
    f(unique, len(unique), G, perm, counts)
    return perm[:len(unique)], counts


def orc_init_dense(seed, dim):
    f = orc_fn(64, "init_dense")
    f.argtypes = [C.c_uint64, C.c_uint64, _f64p]
    out = np.zeros(dim)
    f(seed, dim, out)
    return out


def orc_auc(scores, labels):
    f = orc_fn(64, "auc")
    f.restype = C.c_double
    f.argtypes = [_f64p, _i32p, C.c_uint64]
    return f(np.ascontiguousarray(scores, np.float64), np.ascontiguousarray(labels, np.int32), len(scores))


def orc_kstep(bits, alpha, beta1, beta2, eps, k, workers, x0, grads, reset_v=True):
    """grads: [steps][workers][dim] -> dict of [steps][workers][dim] arrays."""
    grads = np.ascontiguousarray(grads, np.float64)
    steps, W, dim = grads.shape
    f = orc_fn(bits, "kstep_run")
    f.argtypes = [C.c_double] * 4 + [C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, _f64p,
                                     C.c_uint64, _f64p, _f64p, _f64p, _f64p, _f64p, _i32p]
    xs, ms, vs, vb = (np.zeros((steps, W, dim)) for _ in range(4))
    merged = np.zeros(steps, np.int32)
    f(alpha, beta1, beta2, eps, k, int(reset_v), W, dim, np.ascontiguousarray(x0, np.float64),
      steps, grads, xs, ms, vs, vb, merged)
    return {"x": xs, "m": ms, "v": vs, "v_bar": vb, "merged": merged}


class Ref:
    """The compiled reference's Trainer (f64), driven through ref_driver.cpp."""

    def __init__(self, cfg: TrainerCfg, cold_dir: str):
        if cfg.n_slots != 1 or cfg.sparse_rule != "adagrad":
            raise ValueError("the reference supports S=1 and AdaGrad only")
        L = _lib("libkpsim_ref.so")
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_trainer_create.restype = C.c_void_p
        L.ref_trainer_create.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                         C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                         C.c_int, C.c_uint64, _u64p, C.c_int, C.c_int, C.c_int,
                                         C.c_uint64]
        L.ref_trainer_destroy.argtypes = [C.c_void_p]
        L.ref_trainer_batch.argtypes = [C.c_void_p, _u64p, _u64p, _i32p, C.c_uint64, C.c_uint64,
                                        C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
        L.ref_trainer_dense_dim.restype = C.c_uint64
        L.ref_trainer_dense_dim.argtypes = [C.c_void_p]
        L.ref_trainer_steps.restype = C.c_uint64
        L.ref_trainer_steps.argtypes = [C.c_void_p]
        L.ref_trainer_merges.restype = C.c_uint64
        L.ref_trainer_merges.argtypes = [C.c_void_p]
        L.ref_trainer_worker_state.argtypes = [C.c_void_p, C.c_uint64, _f64p, _f64p, _f64p, _f64p]
        L.ref_trainer_xbar.argtypes = [C.c_void_p, _f64p]
        L.ref_trainer_table_size.restype = C.c_uint64
        L.ref_trainer_table_size.argtypes = [C.c_void_p]
        L.ref_trainer_table.argtypes = [C.c_void_p, _u64p, _f64p, _f64p]
        L.ref_trainer_trajectory.argtypes = [C.c_void_p, C.c_uint64, _f64p, _f64p, C.POINTER(C.c_double)]
        hid = np.array(list(cfg.hidden) or [0], np.uint64)
        self.cfg = cfg
        self.h = L.ref_trainer_create(cold_dir.encode(), cfg.seed, cfg.n_workers, cfg.minibatch_size,
                                      cfg.sparse_lr, cfg.alpha, cfg.beta1, cfg.beta2, cfg.epsilon,
                                      cfg.k, int(cfg.reset_local_v), cfg.embedding_dim, hid,
                                      len(cfg.hidden), 1 if cfg.activation == "tanh" else 0,
                                      1 if cfg.pooling == "mean" else 0, min(cfg.vocab, (1 << 63)))
        if not self.h:
            raise RuntimeError(L.ref_last_error().decode())
        self.batch_id = 0

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_trainer_destroy(self.h)
            self.h = None

    def batch(self, offs, keys, labels, predict_first=False):
        offs = np.ascontiguousarray(offs, np.uint64)
        keys = np.ascontiguousarray(keys, np.uint64)
        labels = np.ascontiguousarray(labels, np.int32)
        loss, auc, cum = C.c_double(), C.c_double(), C.c_double()
        rc = self.lib.ref_trainer_batch(self.h, offs, keys, labels, len(offs) - 1, self.batch_id,
                                        int(predict_first), C.byref(loss), C.byref(auc), C.byref(cum))
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
        self.batch_id += 1
        return {"loss": loss.value, "auc": auc.value, "cumulative_auc": cum.value}

    def dense_dim(self):
        return int(self.lib.ref_trainer_dense_dim(self.h))

    def steps(self):
        return int(self.lib.ref_trainer_steps(self.h))

    def merges(self):
        return int(self.lib.ref_trainer_merges(self.h))

    def worker_state(self, i):
        D = self.dense_dim()
        x, m, v, vb = (np.zeros(D) for _ in range(4))
        if self.lib.ref_trainer_worker_state(self.h, i, x, m, v, vb):
            raise IndexError(i)
        return {"x": x, "m": m, "v": v, "v_bar": vb}

    def xbar(self):
        out = np.zeros(self.dense_dim())
        self.lib.ref_trainer_xbar(self.h, out)
        return out

    def trajectory(self, step):
        D = self.dense_dim()
        xb, vb, loss = np.zeros(D), np.zeros(D), C.c_double()
        if self.lib.ref_trainer_trajectory(self.h, step, xb, vb, C.byref(loss)):
            raise IndexError(step)
        f = self.lib.ref_trainer_trajectory_flags
        f.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_double),
                      C.POINTER(C.c_uint64)]
        merged, a3, n = C.c_int(), C.c_double(), C.c_uint64()
        f(self.h, step, C.byref(merged), C.byref(a3), C.byref(n))
        return {"x_bar": xb, "v_bar": vb, "loss": loss.value, "merged": bool(merged.value),
                "a3_increment": a3.value, "n_steps": n.value}

    def table(self):
        n = int(self.lib.ref_trainer_table_size(self.h))
        e = self.cfg.embedding_dim
        keys = np.zeros(max(n, 1), np.uint64)
        w, acc = np.zeros(max(n, 1) * e), np.zeros(max(n, 1) * e)
        if self.lib.ref_trainer_table(self.h, keys, w, acc):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return keys[:n], w[:n * e].reshape(n, e), acc[:n * e].reshape(n, e)


def ref_fn(name):
    return getattr(_lib("libkpsim_ref.so"), name)


def ref_dedup(keys):
    f = ref_fn("ref_dedup")
    f.restype = C.c_uint64
    f.argtypes = [_u64p, C.c_uint64, _u64p]
    keys = np.ascontiguousarray(keys, np.uint64)
    out = np.zeros(max(len(keys), 1), np.uint64)
    return out[:f(keys, len(keys), out)]


def ref_init_dense(embedding_dim, hidden, seed):
    f = ref_fn("ref_init_dense")
    f.argtypes = [C.c_uint64, _u64p, C.c_int, C.c_uint64, C.c_void_p, C.POINTER(C.c_uint64)]
    hid = np.array(list(hidden) or [0], np.uint64)
    d = C.c_uint64()
    f(embedding_dim, hid, len(hidden), seed, None, C.byref(d))
    out = np.zeros(d.value)
    f(embedding_dim, hid, len(hidden), seed, out.ctypes.data_as(C.c_void_p), C.byref(d))
    return out


def ref_kstep(alpha, beta1, beta2, eps, k, workers, x0, grads, reset_v=True):
    grads = np.ascontiguousarray(grads, np.float64)
    steps, W, dim = grads.shape
    f = ref_fn("ref_kstep")
    f.argtypes = [C.c_double] * 4 + [C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, _f64p,
                                     C.c_uint64, _f64p, _f64p, _f64p, _f64p, _f64p, _i32p]
    xs, ms, vs, vb = (np.zeros((steps, W, dim)) for _ in range(4))
    merged = np.zeros(steps, np.int32)
    if f(alpha, beta1, beta2, eps, k, int(reset_v), W, dim, np.ascontiguousarray(x0, np.float64),
         steps, grads, xs, ms, vs, vb, merged):
        raise RuntimeError("ref_kstep failed")
    return {"x": xs, "m": ms, "v": vs, "v_bar": vb, "merged": merged}


def ref_adagrad(w, acc, g, lr):
    f = ref_fn("ref_adagrad")
    f.argtypes = [_f64p, _f64p, _f64p, C.c_uint64, C.c_double]
    w = np.array(w, np.float64)
    acc = np.array(acc, np.float64)
    f(w, acc, np.ascontiguousarray(g, np.float64), len(w), lr)
    return w, acc


def ref_auc(scores, labels):
    f = ref_fn("ref_auc")
    f.restype = C.c_double
    f.argtypes = [_f64p, _i32p, C.c_uint64]
    return f(np.ascontiguousarray(scores, np.float64), np.ascontiguousarray(labels, np.int32), len(scores))


def _ref_csr(fn, *args):
    """Two-call CSR export from the compiled reference (sizes, then data)."""
    n, nnz = C.c_uint64(), C.c_uint64()
    if fn(*args, None, None, None, C.byref(n), C.byref(nnz)):
        raise RuntimeError(ref_fn("ref_last_error")().decode())
    offs = np.zeros(n.value + 1, np.uint64)
    keys = np.zeros(max(nnz.value, 1), np.uint64)
    labels = np.zeros(max(n.value, 1), np.int32)
    if fn(*args, offs.ctypes.data_as(C.c_void_p), keys.ctypes.data_as(C.c_void_p),
          labels.ctypes.data_as(C.c_void_p), C.byref(n), C.byref(nnz)):
        raise RuntimeError(ref_fn("ref_last_error")().decode())
    return offs, keys[:nnz.value], labels[:n.value]


def ref_synthetic(seed=42, n_instances=100000, vocab=10000, nnz_mean=10.0, signal_scale=4.0):
    """The reference's SyntheticCtr stream (proj/src/data.cpp:11-57) as CSR
    (offs u64[n+1], keys u64[nnz], labels i32[n]) -- the desk benchmark's
    data when called with ExperimentConfig::defaults() (config.hpp:18-30)."""
    f = ref_fn("ref_synthetic")
    f.restype = C.c_int
    f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_double] + [C.c_void_p] * 3 + \
        [C.POINTER(C.c_uint64)] * 2
    ref_fn("ref_last_error").restype = C.c_char_p
    return _ref_csr(f, seed, n_instances, vocab, nnz_mean, signal_scale)


def ref_read_instances(path):
    """read_instances (proj/src/data.cpp:72-110) through the compiled reference;
    raises RuntimeError with the reference's message on a malformed file."""
    f = ref_fn("ref_read_instances")
    f.restype = C.c_int
    f.argtypes = [C.c_char_p] + [C.c_void_p] * 3 + [C.POINTER(C.c_uint64)] * 2
    ref_fn("ref_last_error").restype = C.c_char_p
    return _ref_csr(f, str(path).encode())
