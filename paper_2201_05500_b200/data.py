"""Synthetic Zipf CTR batches in the hot path's CSR layout (host side).

The reference generator draws keys uniformly (proj/src/data.cpp:30,36); the
north star asks for Zipf(s) keys, so batches are generated here and fed to both
sides (the reference reads the same instances through its Instance/Batch types,
proj/include/kpsim/data.hpp:14-22).

Layout (what the C-ABI consumes):
  offs[B+1]  uint32  CSR over occurrences, instance-major
  keys[O]    uint64  feature ids; with S=1 each instance's ids are sorted and
                     unique (read_instances semantics, proj/src/data.cpp:153-168)
  slots[O]   uint16  slot id per occurrence (None => S=1), non-decreasing within
                     an instance
  labels[B]  int32   0/1, planted logistic model (like proj/src/data.cpp:22-43)

Zipf ranks use rejection-inversion sampling (Hoermann & Derflinger 1996), exact
for the pmf k^-s on {1..V}. Rank r maps to key (A*r + C) mod V with gcd(A,V)=1:
a bijection on [0,V), so hot ranks spread round-robin over key % G shards.
"""
from __future__ import annotations

import math

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """proj/include/kpsim/common.hpp:54-59, vectorised (uint64 wraps)."""
    with np.errstate(over="ignore"):
        x = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


class ZipfSampler:
    """Exact Zipf(s) on {1..V} by rejection-inversion; returns 0-based ranks."""

    def __init__(self, V: int, s: float):
        if V < 1 or s <= 0:
            raise ValueError("need V >= 1 and s > 0")
        self.V, self.s = int(V), float(s)
        self.hx1 = self._H(1.5) - 1.0
        self.hn = self._H(self.V + 0.5)
        self.sq = 2.0 - self._Hinv(self._H(2.5) - self._h(2.0))

    def _helper1(self, x):  # log1p(x)/x
        x = np.asarray(x, np.float64)
        small = np.abs(x) < 1e-8
        return np.where(small, 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x)),
                        np.log1p(np.where(small, 1.0, x)) / np.where(small, 1.0, x))

    def _helper2(self, x):  # expm1(x)/x
        x = np.asarray(x, np.float64)
        small = np.abs(x) < 1e-8
        return np.where(small, 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x)),
                        np.expm1(np.where(small, 1.0, x)) / np.where(small, 1.0, x))

    def _H(self, x):
        lx = np.log(x)
        return self._helper2((1.0 - self.s) * lx) * lx

    def _h(self, x):
        return np.exp(-self.s * np.log(x))

    def _Hinv(self, x):
        t = x * (1.0 - self.s)
        t = np.maximum(t, -1.0)
        return np.exp(self._helper1(t) * x)

    def sample(self, n: int, rng: np.random.Generator) -> np.ndarray:
        out = np.empty(n, np.int64)
        todo = np.arange(n)
        while todo.size:
            u = self.hn + rng.random(todo.size) * (self.hx1 - self.hn)
            x = self._Hinv(u)
            k = np.clip(np.floor(x + 0.5), 1, self.V)
            ok = (k - x <= self.sq) | (u >= self._H(k + 0.5) - self._h(k))
            out[todo[ok]] = k[ok].astype(np.int64) - 1
            todo = todo[~ok]
        return out


def rank_to_key(r: np.ndarray, V: int, A: int = 2654435761, C: int = 12345) -> np.ndarray:
    while math.gcd(A, V) != 1:
        A += 2
    return ((r.astype(np.uint64) * np.uint64(A % V) + np.uint64(C % V)) % np.uint64(V)).astype(np.uint64)


def planted_labels(offs, keys, seed: int, rng: np.random.Generator, scale: float = 4.0):
    """label ~ Bernoulli(sigmoid(scale * sum_f w_f / sqrt(nnz))), w_f in [-1,1) from
    splitmix64(key ^ seed) -- the planted model of proj/src/data.cpp:22-43 with a
    hashed (not tabulated) per-feature weight so V can be 1e8+."""
    h = splitmix64(keys ^ np.uint64(seed * 0x9E3779B1 & 0xFFFFFFFFFFFFFFFF))
    w = (h >> np.uint64(11)).astype(np.float64) * (2.0 / 9007199254740992.0) - 1.0
    nnz = np.diff(offs.astype(np.int64))
    inst = np.repeat(np.arange(len(nnz)), nnz)
    s = np.bincount(inst, weights=w, minlength=len(nnz))
    logit = scale * s / np.sqrt(np.maximum(nnz.mean(), 1.0))
    p = 1.0 / (1.0 + np.exp(-logit))
    return (rng.random(len(nnz)) < p).astype(np.int32)


class CtrBatch:
    __slots__ = ("offs", "keys", "slots", "labels", "n_slots")

    def __init__(self, offs, keys, labels, slots=None, n_slots=1):
        self.offs = np.ascontiguousarray(offs, np.uint32)
        self.keys = np.ascontiguousarray(keys, np.uint64)
        self.labels = np.ascontiguousarray(labels, np.int32)
        self.slots = None if slots is None else np.ascontiguousarray(slots, np.uint16)
        self.n_slots = int(n_slots)

    @property
    def n(self) -> int:
        return len(self.offs) - 1

    @property
    def occurrences(self) -> int:
        return int(self.offs[-1])

    def slice(self, lo: int, hi: int) -> "CtrBatch":
        a, b = int(self.offs[lo]), int(self.offs[hi])
        return CtrBatch(self.offs[lo:hi + 1] - self.offs[lo], self.keys[a:b], self.labels[lo:hi],
                        None if self.slots is None else self.slots[a:b], self.n_slots)

    def folded(self) -> "CtrBatch":
        """S slots folded into one deduped sorted feature set per instance: the
        reference's Instance semantics (used to feed the CPU reference)."""
        if self.slots is None:
            return self
        offs, keys = [0], []
        for i in range(self.n):
            u = np.unique(self.keys[self.offs[i]:self.offs[i + 1]])
            keys.append(u)
            offs.append(offs[-1] + len(u))
        return CtrBatch(np.array(offs), np.concatenate(keys) if keys else np.zeros(0, np.uint64),
                        self.labels, None, 1)


def make_batch(B: int, *, V: int, zipf_s: float | None = 1.1, nnz: int | float = 26,
               poisson: bool = False, n_slots: int = 1, seed: int = 1, key_space_A: int = 2654435761,
               signal_seed: int = 7) -> CtrBatch:
    """One synthetic batch.

    n_slots == 1: each instance has `nnz` (or Poisson(nnz), clamped >=1) ids drawn
    from Zipf(zipf_s) (uniform when zipf_s is None), deduped+sorted per instance.
    n_slots  > 1: one feature per slot (O = B*S), slot ids 0..S-1 in order.
    """
    rng = np.random.default_rng(seed)
    if n_slots > 1:
        O = B * n_slots
        r = ZipfSampler(V, zipf_s).sample(O, rng) if zipf_s else rng.integers(0, V, O)
        keys = rank_to_key(r, V, key_space_A)
        offs = np.arange(B + 1, dtype=np.int64) * n_slots
        slots = np.tile(np.arange(n_slots, dtype=np.uint16), B)
        labels = planted_labels(offs, keys, signal_seed, rng)
        return CtrBatch(offs, keys, labels, slots, n_slots)
    if poisson:
        counts = np.maximum(rng.poisson(nnz, B), 1)
    else:
        counts = np.full(B, int(nnz))
    O = int(counts.sum())
    r = ZipfSampler(V, zipf_s).sample(O, rng) if zipf_s else rng.integers(0, V, O)
    keys = rank_to_key(r, V, key_space_A)
    inst = np.repeat(np.arange(B), counts)
    order = np.lexsort((keys, inst))
    keys, inst = keys[order], inst[order]
    keep = np.ones(O, bool)
    keep[1:] = (keys[1:] != keys[:-1]) | (inst[1:] != inst[:-1])
    keys, inst = keys[keep], inst[keep]
    nnz_u = np.bincount(inst, minlength=B)
    offs = np.zeros(B + 1, np.int64)
    np.cumsum(nnz_u, out=offs[1:])
    labels = planted_labels(offs, keys, signal_seed, rng)
    return CtrBatch(offs, keys, labels, None, 1)
