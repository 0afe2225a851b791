"""TEST INFRASTRUCTURE ONLY: an f64 restatement of the training step in torch,
for parity checks at BASELINE.json's full sizes (configs[1]: B=65536, S=100,
e=64, MLP [6400->256->128->1]) where the plain-C oracle (kpsim_oracle.c, ~5
CPU-minutes per step there) is too slow for a test. It runs on the GPU in
float64, so it is a checker with ~1e-16 rounding, not a product path.

It restates oracle/kpsim_oracle.c (itself pinned bit-exact against the
compiled reference) for ONE worker (N=1, one minibatch per batch):
  * working set + insert-if-absent with the fresh entry {w=0, acc=1e-6}
    (proj/src/trainer.cpp:121-129, proj/include/kpsim/store.hpp:49);
  * per-slot sum/mean pooling (proj/src/model.cpp:88-99, extended to S slots
    as in kpsim_oracle.c forward());
  * MLP forward, sigmoid, mean BCE, backward with upstream (p-y)/n
    (proj/src/model.cpp:100-191);
  * per-key gradient sum, x 1/N, AdaGrad push (proj/src/trainer.cpp:180-208,
    proj/src/optimizer.cpp:86-95);
  * KStepEngine::step for N=1 (proj/src/optimizer.cpp:39-84,113-144).
Only the summation ORDER differs from the C oracle (torch reductions); in f64
that moves results by ~1e-15 relative, far below the fp32 tolerances it checks.
tests/test_gpu_configs.py pins it against orc64 before using it.
Only tests/ import this module.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle.oracle import orc_init_dense

F64 = torch.float64


class Torch64Trainer:
    def __init__(self, cfg, device="cuda"):
        if cfg.n_workers != 1 or cfg.sparse_rule != "adagrad":
            raise ValueError("Torch64Trainer restates N=1 with AdaGrad rows only")
        self.cfg = cfg
        self.dev = torch.device(device)
        e, S = cfg.embedding_dim, cfg.n_slots
        self.widths = [S * e, *cfg.hidden, 1]
        self.w_off, self.b_off = [], []
        D = 0
        for a, b in zip(self.widths, self.widths[1:]):
            self.w_off.append(D)
            D += a * b
            self.b_off.append(D)
            D += b
        self.D = D
        x0 = orc_init_dense(cfg.seed, D)  # CtrModel::init_dense (model.cpp:68-74)
        self.x = torch.tensor(x0, dtype=F64, device=self.dev)
        self.m = torch.zeros(D, dtype=F64, device=self.dev)
        self.v = torch.full((D,), cfg.epsilon, dtype=F64, device=self.dev)
        self.vbar = self.v.clone()
        self.t = 0
        self.keys = np.zeros(0, np.uint64)
        self.w = torch.zeros((0, e), dtype=F64, device=self.dev)
        self.acc = torch.zeros((0, e), dtype=F64, device=self.dev)

    # -- table ---------------------------------------------------------------
    def _pull(self, keys):
        u = np.unique(keys)
        new = np.setdiff1d(u, self.keys, assume_unique=True)
        if len(new):
            allk = np.union1d(self.keys, new)
            e = self.cfg.embedding_dim
            w = torch.zeros((len(allk), e), dtype=F64, device=self.dev)
            acc = torch.full((len(allk), e), 1e-6, dtype=F64, device=self.dev)
            if len(self.keys):
                old = torch.from_numpy(np.searchsorted(allk, self.keys).astype(np.int64)).to(self.dev)
                w[old] = self.w
                acc[old] = self.acc
            self.keys, self.w, self.acc = allk, w, acc
        return torch.from_numpy(np.searchsorted(self.keys, keys).astype(np.int64)).to(self.dev)

    def table(self):
        return self.keys, self.w.cpu().numpy(), self.acc.cpu().numpy()

    # -- model ---------------------------------------------------------------
    def _layer(self, x, l):
        a, b = self.widths[l], self.widths[l + 1]
        W = x[self.w_off[l]:self.w_off[l] + a * b].view(b, a)
        bias = x[self.b_off[l]:self.b_off[l] + b]
        return W, bias

    def _pool(self, offs, rows, slots, n):
        e, S = self.cfg.embedding_dim, self.cfg.n_slots
        nnz = np.diff(offs.astype(np.int64))
        inst = np.repeat(np.arange(n), nnz)
        sl = slots.astype(np.int64) if slots is not None else np.zeros(len(inst), np.int64)
        bag = torch.from_numpy(inst * S + sl).to(self.dev)
        pooled = torch.zeros((n * S, e), dtype=F64, device=self.dev)
        pooled.index_add_(0, bag, self.w[rows])
        coeff = None
        if self.cfg.pooling == "mean":
            cnt = torch.zeros(n * S, dtype=F64, device=self.dev)
            cnt.index_add_(0, bag, torch.ones(len(inst), dtype=F64, device=self.dev))
            inv = torch.where(cnt > 0, 1.0 / cnt.clamp(min=1), torch.zeros_like(cnt))
            pooled *= inv[:, None]
            coeff = inv[bag]
        return pooled.view(n, S * e), bag, coeff

    def _forward(self, x, pooled):
        L = len(self.widths) - 1
        h, pre, act = pooled, [], []
        for l in range(L):
            W, b = self._layer(x, l)
            z = h @ W.T + b
            pre.append(z)
            if l + 1 < L:
                h = torch.relu(z) if self.cfg.activation == "relu" else torch.tanh(z)
            else:
                h = z
            act.append(h)
        logit = act[-1][:, 0]
        return pre, act, logit, torch.sigmoid(logit)

    def batch(self, offs, keys, labels, slots=None, predict_first=False):
        cfg = self.cfg
        n = len(offs) - 1
        e, S = cfg.embedding_dim, cfg.n_slots
        rows = self._pull(keys)
        y = torch.from_numpy(labels.astype(np.float64)).to(self.dev)
        out = {}
        pooled, bag, coeff = self._pool(offs, rows, slots, n)
        pre, act, logit, pred = self._forward(self.x, pooled)
        if predict_first:  # x_bar of one worker is its x: the training forward
            out["preds"] = pred.cpu().numpy()
        # mean_bce (model.cpp:126-135); softplus(z) = max(z,0) + log1p(exp(-|z|))
        sp = torch.clamp(logit, min=0) + torch.log1p(torch.exp(-logit.abs()))
        out["loss"] = float((sp - y * logit).mean())
        # backward (model.cpp:137-191)
        g = torch.zeros(self.D, dtype=F64, device=self.dev)
        delta = ((pred - y) / n)[:, None]
        L = len(self.widths) - 1
        for l in range(L - 1, -1, -1):
            W, _ = self._layer(self.x, l)
            if l + 1 < L:
                if cfg.activation == "relu":
                    delta = delta * (pre[l] > 0).to(F64)
                else:
                    delta = delta * (1 - act[l] * act[l])
            inp = pooled if l == 0 else act[l - 1]
            a, b = self.widths[l], self.widths[l + 1]
            g[self.w_off[l]:self.w_off[l] + a * b] = (delta.T @ inp).reshape(-1)
            g[self.b_off[l]:self.b_off[l] + b] = delta.sum(0)
            delta = delta @ W
        dpooled = delta.reshape(n * S, e)
        # sparse grads: sum over occurrences per key (x coeff for mean), x 1/N
        gocc = dpooled[bag]
        if coeff is not None:
            gocc = gocc * coeff[:, None]
        G = torch.zeros_like(self.w)
        G.index_add_(0, rows, gocc)
        touched = torch.unique(rows)
        gt = G[touched] * (1.0 / cfg.n_workers)
        acc = self.acc[touched] + gt * gt
        self.acc[touched] = acc
        self.w[touched] = self.w[touched] - cfg.sparse_lr * gt / torch.sqrt(acc)
        # KStepEngine::step, N = 1
        self.t += 1
        self.m = cfg.beta1 * self.m + (1 - cfg.beta1) * g
        self.v = cfg.beta2 * self.v + (1 - cfg.beta2) * (g * g)
        if self.t % cfg.k:
            self.x = self.x - cfg.alpha * self.m / torch.sqrt(self.vbar)
        else:  # global_merge over one worker: cmean(v) = v, cmean(terms) = terms
            self.vbar = self.v.clone()
            self.x = self.x - cfg.alpha * self.m / torch.sqrt(self.vbar)
            if cfg.reset_local_v:
                self.v = self.vbar.clone()
        return out

    def worker_state(self, i=0):
        return {"x": self.x.cpu().numpy(), "m": self.m.cpu().numpy(), "v": self.v.cpu().numpy(),
                "v_bar": self.vbar.cpu().numpy()}
