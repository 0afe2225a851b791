"""Shared test helpers (fixture loading, GPU/oracle runners, comparisons)."""
from __future__ import annotations

import ast
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    d = {k: z[k] for k in z.files}
    meta = ast.literal_eval(str(d.pop("meta"))) if "meta" in d else None
    return d, meta


def golden_batches(d, n):
    for b in range(n):
        yield d[f"b{b}_offs"], d[f"b{b}_keys"], d[f"b{b}_labels"]


def trainer_kwargs(cfg: dict) -> dict:
    """TrainerCfg field names -> the Trainer binding's kwargs."""
    kw = dict(cfg)
    kw["hidden"] = list(kw.get("hidden", ()))
    return kw


def rel_err(a, b, floor=1e-3):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0
