"""CPU: the C-ABI library loads and exports every symbol include/kpsim_b200.h
declares; the extension imports; without a GPU, compute calls fail loudly
(no CPU fallback)."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import has_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kpsim_b200.h")
LIB = os.path.join(ROOT, "paper_2201_05500_b200", "libkpsim_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["kp_table_create", "kp_store_pull_batch", "kp_store_push_updates", "kp_dedup",
              "kp_shard", "kp_dense_local_step", "kp_kstep_merge", "kp_trainer_train_batch",
              "kp_comm_init", "kp_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {LIB} 2>/dev/null").read()
    assert "sm_100a" in out


def test_extension_imports_and_reexports_reference_names():
    import paper_2201_05500_b200 as kp
    for name in ["AdamHyper", "WorkerState", "TieredStore", "local_adam_step", "global_merge",
                 "adagrad_sparse_update", "compute_auc", "KpsimError", "ConfigError"]:
        assert hasattr(kp, name)
    assert issubclass(kp.ConfigError, ValueError)
    assert issubclass(kp.KpsimError, RuntimeError)
    assert issubclass(kp.StoreError, kp.KpsimError)


def test_host_logic_without_gpu():
    import paper_2201_05500_b200 as kp
    assert kp.compute_auc([0.1, 0.9], [0, 1]) == 1.0
    assert kp.compute_auc([0.5, 0.5], [0, 1]) == 0.5
    assert kp.compute_auc([0.5, 0.6], [1, 1]) is None
    h = kp.AdamHyper()
    assert (h.alpha, h.beta1, h.beta2, h.epsilon, h.k, h.reset_local_v) == (0.01, 0.0, 0.999, 0.01, 1, True)
    s = kp.WorkerState.init([1.0, 2.0], 0.01)
    assert s.m == [0.0, 0.0] and s.v == [0.01, 0.01] and s.v_bar == [0.01, 0.01]


@pytest.mark.skipif(has_gpu(), reason="only meaningful without a GPU")
def test_no_cpu_fallback():
    import paper_2201_05500_b200 as kp
    with pytest.raises(kp.DeviceError):
        kp.dedup(np.arange(4, dtype=np.uint64))
    with pytest.raises(kp.DeviceError):
        kp.Trainer(n_workers=1)
    lib = ctypes.CDLL(LIB)
    lib.kp_last_error.restype = ctypes.c_char_p
    n = ctypes.c_int(-1)
    assert lib.kp_device_count(ctypes.byref(n)) != 0
    assert b"CUDA" in lib.kp_last_error()
