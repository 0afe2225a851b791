"""B200-native rebuild of the kpsim training hot path (arXiv 2201.05500).

Re-exports the reference module's names for the hot path
(proj/python/kpsim/__init__.py:8-62) from the in-tree extension
``_kpsim_b200`` (C++ shim over the C ABI of include/kpsim_b200.h, which runs
sm_100a kernels). There is no CPU fallback: importing fails loudly when the
extension has not been built (``python paper_2201_05500_b200/build.py``).
"""
from __future__ import annotations

try:
    from ._kpsim_b200 import (  # noqa: F401
        AdamHyper,
        Comm,
        ConfigError,
        DeviceError,
        KpsimError,
        KStepEngine,
        StoreError,
        TieredStore,
        Trainer,
        WorkerState,
        accumulate_moments,
        adagrad_sparse_update,
        auc_device,
        comm_unique_id,
        compute_auc,
        dedup,
        dedup_runs,
        gemm_nt,
        gemm_tn,
        device_count,
        global_merge,
        kstep_ratio,
        launch_count,
        local_adam_step,
        read_instances,
        shard,
        version,
        write_instances,
    )
except ImportError as e:  # pragma: no cover - exercised only on broken installs
    raise ImportError(
        "paper_2201_05500_b200: the CUDA extension is not built "
        "(run `python paper_2201_05500_b200/build.py`); there is no CPU fallback"
    ) from e

__all__ = [
    "AdamHyper", "Comm", "ConfigError", "DeviceError", "KpsimError", "KStepEngine", "StoreError",
    "TieredStore", "Trainer", "WorkerState", "accumulate_moments", "adagrad_sparse_update", "auc_device",
    "comm_unique_id", "compute_auc", "dedup", "dedup_runs", "gemm_nt", "gemm_tn", "device_count", "global_merge", "kstep_ratio", "launch_count",
    "local_adam_step", "read_instances", "shard", "version", "write_instances",
]

__version__ = "0.1.0"
