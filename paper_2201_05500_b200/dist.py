"""Multi-process (one process per GPU) plumbing around the Trainer.

- `rank_slice` reproduces shard_batch's cell layout (proj/src/trainer.cpp:32-53,
  153-156): N workers x n_mb minibatches, contiguous cells, the first
  (n % cells) cells one longer; rank r owns workers [r*W, (r+1)*W), i.e. one
  contiguous instance range of the global batch.
- `bootstrap_comm` broadcasts the NCCL unique id over torch.distributed (any
  backend; gloo is enough) and creates the data-path communicator.
- `DistributedTrainer` trains a GLOBAL batch: each rank feeds its slice and
  predictions are all-gathered for the reference's online AUC.
"""
from __future__ import annotations

import numpy as np


def n_minibatches(global_n: int, n_workers: int, minibatch_size: int) -> int:
    per = n_workers * minibatch_size
    return max(1, (global_n + per - 1) // per)


def cell_start(c: int, global_n: int, cells: int) -> int:
    base, extra = divmod(global_n, cells)
    return c * base + min(c, extra)


def rank_slice(global_n: int, n_workers: int, local_workers: int, minibatch_size: int,
               rank: int) -> tuple[int, int]:
    """(first, count) of the instances rank `rank` trains."""
    n_mb = n_minibatches(global_n, n_workers, minibatch_size)
    cells = n_workers * n_mb
    lo = cell_start(rank * local_workers * n_mb, global_n, cells)
    hi = cell_start((rank + 1) * local_workers * n_mb, global_n, cells)
    return lo, hi - lo


def bootstrap_comm(device: int):
    import torch.distributed as dist

    import paper_2201_05500_b200 as kp
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [kp.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return kp.Comm(obj[0], rank, world, device)


class DistributedTrainer:
    """kpsim Trainer over torch.distributed ranks (one GPU each)."""

    def __init__(self, device: int, table_capacity: int = 1 << 22, **cfg):
        import torch.distributed as dist

        import paper_2201_05500_b200 as kp
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.comm = bootstrap_comm(device) if self.world > 1 else None
        cfg.setdefault("n_workers", self.world)
        self.local_workers = cfg["n_workers"] // self.world
        self.minibatch_size = cfg.get("minibatch_size", 128)
        self.tr = kp.Trainer(comm=self.comm, table_capacity=table_capacity, device=device, **cfg)
        self.n_workers = cfg["n_workers"]
        self._scores, self._labels = [], []

    def train_batch(self, batch, predict_first: bool = False) -> dict:
        import torch
        import torch.distributed as dist

        import paper_2201_05500_b200 as kp
        first, n = rank_slice(batch.n, self.n_workers, self.local_workers, self.minibatch_size,
                              self.rank)
        sl = batch.slice(first, first + n)
        r = self.tr.train_batch(sl.offs, sl.keys, sl.labels, slots=sl.slots,
                                predict_first=predict_first, global_n=batch.n, global_first=first)
        # predict_first: r["auc"] / r["cumulative_auc"] are computed on the
        # device over the GLOBAL batch (predictions all-gathered over NCCL)
        return r
