"""CPU, world_size 2 and 8 over gloo: the host-side multi-rank logic.

- rank slices partition the global batch exactly like shard_batch's cells
  (proj/src/trainer.cpp:32-53; test_trainer.cpp:58-99 balance/multiset);
- the NCCL-id bootstrap broadcast delivers identical bytes to every rank;
- key ownership (key % G) splits a working set into disjoint shards whose
  union is the set (the all-to-all's routing invariant).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2201_05500_b200.dist import cell_start, n_minibatches, rank_slice


@pytest.mark.parametrize("n", [1, 7, 23, 64, 101, 65536])
@pytest.mark.parametrize("N,W", [(1, 1), (2, 1), (4, 2), (8, 1), (3, 3)])
@pytest.mark.parametrize("mb", [1, 16, 1 << 20])
def test_rank_slices_partition_batch(n, N, W, mb):
    world = N // W
    spans = [rank_slice(n, N, W, mb, r) for r in range(world)]
    assert spans[0][0] == 0
    for (a, c), (b, _) in zip(spans, spans[1:]):
        assert a + c == b
    assert spans[-1][0] + spans[-1][1] == n
    n_mb = n_minibatches(n, N, mb)
    sizes = [cell_start(c + 1, n, N * n_mb) - cell_start(c, n, N * n_mb) for c in range(N * n_mb)]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # bootstrap broadcast of a 128-byte id (what bootstrap_comm sends)
    obj = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    # each rank's slice of a global batch + its owned keys of the slice's working set
    from paper_2201_05500_b200.data import make_batch
    bt = make_batch(1000, V=5000, zipf_s=1.1, nnz=5, seed=3)
    first, n = rank_slice(bt.n, world, 1, 10**9, rank)
    sl = bt.slice(first, first + n)
    uniq = np.unique(sl.keys)
    owned = [uniq[uniq % np.uint64(world) == np.uint64(g)] for g in range(world)]
    parts = [None] * world
    dist.all_gather_object(parts, (first, n, obj[0], [o.tolist() for o in owned]))
    q.put((rank, parts))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_gloo_world_bootstrap_and_routing(world):
    """world 8: the host-side path of an 8-GPU box (one rank per GPU)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = res[0]
    assert all(res[r] == parts for r in range(world))
    assert all(p[2] == bytes(range(128)) for p in parts)
    assert parts[0][0] == 0
    for r in range(1, world):
        assert parts[r - 1][0] + parts[r - 1][1] == parts[r][0]
    from paper_2201_05500_b200.data import make_batch
    bt = make_batch(1000, V=5000, zipf_s=1.1, nnz=5, seed=3)
    assert parts[world - 1][0] + parts[world - 1][1] == bt.n
    # owner g receives from every rank exactly the keys with key % G == g
    for g in range(world):
        recv = set()
        for src in range(world):
            ks = parts[src][3][g]
            assert all(k % world == g for k in ks)
            recv |= set(ks)
        want = {int(k) for k in np.unique(bt.keys) if int(k) % world == g}
        assert recv == want
