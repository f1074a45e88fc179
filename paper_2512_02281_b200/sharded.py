"""Vector-sharded search across the GPUs of one node (configs C4, bench --gpus N).

Partitioning: rank g owns global ids [g N / G, (g+1) N / G);
the IVF artifact (centroids + list id of every vector) is shared, so every
inverted list is split by id range and load stays balanced however the
probes skew.  Each rank searches its shard (the coarse step is replicated and
deterministic), the per-shard top-k (dist, id) lists are all-gathered and
merged by (dist, id) -- the reference's tie rule (ann_graph.py:8-9, :136) --
which yields exactly the global top-k over the union of the probed lists.

The collective protocol is backend-agnostic (``torch.distributed`` with NCCL
on GPUs; gloo in the CPU tests) and the local search / merge are injected, so
the same code path is exercised with the device kernels in production and
with the CPU oracle in ``tests/test_sharded.py``.
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def shard_bounds(n: int, world: int, rank: int) -> tuple:
    """Row range [lo, hi) of ``rank``'s shard."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} out of range for world {world}")
    return rank * n // world, (rank + 1) * n // world


def pad_results(ids: np.ndarray, dists: np.ndarray, k: int):
    """Right-pad per-query results to width k with (-1, +inf)."""
    B = ids.shape[0]
    oi = np.full((B, k), -1, dtype=np.int64)
    od = np.full((B, k), np.inf, dtype=np.float64)
    w = min(k, ids.shape[1])
    oi[:, :w] = ids[:, :w]
    od[:, :w] = dists[:, :w]
    return oi, od


class ShardedSearch:
    """One rank of a vector-sharded search.

    local_search(queries, k, nprobe) -> (ids int64 [B, k], dists f64 [B, k])
        searches this rank's shard and returns GLOBAL ids (-1 padded);
    merge(dists [G, B, k], ids [G, B, k], k) -> (ids [B, k], dists [B, k])
        the exact (dist, id) merge (device kernel or CPU oracle).
    """

    def __init__(self, local_search: Callable, merge: Callable, group=None, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.local_search = local_search
        self.merge = merge
        self.device = device
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def search(self, queries, k: int, nprobe: int):
        import torch

        ids, dists = self.local_search(queries, k, nprobe)
        ids, dists = pad_results(np.asarray(ids), np.asarray(dists), k)
        dev = self.device or "cpu"
        ti = torch.from_numpy(ids).to(dev)
        td = torch.from_numpy(dists).to(dev)
        gi = [torch.empty_like(ti) for _ in range(self.world)]
        gd = [torch.empty_like(td) for _ in range(self.world)]
        self.dist.all_gather(gi, ti, group=self.group)
        self.dist.all_gather(gd, td, group=self.group)
        return self.merge(torch.stack(gd), torch.stack(gi), k)


def device_merge(dists, ids, k: int):
    """tri_merge_topk on device tensors [G, B, k] -> host (ids, dists)."""
    import torch

    from .ivf import merge_topk_device

    G, B, kin = dists.shape
    od = torch.empty((B, k), dtype=torch.float64, device=dists.device)
    oi = torch.empty((B, k), dtype=torch.int64, device=dists.device)
    merge_topk_device(dists.contiguous(), ids.contiguous(), k, od, oi, torch.cuda.current_stream())
    torch.cuda.current_stream().synchronize()
    return oi.cpu().numpy(), od.cpu().numpy()


def ivf_shard_search(index):
    """local_search backed by this rank's device IVF shard (ids already global)."""

    def run(queries, k, nprobe):
        return index.search(queries, k, nprobe)

    return run
