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


def pack_results(ids: np.ndarray, dists: np.ndarray) -> np.ndarray:
    """[2, B, k] int64: the ids block, then the float64 distance bits.  One
    tensor per rank and batch goes through the gather (16 bytes per (query,
    neighbour)), in the layout ``tri_merge_topk_ld`` reads in place."""
    return np.stack([np.asarray(ids, np.int64), np.ascontiguousarray(dists, np.float64).view(np.int64)])


def unpack_results(packed, k: int):
    """Inverse of ``pack_results`` on [..., 2, B, k] (numpy or torch): (ids, dists)."""
    if not isinstance(packed, np.ndarray):
        import torch

        return packed[..., 0, :, :], packed[..., 1, :, :].contiguous().view(torch.float64)
    return packed[..., 0, :, :], np.ascontiguousarray(packed[..., 1, :, :]).view(np.float64)


class ShardedSearch:
    """One rank of a vector-sharded search (host-side protocol).

    local_search(queries, k, nprobe) -> (ids int64 [B, k], dists f64 [B, k])
        searches this rank's shard and returns GLOBAL ids (-1 padded);
    merge(dists [G, B, k], ids [G, B, k], k) -> (ids [B, k], dists [B, k])
        the exact (dist, id) merge (device kernel or CPU oracle).

    Each rank packs its lists into one [B, 2k] tensor and the ranks exchange
    it in ONE all-gather (``ShardedIVF`` is the device-resident form).
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
        mine = torch.from_numpy(pack_results(ids, dists)).to(dev)
        allp = torch.empty((self.world,) + tuple(mine.shape), dtype=mine.dtype, device=mine.device)
        self.dist.all_gather_into_tensor(allp.view(-1), mine.view(-1), group=self.group)
        gi, gd = unpack_results(allp, k)
        return self.merge(gd.contiguous(), gi.contiguous(), k)


class ShardedIVF:
    """One rank's share of a vector-sharded IVF index on its own GPU (C4).

    ``index`` holds this rank's rows (global ids, ``id_offset`` folded in) built
    from the shared artifact.  A batch runs entirely on the device, on the
    caller's stream:

    1. the local search writes its ids and float64 distances into one [2, B, k]
       block (ids, then dists; ``ldo`` = k);
    2. ONE ``all_gather_into_tensor`` of that buffer (NCCL over NVLink; B*k*16
       bytes per rank, 40 KB at C2 shapes);
    3. ``tri_merge_topk_ld`` merges the gathered [G, 2, B, k] lists in place
       by (dist, id).

    No host round trip between the steps; every rank ends with the merged
    top-k.  k is one value for the batch (nprobe may vary per query).

    ``transport="native"`` runs the same three steps inside the library
    (``tri_ivf_search_sharded``: its own NCCL communicator, created from a
    unique id that rank 0 broadcasts over ``group``); without an initialised
    process group it is a world of one.
    """

    def __init__(self, index, k: int, group=None, transport: str = "torch"):
        import ctypes as C

        import torch.distributed as dist

        from . import _lib

        if transport not in ("torch", "native"):
            raise ValueError(f"transport must be 'torch' or 'native', got {transport!r}")
        self.dist = dist
        self.group = group
        self.index = index
        self.k = int(k)
        if self.k < 1:
            raise ValueError(f"k must be >= 1, got {k}")
        self.transport = transport
        ready = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if ready else 1
        self.rank = dist.get_rank(group) if ready else 0
        self.host_gather = ready and dist.get_backend(group) == "gloo"  # test hook: gloo moves host tensors
        self._bufs = {}
        self._comm = None
        if transport == "native":
            uid = (C.c_uint8 * 128)()
            if self.rank == 0:
                _lib.check(_lib.gpu().tri_comm_unique_id(uid))
            if self.world > 1:
                box = [bytes(uid)]
                dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0, group=group)
                uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
            h = C.c_void_p()
            _lib.check(_lib.gpu().tri_comm_init(uid, self.world, self.rank, int(index.device), C.byref(h)))
            self._comm = h

    def close(self) -> None:
        if self._comm:
            from . import _lib

            _lib.load_library().tri_comm_destroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _lane(self, stream, B: int):
        import torch

        key = (int(getattr(stream, "cuda_stream", 0) or 0), B)
        b = self._bufs.get(key)
        if b is None:
            b = {
                "local": torch.empty((2, B, self.k), dtype=torch.int64, device="cuda"),
                "all": torch.empty((self.world, 2, B, self.k), dtype=torch.int64, device="cuda"),
                "q": torch.empty((B, self.index.dim), dtype=torch.float64, device="cuda"),
                "ids": torch.empty((B, self.k), dtype=torch.int64, device="cuda"),
                "d": torch.empty((B, self.k), dtype=torch.float64, device="cuda"),
            }
            self._bufs[key] = b
        return b

    def search_device(self, q_dev, nprobe, out_ids, out_dists, stream) -> None:
        """Asynchronous sharded search of device queries [B, d] into device
        outputs [B, >= k] (ids int64, dists float64) on ``stream``."""
        import torch

        from . import _lib
        from .ivf import _check_buf, _stream_ptr

        B = int(q_dev.shape[0])
        _check_buf("queries", q_dev, "float64", cols=self.index.dim)
        _check_buf("ids", out_ids, "int64", rows=B)
        _check_buf("dists", out_dists, "float64", cols=int(out_ids.shape[1]), rows=B)
        if int(out_ids.shape[1]) < self.k:
            raise ValueError(f"outputs hold {int(out_ids.shape[1])} columns, k={self.k}")
        ks, nps = self.index._ragged(B, self.k, nprobe)
        if self._comm is not None:
            _lib.check(_lib.gpu().tri_ivf_search_sharded(self.index.handle, self._comm, _lib.ptr(q_dev), B, self.k,
                                                         nps.ctypes.data, int(out_ids.shape[1]), _lib.ptr(out_ids),
                                                         _lib.ptr(out_dists), _stream_ptr(stream)))
            return
        b = self._lane(stream, B)
        loc, k, st = b["local"], self.k, _stream_ptr(stream)
        lib = _lib.gpu()
        _lib.check(lib.tri_ivf_search_dev(self.index.handle, _lib.ptr(q_dev), B, ks.ctypes.data, nps.ctypes.data,
                                          k, loc.data_ptr(), loc.data_ptr() + 8 * B * k, st))
        with torch.cuda.stream(stream):
            if self.host_gather:
                h = torch.empty((self.world,) + tuple(loc.shape), dtype=torch.int64)
                self.dist.all_gather_into_tensor(h.view(-1), loc.cpu().view(-1), group=self.group)
                b["all"].copy_(h)
            else:
                self.dist.all_gather_into_tensor(b["all"].view(-1), loc.view(-1), group=self.group)
        allp = b["all"]
        _lib.check(lib.tri_merge_topk_ld(allp.data_ptr() + 8 * B * k, allp.data_ptr(), self.world, B, k, k, 2 * B * k,
                                         k, _lib.ptr(out_dists), _lib.ptr(out_ids), int(out_ids.shape[1]), st))

    def search_async(self, q_host, nprobe, ids_out, dists_out, stream):
        """Host-buffer form, asynchronous: enqueues the H2D copy of the queries
        [B, d] float64 (pinned host), the sharded search and the D2H copy of
        the merged top-k into ``ids_out`` / ``dists_out`` (pinned) on
        ``stream``; returns a CUDA event that completes with the copies.  One
        host thread can keep several streams busy while every rank issues its
        collectives in the same order (a requirement of NCCL)."""
        import torch

        B = int(q_host.shape[0])
        b = self._lane(stream, B)
        with torch.cuda.stream(stream):
            b["q"].copy_(torch.as_tensor(q_host), non_blocking=True)
        self.search_device(b["q"], nprobe, b["ids"], b["d"], stream)
        with torch.cuda.stream(stream):
            torch.as_tensor(ids_out)[:, :self.k].copy_(b["ids"], non_blocking=True)
            torch.as_tensor(dists_out)[:, :self.k].copy_(b["d"], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        return ev

    def search_into(self, q_host, nprobe, ids_out, dists_out, stream) -> None:
        """Host-buffer form (blocking): ``search_async`` then wait."""
        self.search_async(q_host, nprobe, ids_out, dists_out, stream).synchronize()

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
