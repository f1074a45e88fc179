"""torch front end: the library's device entry points as torch custom ops.

SURVEY.md §8(b): "the torch extension wraps the same functions with
torch::Tensor".  Registered with ``torch.library`` (namespace ``trinity``) on
top of the C-ABI, so a torch program calls them like any operator -- on the
current CUDA stream, with CUDA-graph capture and fake-tensor shape inference --
while the C-ABI stays free of torch types:

* ``torch.ops.trinity.ivf_search(handle, queries, k, nprobe, kmax)`` ->
  (ids int64 [B, kmax], dists float64 [B, kmax]); ``k`` / ``nprobe`` are int32
  CPU tensors (per query, scheduler decisions stay on the host);
* ``torch.ops.trinity.knn(handle, queries, k, kmax)`` -> exact brute force
  (``tri_knn_bruteforce_dev``);
* ``torch.ops.trinity.merge_topk(dists, ids, k_out)`` -> the (dist, id) merge of
  per-shard lists [G, B, k_in] (``tri_merge_topk``).

``handle`` is the opaque ``tri_ivf*`` / ``tri_store*`` as an int
(``IVFFlatIndex.handle.value``, ``_DeviceStore.handle.value``).
"""

from __future__ import annotations

import torch

from . import _lib


def _check_q(queries: torch.Tensor) -> None:
    if not queries.is_cuda or queries.dtype != torch.float64 or queries.dim() != 2 or not queries.is_contiguous():
        raise ValueError("queries must be a contiguous float64 CUDA tensor [B, d]")


def _host_i32(t: torch.Tensor, B: int, name: str) -> torch.Tensor:
    t = t.to("cpu", torch.int32).contiguous()
    if t.shape != (B,):
        raise ValueError(f"{name} must hold one value per query ({B}), got shape {tuple(t.shape)}")
    return t


@torch.library.custom_op("trinity::ivf_search", mutates_args=())
def ivf_search(handle: int, queries: torch.Tensor, k: torch.Tensor, nprobe: torch.Tensor,
               kmax: int) -> tuple[torch.Tensor, torch.Tensor]:
    _check_q(queries)
    B = queries.shape[0]
    ks, nps = _host_i32(k, B, "k"), _host_i32(nprobe, B, "nprobe")
    ids = torch.empty((B, kmax), dtype=torch.int64, device=queries.device)
    d = torch.empty((B, kmax), dtype=torch.float64, device=queries.device)
    if B:
        _lib.check(_lib.gpu().tri_ivf_search_dev(handle, queries.data_ptr(), B, ks.data_ptr(), nps.data_ptr(), kmax,
                                                 ids.data_ptr(), d.data_ptr(),
                                                 torch.cuda.current_stream(queries.device).cuda_stream))
    return ids, d


@ivf_search.register_fake
def _(handle, queries, k, nprobe, kmax):
    B = queries.shape[0]
    return queries.new_empty((B, kmax), dtype=torch.int64), queries.new_empty((B, kmax), dtype=torch.float64)


@torch.library.custom_op("trinity::knn", mutates_args=())
def knn(handle: int, queries: torch.Tensor, k: torch.Tensor, kmax: int) -> tuple[torch.Tensor, torch.Tensor]:
    _check_q(queries)
    B = queries.shape[0]
    ks = _host_i32(k, B, "k")
    ids = torch.empty((B, kmax), dtype=torch.int64, device=queries.device)
    d = torch.empty((B, kmax), dtype=torch.float64, device=queries.device)
    if B:
        _lib.check(_lib.gpu().tri_knn_bruteforce_dev(handle, queries.data_ptr(), B, ks.data_ptr(), kmax,
                                                     ids.data_ptr(), d.data_ptr(),
                                                     torch.cuda.current_stream(queries.device).cuda_stream))
    return ids, d


@knn.register_fake
def _(handle, queries, k, kmax):
    B = queries.shape[0]
    return queries.new_empty((B, kmax), dtype=torch.int64), queries.new_empty((B, kmax), dtype=torch.float64)


@torch.library.custom_op("trinity::merge_topk", mutates_args=())
def merge_topk(dists: torch.Tensor, ids: torch.Tensor, k_out: int) -> tuple[torch.Tensor, torch.Tensor]:
    if dists.dim() != 3 or dists.shape != ids.shape or not dists.is_cuda:
        raise ValueError("dists / ids must be CUDA tensors [G, B, k_in] of one shape")
    G, B, k_in = dists.shape
    dc = dists.to(torch.float64).contiguous()
    ic = ids.to(torch.int64).contiguous()
    oi = torch.empty((B, k_out), dtype=torch.int64, device=dists.device)
    od = torch.empty((B, k_out), dtype=torch.float64, device=dists.device)
    if B:
        _lib.check(_lib.gpu().tri_merge_topk(dc.data_ptr(), ic.data_ptr(), G, B, k_in, k_out, od.data_ptr(),
                                             oi.data_ptr(), torch.cuda.current_stream(dists.device).cuda_stream))
    return oi, od


@merge_topk.register_fake
def _(dists, ids, k_out):
    B = dists.shape[1]
    return dists.new_empty((B, k_out), dtype=torch.int64), dists.new_empty((B, k_out), dtype=torch.float64)


__all__ = ["ivf_search", "knn", "merge_topk"]
