"""IVF-Flat index on the B200: k-means lists, exact coarse step, ragged batched search.

The reference has no IVF (SPEC.md:166 lists it as a non-goal) but BASELINE.json
configs C2-C4 name it; the semantics follow SURVEY.md §8c so that results are
exactly those of the reference primitives:

* coarse step  = ``brute_force_knn`` over the centroids (ann_graph.py:124-137)
  with k = nprobe, i.e. probes ordered by (dist, id);
* fine step    = exact top-k by (dist, id) over the union of the probed lists,
  distances in the reference's float64 operation order (ann_graph.py:97-105).

One ``search`` call is one batch: every query carries its own k and nprobe
(prefill k=100/nprobe=64 next to decode k=10/nprobe=16), the device packer
turns the ragged probe sets into list-major work items, and a single
persistent scan kernel serves them all -- no per-class padding launches.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .ann_graph import VectorStore, _DeviceStore


def _stream_ptr(stream):
    """torch.cuda.Stream / raw cudaStream_t int / None (the handle's own stream)."""
    if stream is None:
        return None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check_buf(name, a, dtype: str, cols=None, rows=None) -> None:
    """Raw-buffer APIs read memory directly: reject wrong dtype / layout loudly."""
    dt = str(a.dtype).replace("torch.", "")
    if dt != dtype:
        raise ValueError(f"{name} must be {dtype}, got {dt}")
    if a.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {tuple(a.shape)}")
    contig = a.is_contiguous() if hasattr(a, "is_contiguous") else a.flags["C_CONTIGUOUS"]
    if not contig:
        raise ValueError(f"{name} must be C-contiguous")
    if cols is not None and int(a.shape[1]) != cols:
        raise ValueError(f"{name} has {int(a.shape[1])} columns, expected {cols}")
    if rows is not None and int(a.shape[0]) < rows:
        raise ValueError(f"{name} has {int(a.shape[0])} rows, expected >= {rows}")


def init_rows(n: int, nlist: int, seed: int) -> np.ndarray:
    """Seeded k-means initial rows (same rule as the oracle's CPU k-means)."""
    rng = np.random.Generator(np.random.Philox(seed))
    return np.sort(rng.choice(n, size=nlist, replace=False)).astype(np.int64)


class IVFFlatIndex:
    """Device-resident inverted lists (list-major fp32 rows, ascending ids per list)."""

    def __init__(self, handle, nlist: int, n: int, dim: int, device: int = 0):
        self.handle = handle
        self.nlist = nlist
        self.count = n
        self.dim = dim
        self.device = device

    # -- construction -----------------------------------------------------
    @classmethod
    def train(cls, store, nlist: int, iters: int = 5, seed: int = 0) -> "IVFFlatIndex":
        """GPU Lloyd k-means (``iters`` updates) from seeded initial rows.

        Deterministic: exact nearest-centroid assignment and float64 centroid
        sums in ascending id order, so ``oracle.kmeans`` reproduces the
        artifact bit-for-bit (the bench's CPU arm builds the same index)."""
        dev = store.device() if isinstance(store, VectorStore) else store
        rows = init_rows(dev.n, nlist, seed)
        h = C.c_void_p()
        _lib.check(_lib.gpu().tri_ivf_train(dev.handle, int(nlist), int(iters), rows.ctypes.data, C.byref(h)))
        return cls(h, nlist, dev.n, dev.d, dev.device)

    @staticmethod
    def assign(store, centroids: np.ndarray) -> np.ndarray:
        """Exact nearest-centroid list id of every store row (tri_kmeans_assign):
        k = 1 brute force over the centroids, ties to the smaller id."""
        dev = store.device() if isinstance(store, VectorStore) else store
        cen = np.ascontiguousarray(centroids, dtype=np.float32)
        if cen.ndim != 2 or cen.shape[1] != dev.d:
            raise ValueError(f"centroids must be (nlist, {dev.d}), got {cen.shape}")
        out = np.empty(dev.n, dtype=np.int32)
        _lib.check(_lib.gpu().tri_kmeans_assign(dev.handle, cen.ctypes.data, cen.shape[0], out.ctypes.data))
        return out

    @classmethod
    def from_centroids(cls, store, centroids: np.ndarray, id_offset: int = 0) -> "IVFFlatIndex":
        """Lists from given centroids (each row to its exact nearest centroid):
        how a shard of a larger database joins a shared coarse quantiser."""
        return cls.from_artifact(store, centroids, cls.assign(store, centroids), id_offset=id_offset)

    @classmethod
    def from_artifact(cls, store, centroids: np.ndarray, assign: np.ndarray, id_offset: int = 0) -> "IVFFlatIndex":
        """Build the lists from a shared artifact (fp32 centroids + list id per row)."""
        dev = store.device() if isinstance(store, VectorStore) else store
        cen = np.ascontiguousarray(centroids, dtype=np.float32)
        asg = np.ascontiguousarray(assign, dtype=np.int32)
        if cen.ndim != 2 or cen.shape[1] != dev.d:
            raise ValueError(f"centroids must be (nlist, {dev.d}), got {cen.shape}")
        if asg.shape != (dev.n,):
            raise ValueError(f"assign must have {dev.n} entries, got {asg.shape}")
        h = C.c_void_p()
        _lib.check(_lib.gpu().tri_ivf_create(dev.handle, cen.ctypes.data, cen.shape[0], asg.ctypes.data,
                                             int(id_offset), C.byref(h)))
        return cls(h, cen.shape[0], dev.n, dev.d, dev.device)

    def close(self) -> None:
        if self.handle:
            _lib.load_library().tri_ivf_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- artifact -----------------------------------------------------------
    def export(self):
        """(centroids f32[nlist, d], assign i32[n]) -- the shared index artifact."""
        cen = np.empty((self.nlist, self.dim), dtype=np.float32)
        asg = np.empty(self.count, dtype=np.int32)
        _lib.check(_lib.gpu().tri_ivf_export(self.handle, cen.ctypes.data, asg.ctypes.data))
        return cen, asg

    def save(self, path: str) -> None:
        """IVF index file, little-endian like the reference's vector / graph files
        (ann_graph.py:186-244): magic b"TRIVF001", `<u8 nlist`, `<u8 n`, `<u8 d`,
        nlist x d `<f4` centroids, n `<i4` list ids (the shared artifact)."""
        write_ivf(path, *self.export())

    @classmethod
    def load(cls, store, path: str, id_offset: int = 0) -> "IVFFlatIndex":
        """Rebuild the device lists of ``store`` from an index file (see ``save``)."""
        cen, asg = read_ivf(path)
        dev = store.device() if isinstance(store, VectorStore) else store
        if asg.shape[0] != dev.n or cen.shape[1] != dev.d:
            raise ValueError(f"{path}: index for {asg.shape[0]} x {cen.shape[1]} vectors, store is {dev.n} x {dev.d}")
        return cls.from_artifact(store, cen, asg, id_offset=id_offset)

    def list_sizes(self) -> np.ndarray:
        out = np.empty(self.nlist, dtype=np.int64)
        _lib.check(_lib.gpu().tri_ivf_list_sizes(self.handle, out.ctypes.data))
        return out

    # -- search -------------------------------------------------------------
    def _ragged(self, B: int, k, nprobe):
        ks = np.ascontiguousarray(np.broadcast_to(np.asarray(k, dtype=np.int64), (B,)), dtype=np.int32)
        nps = np.ascontiguousarray(np.broadcast_to(np.asarray(nprobe, dtype=np.int64), (B,)), dtype=np.int32)
        if B and (ks.min() < 1):
            raise ValueError(f"k must be >= 1, got {int(ks.min())}")
        if B and (nps.min() < 1 or nps.max() > self.nlist):
            raise ValueError(f"nprobe must be in [1, {self.nlist}]")
        return ks, nps

    def search(self, queries, k, nprobe):
        """Ragged batched search with host buffers.

        Returns (ids int64[B, kmax], dists f64[B, kmax]); row i holds the exact
        top-k[i] over its nprobe[i] lists, padded with id -1 / inf (when those
        lists hold fewer than k[i] vectors, and in the columns past k[i]).
        """
        q = np.ascontiguousarray(np.atleast_2d(np.asarray(queries, dtype=np.float64)))
        if q.shape[1] != self.dim:
            raise ValueError(f"query dim {q.shape[1]} != index dim {self.dim}")
        B = q.shape[0]
        ks, nps = self._ragged(B, k, nprobe)
        kmax = int(ks.max()) if B else 1
        ids = np.full((B, kmax), -1, dtype=np.int64)  # columns past k[i] stay -1 / inf
        dists = np.full((B, kmax), np.inf, dtype=np.float64)
        if B:
            _lib.check(_lib.gpu().tri_ivf_search(self.handle, q.ctypes.data, B, ks.ctypes.data, nps.ctypes.data,
                                                  kmax, ids.ctypes.data, dists.ctypes.data, None))
        return ids, dists

    def search_into(self, q_host, k, nprobe, ids_out, dists_out, stream=None) -> None:
        """Host-buffer search into caller-owned (ideally pinned) arrays [B, ldo].

        Blocking.  Calls on different ``stream``s use separate library
        workspaces, so host threads driving one stream each overlap on the GPU.
        """
        B = int(q_host.shape[0])
        _check_buf("queries", q_host, "float64", cols=self.dim)
        _check_buf("ids_out", ids_out, "int64", rows=B)
        _check_buf("dists_out", dists_out, "float64", cols=int(ids_out.shape[1]), rows=B)
        ks, nps = self._ragged(B, k, nprobe)
        _lib.check(_lib.gpu().tri_ivf_search(self.handle, _lib.ptr(q_host), B, ks.ctypes.data, nps.ctypes.data,
                                              int(ids_out.shape[1]), _lib.ptr(ids_out), _lib.ptr(dists_out),
                                              _stream_ptr(stream)))

    def search_device(self, q_dev, k, nprobe, ids_dev, dists_dev, stream=None) -> None:
        """Asynchronous search on device buffers (torch CUDA tensors or raw pointers).

        q_dev: float64 [B, d]; ids_dev int64 / dists_dev float64 [B, ldo].
        """
        B = int(q_dev.shape[0])
        _check_buf("queries", q_dev, "float64", cols=self.dim)
        _check_buf("ids", ids_dev, "int64", rows=B)
        _check_buf("dists", dists_dev, "float64", cols=int(ids_dev.shape[1]), rows=B)
        ks, nps = self._ragged(B, k, nprobe)
        ldo = int(ids_dev.shape[1])
        _lib.check(_lib.gpu().tri_ivf_search_dev(self.handle, _lib.ptr(q_dev), B, ks.ctypes.data, nps.ctypes.data,
                                                  ldo, _lib.ptr(ids_dev), _lib.ptr(dists_dev), _stream_ptr(stream)))

    # -- introspection --------------------------------------------------------
    def last_probes(self, B: int, ld: int) -> np.ndarray:
        out = np.empty((B, ld), dtype=np.int64)
        _lib.check(_lib.gpu().tri_ivf_last_probes(self.handle, out.ctypes.data, ld))
        return out

    def last_fixups(self) -> int:
        n = C.c_int32(0)
        _lib.check(_lib.gpu().tri_ivf_last_fixups(self.handle, C.byref(n)))
        return n.value

    def set_profiling(self, on: bool) -> None:
        _lib.check(_lib.gpu().tri_ivf_set_profiling(self.handle, 1 if on else 0))

    def scan_time(self):
        ms = C.c_double(0.0)
        n = C.c_int32(0)
        _lib.check(_lib.gpu().tri_ivf_scan_time(self.handle, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    STAGES = ("coarse", "pack", "scan", "merge", "rerank", "fixup")

    def stage_times(self):
        """Accumulated per-stage device ms over profiled searches: (dict, n_searches)."""
        ms = np.zeros(6, dtype=np.float64)
        n = C.c_int32(0)
        _lib.check(_lib.gpu().tri_ivf_stage_times(self.handle, ms.ctypes.data, C.byref(n)))
        return dict(zip(self.STAGES, ms.tolist())), n.value

    def last_scan_bytes(self):
        b = C.c_int64(0)
        p = C.c_int64(0)
        _lib.check(_lib.gpu().tri_ivf_last_scan_bytes(self.handle, C.byref(b), C.byref(p)))
        return b.value, p.value

    def last_scan_kind(self) -> str:
        """"f16" (fp16 tensor-core candidates), "f32" (fp32 / TF32 candidates) or "none"."""
        k = C.c_int32(0)
        _lib.check(_lib.gpu().tri_ivf_last_scan_kind(self.handle, C.byref(k)))
        return {2: "f16", 1: "f32"}.get(k.value, "none")


IVF_MAGIC = b"TRIVF001"


def write_ivf(path: str, centroids: np.ndarray, assign: np.ndarray) -> None:
    cen = np.ascontiguousarray(centroids, dtype="<f4")
    asg = np.ascontiguousarray(assign, dtype="<i4")
    if cen.ndim != 2 or asg.ndim != 1:
        raise ValueError("centroids must be 2-D and assign 1-D")
    if asg.size and (asg.min() < 0 or asg.max() >= cen.shape[0]):
        raise ValueError("assign holds list ids outside [0, nlist)")
    with open(path, "wb") as f:
        f.write(IVF_MAGIC)
        f.write(np.array([cen.shape[0], asg.shape[0], cen.shape[1]], dtype="<u8").tobytes())
        f.write(cen.tobytes())
        f.write(asg.tobytes())


def read_ivf(path: str):
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < 32 or raw[:8] != IVF_MAGIC:
        raise ValueError(f"{path}: not an IVF index file")
    nlist, n, d = (int(v) for v in np.frombuffer(raw[8:32], dtype="<u8"))
    want = 32 + 4 * nlist * d + 4 * n
    if len(raw) != want:
        raise ValueError(f"{path}: expected {want} bytes for nlist={nlist}, n={n}, d={d}, got {len(raw)}")
    cen = np.frombuffer(raw[32:32 + 4 * nlist * d], dtype="<f4").reshape(nlist, d).astype(np.float32)
    asg = np.frombuffer(raw[32 + 4 * nlist * d:], dtype="<i4").astype(np.int32)
    if asg.size and (asg.min() < 0 or asg.max() >= nlist):
        raise ValueError(f"{path}: list ids outside [0, {nlist})")
    return cen, asg


def merge_topk_device(dists, ids, k_out: int, out_dists, out_ids, stream=None) -> None:
    """Exact (dist, id) merge of per-shard lists on the device (tensors [G, B, k_in])."""
    G, B, k_in = (int(x) for x in dists.shape)
    st = None
    if stream is not None:
        st = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    _lib.check(_lib.gpu().tri_merge_topk(_lib.ptr(dists), _lib.ptr(ids), G, B, k_in, int(k_out), _lib.ptr(out_dists),
                                         _lib.ptr(out_ids), st))


__all__ = ["IVFFlatIndex", "init_rows", "merge_topk_device", "_DeviceStore"]
