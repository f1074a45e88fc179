"""Vector store, exact kNN and neighbor graphs -- the reference's ``ann_graph``
API (pkg/src/trinity/ann_graph.py) backed by the B200 library.

Drop-in surface: ``VectorStore``, ``NeighborGraph``, ``Neighbor``,
``rowwise_sq_dists``, ``pair_sq_dist``, ``distance``, ``brute_force_knn``,
``build_knn_graph``, ``validate_graph`` and the binary file formats keep the
reference's names, argument meaning and errors.  Distances are computed on the
GPU in the reference's exact float64 operation order, so results are
bit-identical.  New: ``brute_force_knn_batch`` (one launch
for many queries, per-query k).

Differences, all deliberate:
* ``VectorStore`` keeps NO eager float64 copy (ann_graph.py:40 doubles host
  memory); ``data64`` is a lazily computed host convenience that the search
  path never touches.  The device copy is created on first GPU use.
* Non-finite queries raise ValueError (the reference silently returns NaN
  distances).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

SUPPORTED_METRICS = ("l2sq",)


class _DeviceStore:
    """Owner of one ``tri_store`` handle (device-resident fp32 rows)."""

    def __init__(self, data: np.ndarray, device: int = 0, id_offset: int = 0):
        lib = _lib.gpu()
        h = C.c_void_p()
        data = np.ascontiguousarray(data, dtype=np.float32)
        _lib.check(lib.tri_store_create(data.ctypes.data, data.shape[0], data.shape[1], device, C.byref(h)))
        self.handle = h
        self.n, self.d = data.shape
        self.device = device
        if id_offset:
            _lib.check(lib.tri_store_set_id_offset(h, int(id_offset)))

    def close(self) -> None:
        if self.handle:
            _lib.load_library().tri_store_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def knn(self, queries64: np.ndarray, ks: np.ndarray):
        """Batched exact kNN: (ids int64[B, kmax], dists f64[B, kmax])."""
        lib = _lib.gpu()
        q = np.ascontiguousarray(queries64, dtype=np.float64)
        B = q.shape[0]
        ks = np.ascontiguousarray(ks, dtype=np.int32)
        kmax = int(ks.max()) if B else 1
        ids = np.empty((B, kmax), dtype=np.int64)
        dists = np.empty((B, kmax), dtype=np.float64)
        if B:
            _lib.check(lib.tri_knn_bruteforce(self.handle, q.ctypes.data, B, ks.ctypes.data, kmax,
                                              ids.ctypes.data, dists.ctypes.data, None))
        return ids, dists

    def knn_into(self, q_host, ks, ids_out, dists_out, stream=None) -> None:
        """Blocking batched exact kNN into caller-owned host arrays [B, ldo]
        (pinned buffers let a repeated shape replay as one CUDA graph)."""
        from .ivf import _check_buf, _stream_ptr

        B = int(q_host.shape[0])
        _check_buf("queries", q_host, "float64", cols=self.d)
        _check_buf("ids_out", ids_out, "int64", rows=B)
        _check_buf("dists_out", dists_out, "float64", cols=int(ids_out.shape[1]), rows=B)
        ks = np.ascontiguousarray(np.broadcast_to(np.asarray(ks, dtype=np.int64), (B,)), dtype=np.int32)
        if B:
            _lib.check(_lib.gpu().tri_knn_bruteforce(self.handle, _lib.ptr(q_host), B, ks.ctypes.data,
                                                     int(ids_out.shape[1]), _lib.ptr(ids_out), _lib.ptr(dists_out),
                                                     _stream_ptr(stream)))

    def task_dists(self, owner: np.ndarray, cand: np.ndarray, queries64: np.ndarray) -> np.ndarray:
        lib = _lib.gpu()
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        cand = np.ascontiguousarray(cand, dtype=np.int64)
        q = np.ascontiguousarray(queries64, dtype=np.float64)
        if q.ndim != 2 or q.shape[1] != self.d:
            raise ValueError(f"queries must be (n, {self.d}), got shape {q.shape}")
        if owner.shape != cand.shape:
            raise ValueError(f"owner {owner.shape} and cand {cand.shape} differ in length")
        out = np.empty(owner.shape[0], dtype=np.float64)
        if owner.shape[0]:
            _lib.check(lib.tri_distance_tasks(self.handle, owner.ctypes.data, cand.ctypes.data, owner.shape[0],
                                              q.ctypes.data, q.shape[0], out.ctypes.data, None))
        return out

    def last_fixups(self) -> int:
        n = C.c_int32(0)
        _lib.check(_lib.gpu().tri_store_last_fixups(self.handle, C.byref(n)))
        return n.value


@dataclass(frozen=True)
class VectorStore:
    """N x d matrix of finite float32 vectors (ann_graph.py:21-48), device-backed."""

    data: np.ndarray

    def __post_init__(self) -> None:
        arr = np.asarray(self.data)
        if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
            raise ValueError(f"vector store must be a nonempty 2-D matrix, got shape {arr.shape}")
        arr = np.ascontiguousarray(arr, dtype=np.float32)
        if not np.isfinite(arr).all():
            raise ValueError("vector store entries must all be finite")
        object.__setattr__(self, "data", arr)
        object.__setattr__(self, "_dev", None)

    @property
    def count(self) -> int:
        return self.data.shape[0]

    @property
    def dim(self) -> int:
        return self.data.shape[1]

    @property
    def data64(self) -> np.ndarray:
        """Host float64 view for compatibility; the GPU path never uses it."""
        return self.data.astype(np.float64)

    def device(self) -> _DeviceStore:
        """The device copy (created on first use; requires a CUDA device)."""
        dev = self.__dict__.get("_dev")
        if dev is None:
            dev = _DeviceStore(self.data)
            object.__setattr__(self, "_dev", dev)
        return dev


@dataclass(frozen=True)
class NeighborGraph:
    """Fixed out-degree adjacency, row i = neighbor ids of vector i (ann_graph.py:51-70)."""

    degree: int
    adjacency: np.ndarray

    def __post_init__(self) -> None:
        adj = np.asarray(self.adjacency)
        if adj.ndim != 2:
            raise ValueError(f"adjacency must be 2-D, got shape {adj.shape}")
        if adj.shape[1] != self.degree:
            raise ValueError(f"adjacency has {adj.shape[1]} columns but degree is {self.degree}")
        object.__setattr__(self, "adjacency", np.ascontiguousarray(adj, dtype=np.uint32))

    @property
    def count(self) -> int:
        return self.adjacency.shape[0]


@dataclass(frozen=True)
class Neighbor:
    """One search result: vector id and squared Euclidean distance."""

    id: int
    dist: float


@dataclass
class GraphValidationReport:
    range_violations: list = field(default_factory=list)  # (row, bad id)
    self_loops: list = field(default_factory=list)
    duplicate_rows: list = field(default_factory=list)
    wrong_row_length: list = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not any((self.range_violations, self.self_loops, self.duplicate_rows, self.wrong_row_length))


# ----------------------------------------------------------------------------
# distances


def rowwise_sq_dists(query64: np.ndarray, rows64: np.ndarray) -> np.ndarray:
    """Squared L2 from the query to each row (ann_graph.py:97-105), on the GPU.

    Same broadcasting as the reference's ``query64 - rows64``: a (d,) or (1, d)
    query against (n, d) rows, or one query row per row.  Float64 on both sides
    (``tri_rowwise_sq_dists_f64``), in the reference's einsum operation order.
    """
    q = np.asarray(query64, dtype=np.float64)
    rows = np.asarray(rows64, dtype=np.float64)
    try:
        shape = np.broadcast_shapes(q.shape, rows.shape)
    except ValueError as exc:
        raise ValueError(f"query {q.shape} does not broadcast against rows {rows.shape}") from exc
    if len(shape) != 2:
        raise ValueError(f"query - rows must be 2-D (rows, dim), got shape {shape}")
    n, d = shape
    if n == 0:
        return np.empty(0, dtype=np.float64)
    # (q - x)^2 == (x - q)^2 exactly, so either operand may play the query
    if q.shape[-1:] == (d,) and q.size == d:
        one, full = q.reshape(1, d), rows
    elif rows.size == d:
        one, full = rows.reshape(1, d), q
    else:
        one, full = None, None
    if one is not None and full.shape == (n, d):
        qb, xb, qrows = np.ascontiguousarray(one), np.ascontiguousarray(full), 1
    else:
        qb = np.ascontiguousarray(np.broadcast_to(q, shape))
        xb = np.ascontiguousarray(np.broadcast_to(rows, shape))
        qrows = n
    out = np.empty(n, dtype=np.float64)
    _lib.check(_lib.gpu().tri_rowwise_sq_dists_f64(qb.ctypes.data, qrows, xb.ctypes.data, n, d, 0, out.ctypes.data))
    return out


def store_sq_dists(store: VectorStore, query, rows) -> np.ndarray:
    """rowwise_sq_dists(query, store.data64[rows]) without materialising rows."""
    q = np.asarray(query, dtype=np.float64)
    if q.size != store.dim:
        raise ValueError(f"query has {q.size} values, store dim is {store.dim}")
    rows = np.asarray(rows, dtype=np.int64)
    return store.device().task_dists(np.zeros(rows.shape[0], np.int32), rows, q.reshape(1, -1))


def pair_sq_dist(query64: np.ndarray, row64: np.ndarray) -> float:
    """Unchecked single-pair distance (ann_graph.py:108-110)."""
    return float(rowwise_sq_dists(query64, np.asarray(row64).reshape(1, -1))[0])


def distance(a, b) -> float:
    """Checked squared Euclidean distance (ann_graph.py:113-121)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    if not (np.isfinite(a).all() and np.isfinite(b).all()):
        raise ValueError("vectors must be finite")
    return pair_sq_dist(a, b)


# ----------------------------------------------------------------------------
# exact kNN


def _check_queries(store: VectorStore, queries: np.ndarray) -> None:
    if queries.shape[1] != store.dim:
        raise ValueError(f"query dim {queries.shape[1]} != store dim {store.dim}")


def brute_force_knn_batch(store: VectorStore, queries, k):
    """Exact kNN for a batch (one device launch sequence); k is an int or per-query array.

    Returns (ids int64[B, kmax], dists f64[B, kmax]); row i's first k[i]
    entries are sorted by (dist, id).
    """
    q = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    _check_queries(store, q)
    ks = np.broadcast_to(np.asarray(k, dtype=np.int64), (q.shape[0],))
    bad = (ks < 1) | (ks > store.count)
    if bad.any():
        raise ValueError(f"k must be in [1, {store.count}], got {int(ks[bad][0])}")
    return store.device().knn(q, ks.astype(np.int32))


def brute_force_knn(store: VectorStore, query, k: int) -> list:
    """Exact k nearest neighbors sorted by (dist, id) (ann_graph.py:124-137)."""
    q = np.asarray(query, dtype=np.float64).ravel()
    if q.shape[0] != store.dim:
        raise ValueError(f"query dim {q.shape[0]} != store dim {store.dim}")
    if not 1 <= k <= store.count:
        raise ValueError(f"k must be in [1, {store.count}], got {k}")
    ids, dists = store.device().knn(q.reshape(1, -1), np.array([k], np.int32))
    return [Neighbor(id=int(i), dist=float(d)) for i, d in zip(ids[0], dists[0])]


def build_knn_graph(store: VectorStore, degree: int, block: int = 4096) -> NeighborGraph:
    """Exact kNN graph (ann_graph.py:140-165): row i = the `degree` nearest other vectors.

    Self edges excluded, ties by smaller id.  Every row is a device brute-force
    query with k = degree + 1 (self dropped); distances use the reference's
    einsum order, i.e. the per-row oracle of test_ann_graph.py:98-103.
    """
    n = store.count
    if not 1 <= degree < n:
        raise ValueError(f"degree must be in [1, {n - 1}], got {degree}")
    adjacency = np.empty((n, degree), dtype=np.uint32)
    k = degree + 1
    dev = store.device()
    for s in range(0, n, block):
        e = min(n, s + block)
        ids, _ = dev.knn(store.data[s:e].astype(np.float64), np.full(e - s, k, np.int32))
        for j, row in enumerate(ids):
            i = s + j
            keep = row[row != i][:degree]
            adjacency[i] = keep
    return NeighborGraph(degree=degree, adjacency=adjacency)


def validate_graph(graph: NeighborGraph, n_db: int) -> GraphValidationReport:
    """Out-of-range ids, self loops, duplicate entries, wrong row length (ann_graph.py:168-183)."""
    rep = GraphValidationReport()
    adj = graph.adjacency
    if adj.shape[1] != graph.degree:
        rep.wrong_row_length = list(range(adj.shape[0]))
    for i, row in enumerate(adj):
        rep.range_violations.extend((i, int(v)) for v in row if int(v) >= n_db)
        if (row == i).any():
            rep.self_loops.append(i)
        if np.unique(row).size != row.size:
            rep.duplicate_rows.append(i)
    return rep


# ----------------------------------------------------------------------------
# file formats (ann_graph.py:186-244): vector records `<u4 d` + d x `<f4`;
# graph = `<u8 N, <u8 D` header + N*D `<u4` ids.


def write_vectors(path: str, data: np.ndarray) -> None:
    arr = np.asarray(data, dtype=np.float32)
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"expected a nonempty 2-D matrix, got shape {arr.shape}")
    rec = np.empty((arr.shape[0], arr.shape[1] + 1), dtype="<u4")
    rec[:, 0] = arr.shape[1]
    rec[:, 1:] = arr.astype("<f4").view("<u4")
    with open(path, "wb") as f:
        f.write(rec.tobytes())


def read_vectors(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        raw = f.read()
    if not raw:
        return np.empty((0, 0), dtype=np.float32)  # an empty query file is legal
    if len(raw) < 4:
        raise ValueError(f"{path}: not a vector file (shorter than one header)")
    d = int(np.frombuffer(raw[:4], dtype="<u4")[0])
    if d < 1:
        raise ValueError(f"{path}: record dimension must be >= 1, got {d}")
    rb = 4 * (d + 1)
    if len(raw) % rb:
        raise ValueError(f"{path}: size {len(raw)} is not a multiple of the record size {rb}")
    rec = np.frombuffer(raw, dtype="<u4").reshape(-1, d + 1)
    if not (rec[:, 0] == d).all():
        raise ValueError(f"{path}: records disagree on dimension")
    return rec[:, 1:].copy().view("<f4").astype(np.float32)


def write_graph(path: str, graph: NeighborGraph) -> None:
    with open(path, "wb") as f:
        f.write(np.array([graph.adjacency.shape[0], graph.degree], dtype="<u8").tobytes())
        f.write(graph.adjacency.astype("<u4").tobytes())


def read_graph(path: str) -> NeighborGraph:
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < 16:
        raise ValueError(f"{path}: not a graph file (missing 16-byte header)")
    n, d = (int(v) for v in np.frombuffer(raw[:16], dtype="<u8"))
    if len(raw) != 16 + 4 * n * d:
        raise ValueError(f"{path}: expected {16 + 4 * n * d} bytes for a {n}x{d} graph, got {len(raw)}")
    return NeighborGraph(degree=d, adjacency=np.frombuffer(raw[16:], dtype="<u4").reshape(n, d).copy())
