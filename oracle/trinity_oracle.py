"""CPU oracle for the Trinity vector-search hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2512_02281_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may call it, and only as the
checker or as the timed CPU baseline -- never as the product path.

It restates, in numpy, the reference's algorithm for the path named by
BASELINE.json (citations are ``path:line`` under the read-only reference
``pkg/src/trinity/``):

* ``sq_dists``            <- ``ann_graph.rowwise_sq_dists``  (ann_graph.py:97-105)
* ``pair_distance``       <- ``ann_graph.distance``          (ann_graph.py:113-121)
* ``exact_knn``           <- ``ann_graph.brute_force_knn``   (ann_graph.py:124-137)
* ``ivf_search``          <- composition of the two above: the
  reference has no IVF, so the IVF oracle is built from its primitives with the
  same (dist, id) tie semantics.
* ``merge_shards``        <- (dist, id) lexicographic merge, the tie rule of
  ann_graph.py:8-9 applied to per-shard lists.
* ``engine_run``          <- ``engine.ContinuousBatchEngine`` driven by a
  submit/step schedule (engine.py:136-422): seed, parents, expand, task-array
  accounting, distances, merge, early stop, finalize.

Parity pin: ``tests/golden/`` holds vectors produced by importing the reference
itself (``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py`` checks
this module against them bit-for-bit.

Summation order.  The reference's distance is ``np.einsum("ij,ij->i", diff,
diff)`` on float64.  numpy evaluates that contraction with its SSE2 baseline
kernel: two float64 lanes, the row walked in blocks of 8 elements whose four
2-lane sub-blocks are accumulated in *reverse* order, unfused multiply then
add, a 2-lane tail, and finally ``lane0 + lane1``.  ``sq_dist_scalar_order``
spells that order out in pure Python; the CUDA re-rank kernel implements the
same order, which is why GPU distances are bit-identical to the reference's.
"""

from __future__ import annotations

import numpy as np

# ----------------------------------------------------------------------------
# distances


def sq_dists(query64: np.ndarray, rows64: np.ndarray) -> np.ndarray:
    """Squared L2 from one float64 query to each float64 row (ann_graph.py:97-105)."""
    delta = query64 - rows64
    return np.einsum("ij,ij->i", delta, delta)


def sq_dist_scalar_order(q64, x64) -> float:
    """The exact float64 operation order numpy's einsum uses for one row.

    Slow pure-Python statement of the order the GPU re-rank kernel follows
    (see module docstring); used by tests to pin that order against numpy.
    """
    d = len(q64)
    lane = [0.0, 0.0]
    i = 0
    while d - i >= 8:
        for sub in (3, 2, 1, 0):
            for ln in (0, 1):
                t = float(q64[i + 2 * sub + ln]) - float(x64[i + 2 * sub + ln])
                lane[ln] = t * t + lane[ln]
        i += 8
    while i < d:
        for ln in (0, 1):
            if i + ln < d:
                t = float(q64[i + ln]) - float(x64[i + ln])
                lane[ln] = t * t + lane[ln]
        i += 2
    return lane[0] + lane[1]


def pair_distance(a, b) -> float:
    """Checked single-pair squared distance (ann_graph.py:113-121)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    if not (np.isfinite(a).all() and np.isfinite(b).all()):
        raise ValueError("vectors must be finite")
    return float(sq_dists(a, b.reshape(1, -1))[0])


def _chunked_sq_dists(q64: np.ndarray, data32: np.ndarray, rows=None, chunk: int = 65536) -> np.ndarray:
    """sq_dists over (a subset of) a float32 matrix without a full float64 copy.

    Equal bit-for-bit to one big call: the reference's per-row reduction does
    not depend on how many rows share the call (ann_graph.py:98-103).
    """
    n = data32.shape[0] if rows is None else len(rows)
    out = np.empty(n, dtype=np.float64)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        block = data32[s:e] if rows is None else data32[rows[s:e]]
        out[s:e] = sq_dists(q64, block.astype(np.float64))
    return out


def _lex_topk(dists: np.ndarray, ids: np.ndarray, k: int):
    """k smallest by (dist, id), the rule of ann_graph.py:136."""
    order = np.lexsort((ids, dists))[:k]
    return ids[order].astype(np.int64), dists[order]


# ----------------------------------------------------------------------------
# exact kNN


def exact_knn(data32: np.ndarray, query, k: int):
    """brute_force_knn restated (ann_graph.py:124-137): (ids int64[k], dists f64[k])."""
    q = np.asarray(query, dtype=np.float64).ravel()
    n, d = data32.shape
    if q.shape[0] != d:
        raise ValueError(f"query dim {q.shape[0]} != store dim {d}")
    if not 1 <= k <= n:
        raise ValueError(f"k must be in [1, {n}], got {k}")
    dists = _chunked_sq_dists(q, data32)
    return _lex_topk(dists, np.arange(n, dtype=np.int64), k)


def exact_knn_batch(data32: np.ndarray, queries, ks):
    """exact_knn per row of ``queries``; ``ks`` is an int or one k per query."""
    queries = np.asarray(queries)
    ks = np.broadcast_to(np.asarray(ks, dtype=np.int64), (queries.shape[0],))
    return [exact_knn(data32, queries[i], int(ks[i])) for i in range(queries.shape[0])]


# ----------------------------------------------------------------------------
# IVF-Flat (composed from the reference primitives)


class IVFArtifact:
    """Shared index artifact: fp32 centroids + the list id of every vector.

    The GPU index and this oracle consume the same artifact, so parity checks
    isolate search from training.  Lists hold global ids in ascending order.
    """

    def __init__(self, centroids: np.ndarray, assign: np.ndarray):
        self.centroids = np.ascontiguousarray(centroids, dtype=np.float32)
        self.assign = np.ascontiguousarray(assign, dtype=np.int32)
        nlist = self.centroids.shape[0]
        order = np.argsort(self.assign, kind="stable")
        counts = np.bincount(self.assign, minlength=nlist)
        self.offsets = np.zeros(nlist + 1, dtype=np.int64)
        np.cumsum(counts, out=self.offsets[1:])
        self.list_ids = order.astype(np.int64)  # ascending id inside every list

    @property
    def nlist(self) -> int:
        return self.centroids.shape[0]

    def members(self, lst: int) -> np.ndarray:
        return self.list_ids[self.offsets[lst]:self.offsets[lst + 1]]


def coarse_probe(art: IVFArtifact, query, nprobe: int) -> np.ndarray:
    """Probed list ids: brute_force_knn over the centroids (ann_graph.py:124-137)."""
    ids, _ = exact_knn(art.centroids, query, nprobe)
    return ids


def ivf_search(data32: np.ndarray, art: IVFArtifact, query, k: int, nprobe: int):
    """Exact top-k over the union of the nprobe closest lists.

    Coarse step = brute_force_knn over centroids; fine step = the probed
    lists' ids in ascending order, rowwise_sq_dists, then lexsort by
    (dist, id) -- identical tie semantics to ann_graph.py:136.  Returns fewer
    than k results when the probed lists hold fewer than k vectors.
    """
    q = np.asarray(query, dtype=np.float64).ravel()
    probes = coarse_probe(art, q, nprobe)
    cand = np.sort(np.concatenate([art.members(int(p)) for p in probes]))
    if cand.size == 0:
        return np.empty(0, np.int64), np.empty(0, np.float64)
    dists = _chunked_sq_dists(q, data32, rows=cand)
    return _lex_topk(dists, cand, min(k, cand.size))


def nearest_centroid(data32: np.ndarray, cent32: np.ndarray, chunk: int = 8192) -> np.ndarray:
    """Exact nearest centroid of every row: ``brute_force_knn(VectorStore(cent), row, 1)``
    (ann_graph.py:124-137) per row, i.e. the smallest float64 einsum-order
    distance, ties to the smaller centroid id.

    Vectorised: the float64 score S = |c|^2 - 2 x.c (the row's |x|^2 is a
    common constant) picks the candidates; rows whose runner-up lies within
    twice the error bound of the winner are decided by the exact distances.
    |S + |x|^2 - D| <= eps (|x| + |c|)^2 with eps = 4 (d + 4) 2^-53 covers S's
    rounding (any BLAS order) and D's own einsum rounding, so the exact winner
    is always among the candidates.  Chunks run on a thread pool (numpy and
    BLAS release the GIL; BLAS pinned to one thread per chunk).
    """
    from concurrent.futures import ThreadPoolExecutor
    import os

    from threadpoolctl import threadpool_limits

    n, d = data32.shape
    c64 = cent32.astype(np.float64)
    cn = np.einsum("ij,ij->i", c64, c64)
    c64t = np.ascontiguousarray(c64.T)
    cmax = float(np.sqrt(cn.max()))
    eps = 4.0 * (d + 4) * 2.0 ** -53
    out = np.empty(n, dtype=np.int32)

    def run(s):
        x = data32[s:s + chunk].astype(np.float64)
        S = x @ c64t
        S *= -2.0
        S += cn
        win = S.argmin(axis=1).astype(np.int32)
        smin = S[np.arange(S.shape[0]), win]
        xn = np.einsum("ij,ij->i", x, x)
        S -= (smin + 2.0 * eps * (np.sqrt(xn) + cmax) ** 2)[:, None]
        multi = np.nonzero((S <= 0.0).sum(axis=1) > 1)[0]
        for r in multi:
            cs = np.nonzero(S[r] <= 0.0)[0]
            dd = sq_dists(x[r], c64[cs])
            win[r] = cs[np.lexsort((cs, dd))[0]]
        out[s:s + chunk] = win

    with threadpool_limits(1, "blas"), ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        list(ex.map(run, range(0, n, chunk)))
    return out


def kmeans(data32: np.ndarray, nlist: int, iters: int, seed: int):
    """Lloyd k-means, the restatement of the GPU trainer (tri_ivf_train).

    The reference has no IVF, so there is nothing to pin it to;
    its semantics are chosen to be deterministic so the GPU result can be
    checked bit-for-bit: centroids start from the seeded rows
    ``sort(choice(n, nlist))`` of a Philox(seed) generator; every iteration
    assigns each row to its exact nearest centroid (``nearest_centroid``),
    then each non-empty list's centroid becomes fp32(sum * (1 / count)) with
    the sum taken in float64 over its rows in ascending id order (numpy's
    axis-0 sum is that sequential chain); empty lists keep their centroid.
    After ``iters`` updates a final assignment gives the artifact.
    """
    rng = np.random.Generator(np.random.Philox(seed))
    n = data32.shape[0]
    cent = np.ascontiguousarray(data32[np.sort(rng.choice(n, size=nlist, replace=False))], dtype=np.float32)
    for it in range(iters + 1):
        assign = nearest_centroid(data32, cent)
        if it == iters:
            break
        order = np.argsort(assign, kind="stable")
        counts = np.bincount(assign, minlength=nlist)
        off = np.zeros(nlist + 1, dtype=np.int64)
        np.cumsum(counts, out=off[1:])
        for lst in np.nonzero(counts)[0]:
            rows = order[off[lst]:off[lst + 1]]
            s = data32[rows].astype(np.float64).sum(axis=0)
            cent[lst] = (s * (1.0 / counts[lst])).astype(np.float32)
    return IVFArtifact(cent, assign)


def artifact_digest(art: "IVFArtifact") -> str:
    """sha256 prefix of (centroids, assign): both bench arms print it."""
    import hashlib

    h = hashlib.sha256(np.ascontiguousarray(art.centroids, dtype="<f4").tobytes())
    h.update(np.ascontiguousarray(art.assign, dtype="<i4").tobytes())
    return h.hexdigest()[:16]


# ----------------------------------------------------------------------------
# shard merge


def merge_shards(parts, k: int):
    """Merge per-shard (ids, dists) lists into the global top-k by (dist, id)."""
    ids = np.concatenate([np.asarray(p[0], dtype=np.int64) for p in parts])
    dists = np.concatenate([np.asarray(p[1], dtype=np.float64) for p in parts])
    keep = ids >= 0
    ids, dists = ids[keep], dists[keep]
    return _lex_topk(dists, ids, min(k, ids.size))


# ----------------------------------------------------------------------------
# continuous-batching graph engine


def engine_run(data32: np.ndarray, adjacency: np.ndarray, queries, ks, admit_step, m: int = 64, p: int = 2,
               entry_count: int = 8, batch_capacity: int = 512, stop_streak: int = 1, max_extends: int = 256):
    """Restatement of the reference engine's state machine (engine.py:136-422).

    Query i is submitted just before step ``admit_step[i]`` (a non-decreasing
    schedule); steps continue until no request is active, as
    ``step()`` x waves followed by ``run_to_completion()``.  Returns
    (ids list, dists list, extends array, batch_real_counts, n_steps).
    """
    n = data32.shape[0]
    queries = np.asarray(queries, dtype=np.float64)
    nq = queries.shape[0]
    entries = list(dict.fromkeys(i * n // entry_count for i in range(entry_count)))  # engine.py:136-143
    states = {}
    out_ids, out_d = [None] * nq, [None] * nq
    extends = np.zeros(nq, dtype=np.int64)
    batch_real_counts = []
    nxt = 0
    step = 0
    while nxt < nq or states:
        while nxt < nq and admit_step[nxt] <= step:  # seed at submit, admitted at step start
            q = queries[nxt]
            dd = sq_dists(q, data32[entries].astype(np.float64))
            top = sorted(((float(d), v, False) for v, d in zip(entries, dd)))
            states[nxt] = {"q": q, "top": [list(t) for t in top], "vis": set(entries), "ext": 0, "streak": 0}
            nxt += 1
        total = 0
        emitted = {}
        for rid in sorted(states):  # engine.py:379-385
            st = states[rid]
            parents = [e for e in st["top"] if not e[2]][:p]  # engine.py:176-184
            em = []
            for e in parents:  # engine.py:187-205
                for nid in adjacency[e[1]]:
                    nid = int(nid)
                    if nid not in st["vis"]:
                        st["vis"].add(nid)
                        em.append(nid)
                e[2] = True
            emitted[rid] = em
            total += len(em)
        for s0 in range(0, total, batch_capacity):  # build_task_array accounting, engine.py:208-226
            batch_real_counts.append(min(batch_capacity, total - s0))
        for rid in sorted(states):
            st = states[rid]
            em = emitted[rid]
            changed = False
            if em:  # scatter_merge, engine.py:259-275
                dd = sq_dists(st["q"], data32[em].astype(np.float64))
                before = [e[1] for e in st["top"]]
                pool = st["top"] + [[float(d), c, False] for c, d in zip(em, dd)]
                pool.sort(key=lambda e: (e[0], e[1]))
                st["top"] = pool[:m]
                changed = [e[1] for e in st["top"]] != before
            st["ext"] += 1
            st["streak"] = 0 if changed else st["streak"] + 1  # engine.py:278-290
            if (st["streak"] >= stop_streak or all(e[2] for e in st["top"]) or st["ext"] >= max_extends):
                k = int(ks[rid])
                out_ids[rid] = np.array([e[1] for e in st["top"][:k]], dtype=np.int64)
                out_d[rid] = np.array([e[0] for e in st["top"][:k]], dtype=np.float64)
                extends[rid] = st["ext"]
                del states[rid]
        step += 1
    return out_ids, out_d, extends, batch_real_counts, step
