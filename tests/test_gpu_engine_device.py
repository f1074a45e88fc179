"""Device-resident engine (csrc/tri_engine.cu) against the CPU engine oracle.

The oracle (oracle.engine_run) is pinned to the reference's own acceptance run
(tests/test_oracle_golden.py::test_engine_oracle_matches_reference_run); here
the device engine must reproduce it bit-for-bit -- ids, float64 distances,
extends and fixed-shape batch accounting -- over configurations and
admission schedules the acceptance run does not cover.
"""

import numpy as np
import pytest

from oracle import trinity_oracle as orc
from paper_2512_02281_b200.ann_graph import NeighborGraph, VectorStore, build_knn_graph
from paper_2512_02281_b200.engine import ContinuousBatchEngine, EngineConfig, HostSteppedEngine
from paper_2512_02281_b200.workload import gen_matrix

pytestmark = pytest.mark.gpu


def _drive(eng, queries, ks, admit_step):
    rids = [None] * len(queries)
    step = 0
    i = 0
    while i < len(queries):
        while i < len(queries) and admit_step[i] <= step:
            rids[i] = eng.submit(queries[i], k=int(ks[i]))
            i += 1
        eng.step()
        step += 1
    step += eng.run_to_completion()
    return rids, step


def _check(eng, rids, ref):
    ids, d, ext, brc, _ = ref
    for i, rid in enumerate(rids):
        res = eng.result(rid)
        assert res is not None, f"request {i} never retired"
        assert [n.id for n in res.neighbors] == ids[i].tolist(), f"ids differ on request {i}"
        assert [n.dist for n in res.neighbors] == d[i].tolist(), f"dists differ on request {i}"
        assert res.extends == int(ext[i])
    assert eng.stats.batch_real_counts == brc


@pytest.mark.parametrize(
    "n,d,deg,cfg",
    [
        (20000, 128, 16, dict(m=64, p=2, entry_count=8, batch_capacity=512)),
        (8000, 768, 16, dict(m=64, p=2, entry_count=8, batch_capacity=512)),
        (6000, 32, 24, dict(m=128, p=4, entry_count=16, batch_capacity=100, stop_streak=3, max_extends=40)),
        (3000, 16, 8, dict(m=16, p=1, entry_count=3, batch_capacity=7, stop_streak=2, max_extends=5)),
        # p > 32: parents beyond one warp's lanes must be marked expanded too
        (4000, 16, 8, dict(m=64, p=40, entry_count=8, batch_capacity=256, stop_streak=2, max_extends=12)),
        # m beyond one warp's register reach and p * degree > 512 (round-1 caps lifted)
        (3000, 16, 16, dict(m=1024, p=40, entry_count=16, batch_capacity=512, stop_streak=2, max_extends=8)),
    ],
)
def test_device_engine_matches_oracle(n, d, deg, cfg):
    data = gen_matrix(n, d, 1000 + d)
    store = VectorStore(data=data)
    graph = build_knn_graph(store, deg)
    nq = 96
    queries = gen_matrix(nq, d, 2000 + d).astype(np.float64)
    rng = np.random.default_rng(d)
    ks = rng.integers(1, cfg["m"] + 1, nq)
    admit = np.sort(rng.integers(0, 12, nq))
    ref = orc.engine_run(data, graph.adjacency, queries, ks, admit, **cfg)
    eng = ContinuousBatchEngine(store, graph, EngineConfig(**cfg))
    rids, steps = _drive(eng, queries, ks, admit)
    _check(eng, rids, ref)
    assert steps == ref[4]
    assert eng.active_count == 0 and eng.pending_admissions == 0


def test_device_engine_equals_host_stepped_engine():
    data = gen_matrix(4000, 24, 7)
    store = VectorStore(data=data)
    graph = build_knn_graph(store, 12)
    cfg = EngineConfig(m=32, p=2, entry_count=5, batch_capacity=64)
    queries = gen_matrix(40, 24, 8)
    a = ContinuousBatchEngine(store, graph, cfg)
    b = HostSteppedEngine(store, graph, cfg)
    for i, q in enumerate(queries):
        ra, rb = a.submit(q, k=7), b.submit(q, k=7)
        assert ra == rb
        if i % 5 == 4:
            sa, sb = a.step(), b.step()
            assert sa == sb
            assert sorted(r.request_id for r in a.drain_retired()) == sorted(r.request_id for r in b.drain_retired())
    assert a.run_to_completion() == b.run_to_completion()
    for rid in range(len(queries)):
        x, y = a.result(rid), b.result(rid)
        assert (x.neighbors, x.extends) == (y.neighbors, y.extends)
    assert a.stats == b.stats


def test_device_engine_small_store_and_slot_reuse():
    """n < entry_count (duplicate seeds dropped, engine.py:136-143), then many
    waves so retired slots are reused."""
    data = gen_matrix(6, 3, 11)
    store = VectorStore(data=data)
    adj = np.array([[(i + j + 1) % 6 for j in range(2)] for i in range(6)], dtype=np.uint32)
    graph = NeighborGraph(degree=2, adjacency=adj)
    cfg = dict(m=8, p=1, entry_count=8, batch_capacity=4)
    queries = gen_matrix(300, 3, 12).astype(np.float64)
    ks = np.full(300, 3)
    admit = np.repeat(np.arange(30), 10)
    ref = orc.engine_run(data, adj, queries, ks, admit, **cfg)
    eng = ContinuousBatchEngine(store, graph, EngineConfig(**cfg))
    rids, steps = _drive(eng, queries, ks, admit)
    _check(eng, rids, ref)
    assert steps == ref[4]


def test_device_engine_errors():
    store = VectorStore(data=gen_matrix(50, 4, 1))
    graph = build_knn_graph(store, 4)
    eng = ContinuousBatchEngine(store, graph, EngineConfig(m=8, p=1, entry_count=2))
    with pytest.raises(ValueError):
        eng.submit(np.zeros(3), k=1)
    with pytest.raises(ValueError):
        eng.submit(np.full(4, np.nan), k=1)
    with pytest.raises(ValueError):
        eng.submit(np.zeros(4), k=9)
    # k larger than the reachable top-M: finalize raises ValueError (engine.py:299-300)
    tiny = VectorStore(data=gen_matrix(3, 2, 2))
    g2 = NeighborGraph(degree=1, adjacency=np.array([[1], [0], [0]], dtype=np.uint32))
    e2 = ContinuousBatchEngine(tiny, g2, EngineConfig(m=8, p=1, entry_count=1))
    e2.submit(np.zeros(2), k=8)
    with pytest.raises(ValueError):
        e2.run_to_completion()
    assert eng.run_to_completion() == 0


def test_device_engine_limits_and_bad_graph():
    """Config limits of the device engine and an adjacency id out of range
    (the reference raises RuntimeError for such a candidate, engine.py:249-250)."""
    store = VectorStore(data=gen_matrix(40, 4, 3))
    good = build_knn_graph(store, 4)
    with pytest.raises(ValueError):
        ContinuousBatchEngine(store, good, EngineConfig(m=5000, p=1, entry_count=2))
    wide = NeighborGraph(degree=4, adjacency=good.adjacency)
    with pytest.raises(ValueError):
        ContinuousBatchEngine(store, wide, EngineConfig(m=256, p=3000, entry_count=2))
    bad_adj = good.adjacency.copy()
    bad_adj[:, 0] = 10_000
    eng = ContinuousBatchEngine(store, NeighborGraph(degree=4, adjacency=bad_adj), EngineConfig(m=8, p=1, entry_count=2))
    eng.submit(gen_matrix(1, 4, 5)[0], k=3)
    with pytest.raises(RuntimeError):
        eng.run_to_completion()


def test_device_engine_one_slot_per_cta():
    """m = 4096 with p * degree = 4096: the per-request lists need ~160 KB of
    shared memory, so the step kernel runs one request slot per CTA."""
    data = gen_matrix(5000, 8, 31)
    store = VectorStore(data=data)
    graph = build_knn_graph(store, 64)
    cfg = dict(m=4096, p=64, entry_count=64, batch_capacity=1024, stop_streak=1, max_extends=3)
    queries = gen_matrix(4, 8, 32).astype(np.float64)
    ks = np.array([5, 50, 500, 17])
    admit = np.zeros(4, np.int64)
    ref = orc.engine_run(data, graph.adjacency, queries, ks, admit, **cfg)
    eng = ContinuousBatchEngine(store, graph, EngineConfig(**cfg))
    rids, steps = _drive(eng, queries, ks, admit)
    _check(eng, rids, ref)
