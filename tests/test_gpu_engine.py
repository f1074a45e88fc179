"""Engine drop-in on the GPU: bit-exact against the reference's acceptance run."""

import os

import numpy as np
import pytest

from paper_2512_02281_b200.ann_graph import NeighborGraph, VectorStore, build_knn_graph, distance
from paper_2512_02281_b200.engine import (
    ContinuousBatchEngine,
    EngineConfig,
    build_task_array,
    execute_distance_batch,
    search_sequential,
    seed_request,
)
from paper_2512_02281_b200.workload import gen_matrix

pytestmark = pytest.mark.gpu


def test_acceptance_workload_bit_exact(golden_dir):
    """test_acceptance.py:47-81 workload (200 queries, 10 waves): ids, dists,
    extends and fixed-shape accounting equal the reference's run exactly."""
    g = np.load(os.path.join(golden_dir, "engine_c1.npz"))
    store = VectorStore(data=gen_matrix(5000, 16, 20_240_601))
    graph = NeighborGraph(degree=16, adjacency=g["adjacency"])
    queries = gen_matrix(200, 16, 20_240_602)
    eng = ContinuousBatchEngine(store, graph, EngineConfig(m=64, p=2, entry_count=8, batch_capacity=512))
    rids = []
    for wave in range(10):
        for q in queries[wave * 20:(wave + 1) * 20]:
            rids.append(eng.submit(q, k=10))
        eng.step()
    eng.run_to_completion()
    for i, rid in enumerate(rids):
        res = eng.result(rid)
        assert [n.id for n in res.neighbors] == g["ids"][i].tolist()
        assert [n.dist for n in res.neighbors] == g["dists"][i].tolist()
        assert res.extends == int(g["extends"][i])
    st = eng.stats
    assert st.batch_real_counts == g["batch_real_counts"].tolist()
    assert (st.emissions, st.real_tasks, st.dummy_tasks) == (int(g["emissions"]), int(g["real_tasks"]),
                                                              int(g["dummy_tasks"]))
    assert st.batches_launched == 144 and st.real_tasks == 62736  # pkg/test_output.txt:16


def test_staggered_equals_solo():
    store = VectorStore(data=gen_matrix(1000, 8, 101))
    graph = build_knn_graph(store, 8)
    cfg = EngineConfig(m=16, p=2, entry_count=4, batch_capacity=32)
    queries = gen_matrix(12, 8, 55)
    eng = ContinuousBatchEngine(store, graph, cfg)
    rids = []
    for i, q in enumerate(queries):
        rids.append(eng.submit(q, k=5))
        if i % 3 == 2:
            eng.step()
    eng.run_to_completion()
    for q, rid in zip(queries, rids):
        solo = search_sequential(q, store, graph, cfg, 5)
        got = eng.result(rid)
        assert [(n.id, n.dist) for n in solo.neighbors] == [(n.id, n.dist) for n in got.neighbors]
        assert solo.extends == got.extends


def test_distance_batch_semantics(golden_dir):
    g = np.load(os.path.join(golden_dir, "mixed_batch.npz"))
    store = VectorStore(data=gen_matrix(50, 4, 3))
    qd = {0: g["q0"], 1: g["q1"]}
    batch = build_task_array({0: [5, 9, 11], 1: [2, 5, 40, 41, 42]}, 8)[0]
    res = execute_distance_batch(batch, store, qd)
    assert [(o, c) for o, c, _ in res] == list(zip(g["owners"].tolist(), g["cands"].tolist()))
    assert [x for _, _, x in res] == g["dists"].tolist()
    line = VectorStore(data=np.array([[0.0], [1.0], [2.0]], np.float32))
    with pytest.raises(RuntimeError):
        execute_distance_batch(build_task_array({0: [7]}, 2)[0], line, {0: np.array([0.0])})
    r = execute_distance_batch(build_task_array({0: [1]}, 4)[0], line, {0: np.array([0.9])})
    assert r[0][2] == distance(np.array([0.9]), np.array([1.0], np.float32))


def test_seed_request_validation():
    line = VectorStore(data=np.array([[0.0], [1.0], [2.0]], np.float32))
    cfg = EngineConfig(m=3, entry_count=1, p=1)
    st = seed_request(line.data[0], "prefill", 0.0, None, 1, cfg, line)
    assert st.top_m[0].id == 0 and st.top_m[0].dist == 0.0 and st.visited == {0}
    with pytest.raises(ValueError):
        seed_request(line.data[0], "prefill", 0.0, None, 4, cfg, line)
    with pytest.raises(ValueError):
        seed_request(np.zeros(2), "prefill", 0.0, None, 1, cfg, line)
    with pytest.raises(ValueError):
        seed_request(np.array([np.nan]), "prefill", 0.0, None, 1, cfg, line)
