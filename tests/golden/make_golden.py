"""Generate the golden fixtures by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--reference /root/reference]

The reference package is imported read-only from its source tree; nothing is
copied into this repo except the small output arrays written next to this
script.  The GPU box never runs this file (the reference is absent there).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True


def _import_reference(root: str):
    sys.path.insert(0, os.path.join(root, "pkg", "src"))
    import trinity  # noqa: F401
    from trinity import ann_graph, engine, workload

    return ann_graph, engine, workload


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_distance_kats(ag):
    rng = np.random.Generator(np.random.Philox(5))
    cases = []
    for _ in range(50):
        d = int(rng.integers(1, 48))
        a = rng.standard_normal(d).astype(np.float32)
        b = rng.standard_normal(d).astype(np.float32)
        cases.append({"a": a.tolist(), "b": b.tolist(), "dist": ag.distance(a, b)})
    cases.append({"a": [0.0, 0.0], "b": [3.0, 4.0], "dist": ag.distance(np.zeros(2), np.array([3.0, 4.0]))})
    v = [1.5, -2.0, 0.25]
    cases.append({"a": v, "b": v, "dist": ag.distance(np.array(v, np.float32), np.array(v, np.float32))})
    with open(os.path.join(HERE, "distance_kats.json"), "w") as f:
        json.dump(cases, f)


def gen_bruteforce(ag, wl):
    # test_ann_graph.py:65-75 workload: 1000 x 8 (seed 11), 20 float64 Philox(12) queries.
    store = wl.gen_vectors(1000, 8, seed=11)
    rng = np.random.Generator(np.random.Philox(12))
    queries = np.stack([rng.standard_normal(8) for _ in range(20)])
    ks = [10, 1, 37, 1000]
    out = {"queries": queries, "db_sha": np.array(_sha(store.data))}
    for k in ks:
        res = [ag.brute_force_knn(store, q, k) for q in queries]
        out[f"ids_k{k}"] = np.array([[n.id for n in r] for r in res], dtype=np.int64)
        out[f"dists_k{k}"] = np.array([[n.dist for n in r] for r in res], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "bf_small.npz"), **out)

    # line store (conftest.py:16-19) cases from test_ann_graph.py:56-79
    line = ag.VectorStore(data=np.array([[0.0], [1.0], [2.0]], dtype=np.float32))
    cases = []
    for q, k in [(0.9, 1), (2.0, 1), (0.4, 3), (1.0, 3), (1.5, 2), (-7.25, 2)]:
        r = ag.brute_force_knn(line, np.array([q]), k)
        cases.append({"q": q, "k": k, "ids": [n.id for n in r], "dists": [n.dist for n in r]})
    with open(os.path.join(HERE, "bf_line.json"), "w") as f:
        json.dump(cases, f)

    # C1 KAT: 100K x 128 seed 1, queries 64 x 128 seed 2, k = 10.
    db = wl.gen_vectors(100_000, 128, seed=1)
    qs = wl.gen_vectors(64, 128, seed=2).data
    res = [ag.brute_force_knn(db, q, 10) for q in qs]
    np.savez_compressed(
        os.path.join(HERE, "bf_c1.npz"),
        ids=np.array([[n.id for n in r] for r in res], dtype=np.int64),
        dists=np.array([[n.dist for n in r] for r in res], dtype=np.float64),
        db_sha=np.array(_sha(db.data)),
        q_sha=np.array(_sha(qs)),
    )


def gen_ivf(ag, wl):
    """IVF golden from reference primitives over a shared artifact."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from oracle.trinity_oracle import kmeans

    db = wl.gen_vectors(20_000, 32, seed=5)
    art = kmeans(db.data, nlist=64, iters=5, seed=6)
    queries = wl.gen_vectors(40, 32, seed=7).data
    ks = np.array([100 if i % 3 == 0 else 10 for i in range(40)], dtype=np.int64)
    nprobes = np.array([16 if i % 3 == 0 else 4 for i in range(40)], dtype=np.int64)
    cstore = ag.VectorStore(data=art.centroids)
    ids_out = np.full((40, 100), -1, dtype=np.int64)
    d_out = np.full((40, 100), np.inf)
    probes_out = np.full((40, 16), -1, dtype=np.int64)
    for i, q in enumerate(queries):
        probes = [n.id for n in ag.brute_force_knn(cstore, q, int(nprobes[i]))]
        probes_out[i, : len(probes)] = probes
        cand = np.sort(np.concatenate([np.nonzero(art.assign == p)[0] for p in probes]))
        dist = ag.rowwise_sq_dists(np.asarray(q, np.float64), db.data64[cand])
        order = np.lexsort((cand, dist))[: ks[i]]
        ids_out[i, : order.size] = cand[order]
        d_out[i, : order.size] = dist[order]
    np.savez_compressed(
        os.path.join(HERE, "ivf_small.npz"),
        centroids=art.centroids, assign=art.assign, ks=ks, nprobes=nprobes,
        probes=probes_out, ids=ids_out, dists=d_out, db_sha=np.array(_sha(db.data)),
    )


def gen_engine(ag, en, wl):
    """Acceptance criterion 1/3 workload (test_acceptance.py:47-81,170-180)."""
    store = wl.gen_vectors(5000, 16, seed=20_240_601)
    graph = ag.build_knn_graph(store, 16)
    queries = wl.gen_vectors(200, 16, seed=20_240_602).data
    cfg = en.EngineConfig(m=64, p=2, entry_count=8, batch_capacity=512)
    eng = en.ContinuousBatchEngine(store, graph, cfg)
    rids = []
    for wave in range(10):
        for q in queries[wave * 20:(wave + 1) * 20]:
            rids.append(eng.submit(q, k=10))
        eng.step()
    eng.run_to_completion()
    res = [eng.result(r) for r in rids]
    st = eng.stats
    np.savez_compressed(
        os.path.join(HERE, "engine_c1.npz"),
        adjacency=graph.adjacency,
        ids=np.array([[n.id for n in r.neighbors] for r in res], dtype=np.int64),
        dists=np.array([[n.dist for n in r.neighbors] for r in res], dtype=np.float64),
        extends=np.array([r.extends for r in res], dtype=np.int64),
        batch_real_counts=np.array(st.batch_real_counts, dtype=np.int64),
        emissions=np.array(st.emissions),
        real_tasks=np.array(st.real_tasks),
        dummy_tasks=np.array(st.dummy_tasks),
    )
    # mixed-owner distance batch (test_engine.py:149-158)
    s2 = wl.gen_vectors(50, 4, seed=3)
    rng = np.random.Generator(np.random.Philox(4))
    qd = {0: rng.standard_normal(4), 1: rng.standard_normal(4)}
    batches = en.build_task_array({0: [5, 9, 11], 1: [2, 5, 40, 41, 42]}, 8)
    r = en.execute_distance_batch(batches[0], s2, qd)
    np.savez_compressed(
        os.path.join(HERE, "mixed_batch.npz"),
        q0=qd[0], q1=qd[1],
        owners=np.array([o for o, _, _ in r]), cands=np.array([c for _, c, _ in r]),
        dists=np.array([x for _, _, x in r]),
    )


def gen_trace_fixture(wl):
    spec = wl.WorkloadSpec(n_db=100, dim=4, n_requests=50, arrival_rate=10.0,
                           prompt_len_dist=wl.LengthDist.uniform(16, 64),
                           output_len_dist=wl.LengthDist.geometric(40.0), delta=32, seed=5)
    tr = wl.gen_trace(spec)
    np.savez_compressed(
        os.path.join(HERE, "trace_small.npz"),
        arrivals=np.array([r.arrival_time for r in tr]),
        prompt=np.array([r.prompt_len for r in tr]),
        output=np.array([r.output_len for r in tr]),
        queries=np.concatenate([r.queries for r in tr]),
        counts=np.array([r.queries.shape[0] for r in tr]),
    )


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference")
    args = ap.parse_args()
    ag, en, wl = _import_reference(args.reference)
    gen_distance_kats(ag)
    gen_bruteforce(ag, wl)
    gen_ivf(ag, wl)
    gen_engine(ag, en, wl)
    gen_trace_fixture(wl)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
