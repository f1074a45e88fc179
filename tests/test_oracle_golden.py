"""Pin the CPU oracle against fixtures produced by the reference itself (CPU only)."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import trinity_oracle as orc
from paper_2512_02281_b200.workload import gen_matrix


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_distance_kats(golden_dir):
    with open(os.path.join(golden_dir, "distance_kats.json")) as f:
        cases = json.load(f)
    for c in cases:
        a = np.array(c["a"], np.float32)
        b = np.array(c["b"], np.float32)
        assert orc.pair_distance(a, b) == c["dist"]  # bit-exact


def test_distance_errors():
    with pytest.raises(ValueError, match="dimension"):
        orc.pair_distance(np.zeros(3), np.zeros(4))
    with pytest.raises(ValueError):
        orc.pair_distance(np.array([np.nan]), np.array([0.0]))


def test_scalar_order_matches_numpy_einsum():
    """The documented summation order (GPU re-rank kernel) equals numpy's einsum bit-for-bit."""
    rng = np.random.Generator(np.random.Philox(99))
    for d in [1, 2, 3, 5, 7, 8, 9, 15, 16, 17, 31, 33, 64, 128, 130, 768]:
        rows = rng.standard_normal((6, d)).astype(np.float32).astype(np.float64)
        q = rng.standard_normal(d)
        ref = orc.sq_dists(q, rows)
        for i in range(rows.shape[0]):
            assert orc.sq_dist_scalar_order(q, rows[i]) == ref[i]


def test_bruteforce_small(golden_dir):
    g = _load(golden_dir, "bf_small.npz")
    data = gen_matrix(1000, 8, 11)
    assert _sha(data) == str(g["db_sha"])
    for k in (10, 1, 37, 1000):
        for i, q in enumerate(g["queries"]):
            ids, d = orc.exact_knn(data, q, k)
            assert np.array_equal(ids, g[f"ids_k{k}"][i])
            assert np.array_equal(d, g[f"dists_k{k}"][i])


def test_bruteforce_line(golden_dir):
    with open(os.path.join(golden_dir, "bf_line.json")) as f:
        cases = json.load(f)
    data = np.array([[0.0], [1.0], [2.0]], np.float32)
    for c in cases:
        ids, d = orc.exact_knn(data, np.array([c["q"]]), c["k"])
        assert ids.tolist() == c["ids"] and d.tolist() == c["dists"]
    with pytest.raises(ValueError):
        orc.exact_knn(data, np.array([0.0]), 4)
    with pytest.raises(ValueError):
        orc.exact_knn(data, np.array([0.0]), 0)


def test_bruteforce_c1_kat(golden_dir):
    g = _load(golden_dir, "bf_c1.npz")
    data = gen_matrix(100_000, 128, 1)
    qs = gen_matrix(64, 128, 2)
    assert _sha(data) == str(g["db_sha"]) and _sha(qs) == str(g["q_sha"])
    assert g["ids"][0].tolist() == [59490, 38487, 35446, 99216, 6554, 22818, 32553, 55596, 62594, 68612]
    for i in range(0, 64, 9):
        ids, d = orc.exact_knn(data, qs[i], 10)
        assert np.array_equal(ids, g["ids"][i]) and np.array_equal(d, g["dists"][i])


def test_ivf_composition(golden_dir):
    g = _load(golden_dir, "ivf_small.npz")
    data = gen_matrix(20_000, 32, 5)
    assert _sha(data) == str(g["db_sha"])
    art = orc.IVFArtifact(g["centroids"], g["assign"])
    qs = gen_matrix(40, 32, 7)
    for i in range(40):
        k, npb = int(g["ks"][i]), int(g["nprobes"][i])
        probes = orc.coarse_probe(art, qs[i], npb)
        assert probes.tolist() == g["probes"][i][:npb].tolist()
        ids, d = orc.ivf_search(data, art, qs[i], k, npb)
        n = ids.size
        assert np.array_equal(ids, g["ids"][i][:n]) and np.array_equal(d, g["dists"][i][:n])
        assert n == min(k, int((g["ids"][i] >= 0).sum()))


def test_ivf_lists_ascending():
    rng = np.random.Generator(np.random.Philox(3))
    assign = rng.integers(0, 7, size=500).astype(np.int32)
    art = orc.IVFArtifact(np.zeros((7, 2), np.float32), assign)
    for lst in range(7):
        m = art.members(lst)
        assert np.all(np.diff(m) > 0) and np.all(assign[m] == lst)
    assert art.offsets[-1] == 500


def test_merge_shards_is_global_topk():
    rng = np.random.Generator(np.random.Philox(8))
    data = rng.standard_normal((3000, 12)).astype(np.float32)
    q = rng.standard_normal(12)
    full_ids, full_d = orc.exact_knn(data, q, 25)
    parts = []
    for lo, hi in [(0, 1000), (1000, 1700), (1700, 3000)]:
        ids, d = orc.exact_knn(data[lo:hi], q, 25)
        parts.append((ids + lo, d))
    ids, d = orc.merge_shards(parts, 25)
    assert np.array_equal(ids, full_ids) and np.array_equal(d, full_d)


def test_gen_trace_matches_reference(golden_dir):
    from paper_2512_02281_b200 import workload as wl

    g = _load(golden_dir, "trace_small.npz")
    spec = wl.WorkloadSpec(n_db=100, dim=4, n_requests=50, arrival_rate=10.0,
                           prompt_len_dist=wl.LengthDist.uniform(16, 64),
                           output_len_dist=wl.LengthDist.geometric(40.0), delta=32, seed=5)
    tr = wl.gen_trace(spec)
    assert np.array_equal([r.arrival_time for r in tr], g["arrivals"])
    assert np.array_equal([r.prompt_len for r in tr], g["prompt"])
    assert np.array_equal([r.output_len for r in tr], g["output"])
    assert np.array_equal(np.concatenate([r.queries for r in tr]), g["queries"])
    assert [r.queries.shape[0] for r in tr] == g["counts"].tolist()


def test_engine_oracle_matches_reference_run(golden_dir):
    """The engine restatement reproduces the reference's acceptance run
    (test_acceptance.py:47-81; pkg/test_output.txt:16: 144 batches, 62736 tasks)."""
    from paper_2512_02281_b200.workload import gen_matrix

    g = np.load(os.path.join(golden_dir, "engine_c1.npz"))
    data = gen_matrix(5000, 16, 20_240_601)
    queries = gen_matrix(200, 16, 20_240_602)
    ids, d, ext, brc, _ = orc.engine_run(data, g["adjacency"], queries, np.full(200, 10),
                                         np.repeat(np.arange(10), 20))
    assert all(np.array_equal(ids[i], g["ids"][i]) for i in range(200))
    assert all(np.array_equal(d[i], g["dists"][i]) for i in range(200))
    assert np.array_equal(ext, g["extends"])
    assert brc == g["batch_real_counts"].tolist()
    assert len(brc) == 144 and sum(brc) == 62736
