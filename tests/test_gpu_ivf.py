"""IVF-Flat on the GPU vs the reference-primitive golden vectors and the oracle."""

import os

import numpy as np
import pytest

from oracle import trinity_oracle as orc
from paper_2512_02281_b200 import _lib
from paper_2512_02281_b200.ann_graph import VectorStore
from paper_2512_02281_b200.ivf import IVFFlatIndex
from paper_2512_02281_b200.workload import gen_matrix, gen_vectors_chunked

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["auto", "simt", "tf32", "nodense"], autouse=True)
def scan_kernel(request):
    """Run every test on each candidate-generation path: auto (dense small-store
    brute force + tcgen05 fp16 list scan), fp32 SIMT scan only, the TF32
    tensor-core scan, and scan-only (no dense)."""
    _lib.set_option("scan_kernel", {"simt": 1, "tf32": 2}.get(request.param, 0))
    _lib.set_option("dense_off", 1 if request.param != "auto" else 0)
    yield request.param
    _lib.set_option("scan_kernel", 0)
    _lib.set_option("dense_off", 0)
    _lib.set_option("force_fixup", 0)


@pytest.fixture(scope="module")
def small(golden_dir):
    g = np.load(os.path.join(golden_dir, "ivf_small.npz"))
    data = gen_matrix(20_000, 32, 5)
    store = VectorStore(data=data)
    idx = IVFFlatIndex.from_artifact(store, g["centroids"], g["assign"])
    return g, data, idx


def _check_rows(ids, d, g, ks):
    for i in range(ids.shape[0]):
        n = int((g["ids"][i] >= 0).sum())
        k = int(ks[i])
        m = min(k, n)
        assert np.array_equal(ids[i, :m], g["ids"][i, :m]), i
        assert np.array_equal(d[i, :m], g["dists"][i, :m]), i
        assert (ids[i, m:k] == -1).all()


def test_ivf_golden_ragged(small):
    g, data, idx = small
    qs = gen_matrix(40, 32, 7)
    ids, d = idx.search(qs, g["ks"], g["nprobes"])
    _check_rows(ids, d, g, g["ks"])
    probes = idx.last_probes(40, 16)
    for i in range(40):  # the top-nprobe SET (coarse_set: approximate order)
        npb = int(g["nprobes"][i])
        assert sorted(probes[i, :npb].tolist()) == sorted(g["probes"][i, :npb].tolist())
    _lib.set_option("coarse_set", 0)  # the full re-rank: exact (dist, id) order
    try:
        ids0, d0 = idx.search(qs, g["ks"], g["nprobes"])
        probes = idx.last_probes(40, 16)
    finally:
        _lib.set_option("coarse_set", 1)
    assert np.array_equal(ids0, ids) and np.array_equal(d0, d)
    for i in range(40):
        npb = int(g["nprobes"][i])
        assert probes[i, :npb].tolist() == g["probes"][i, :npb].tolist()


def test_ivf_forced_fixup(small):
    g, data, idx = small
    qs = gen_matrix(40, 32, 7)
    _lib.set_option("force_fixup", 1)
    ids, d = idx.search(qs, g["ks"], g["nprobes"])
    assert idx.last_fixups() > 0
    _check_rows(ids, d, g, g["ks"])


def test_ivf_export_roundtrip(small):
    g, data, idx = small
    cen, asg = idx.export()
    assert np.array_equal(cen, g["centroids"]) and np.array_equal(asg, g["assign"])
    sizes = idx.list_sizes()
    assert np.array_equal(sizes, np.bincount(g["assign"], minlength=64))


def test_ivf_single_and_full_probe(small):
    g, data, idx = small
    art = orc.IVFArtifact(g["centroids"], g["assign"])
    qs = gen_matrix(5, 32, 99)
    for npb in (1, 64):
        ids, d = idx.search(qs, 10, npb)
        for i in range(5):
            oi, od = orc.ivf_search(data, art, qs[i], 10, npb)
            assert np.array_equal(ids[i], oi) and np.array_equal(d[i], od)
    # nprobe = nlist is exact brute force
    bi, bd = orc.exact_knn(data, qs[0], 10)
    ids, d = idx.search(qs[:1], 10, 64)
    assert np.array_equal(ids[0], bi) and np.array_equal(d[0], bd)


def test_ivf_trained_index_parity_and_balance():
    data = gen_matrix(30_000, 48, 11)
    store = VectorStore(data=data)
    idx = IVFFlatIndex.train(store, nlist=100, iters=5, seed=3)
    cen, asg = idx.export()
    sizes = np.bincount(asg, minlength=100)
    assert sizes.sum() == 30_000 and sizes.max() < 5 * 300
    # assignment is the exact nearest centroid (ties to the smaller id)
    assert np.array_equal(asg, orc.nearest_centroid(data, cen))
    art = orc.IVFArtifact(cen, asg)
    qs = gen_matrix(24, 48, 12)
    ks = np.array([10, 100, 10] * 8)
    nps = np.array([8, 32, 4] * 8)
    ids, d = idx.search(qs, ks, nps)
    for i in range(24):
        oi, od = orc.ivf_search(data, art, qs[i], int(ks[i]), int(nps[i]))
        assert np.array_equal(ids[i, : oi.size], oi) and np.array_equal(d[i, : oi.size], od)


def test_ivf_empty_lists_and_tiny_lists():
    rng = np.random.Generator(np.random.Philox(5))
    data = rng.standard_normal((300, 8)).astype(np.float32)
    cen = rng.standard_normal((20, 8)).astype(np.float32)
    asg = rng.integers(0, 5, size=300).astype(np.int32)  # lists 5..19 empty
    store = VectorStore(data=data)
    idx = IVFFlatIndex.from_artifact(store, cen, asg)
    art = orc.IVFArtifact(cen, asg)
    qs = rng.standard_normal((10, 8))
    ids, d = idx.search(qs, 50, 3)
    for i in range(10):
        oi, od = orc.ivf_search(data, art, qs[i], 50, 3)
        n = oi.size
        assert np.array_equal(ids[i, :n], oi) and np.array_equal(d[i, :n], od)
        assert (ids[i, n:] == -1).all()


def test_ivf_id_offset_shard():
    rng = np.random.Generator(np.random.Philox(6))
    data = rng.standard_normal((2000, 16)).astype(np.float32)
    art = orc.kmeans(data, 16, 3, 1)
    store = VectorStore(data=data[1000:])
    idx = IVFFlatIndex.from_artifact(store, art.centroids, art.assign[1000:], id_offset=1000)
    q = rng.standard_normal((3, 16))
    ids, d = idx.search(q, 5, 16)
    for i in range(3):
        oi, od = orc.exact_knn(data[1000:], q[i], 5)
        assert np.array_equal(ids[i], oi + 1000) and np.array_equal(d[i], od)


@pytest.mark.slow
def test_c2_scale_parity():
    """BASELINE C2 (1M x 768, nlist 1024, nprobe 32, B 256, k 10): the GPU-trained
    artifact equals the oracle's k-means bit-for-bit, and ALL 256 queries equal
    the oracle (process pool over the host cores)."""
    from oracle.pool import assert_rows_equal, ivf_oracle_batch

    data = gen_vectors_chunked(1_000_000, 768, seed=3)
    store = VectorStore(data=data)
    idx = IVFFlatIndex.train(store, nlist=1024, iters=5, seed=4)
    qs = gen_matrix(256, 768, 4)
    ids, d = idx.search(qs, 10, 32)
    assert idx.last_fixups() == 0
    cen, asg = idx.export()
    art = orc.IVFArtifact(cen, asg)
    assert_rows_equal(ids, d, ivf_oracle_batch(data, art, qs.astype(np.float64), 10, 32))
    # the exact nearest-centroid step of training, checked on a row sample
    # (the full 1M-row oracle k-means runs in test_kmeans_c2_matches_oracle)
    rows = np.arange(0, 1_000_000, 997)
    assert np.array_equal(asg[rows], orc.nearest_centroid(data[rows], cen))
    # rows are sorted by (dist, id)
    for i in range(256):
        assert np.array_equal(np.lexsort((ids[i], d[i])), np.arange(10))


@pytest.mark.slow
def test_kmeans_c2_matches_oracle(scan_kernel):
    """GPU Lloyd k-means (exact assignment, float64 ascending-id sums) at the C2
    size equals the CPU restatement oracle.kmeans bit-for-bit: the artifact both
    bench arms build is one and the same."""
    if scan_kernel != "auto":
        pytest.skip("training does not depend on the scan options")
    data = gen_vectors_chunked(1_000_000, 768, seed=3)
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=1024, iters=5, seed=4)
    cen, asg = idx.export()
    art = orc.kmeans(data, 1024, 5, 4)
    assert np.array_equal(cen, art.centroids) and np.array_equal(asg, art.assign)


@pytest.mark.parametrize("n,d,nlist,iters", [(20_000, 32, 64, 5), (6_000, 768, 48, 3), (5_000, 7, 100, 4)])
def test_kmeans_matches_oracle(n, d, nlist, iters, scan_kernel):
    """Training and tri_kmeans_assign are bit-identical to the oracle restatement."""
    if scan_kernel == "tf32":
        pytest.skip("training does not use the list scan")
    data = gen_matrix(n, d, 300 + d)
    store = VectorStore(data=data)
    idx = IVFFlatIndex.train(store, nlist=nlist, iters=iters, seed=9)
    cen, asg = idx.export()
    art = orc.kmeans(data, nlist, iters, 9)
    assert np.array_equal(cen, art.centroids)
    assert np.array_equal(asg, art.assign)
    # nearest-centroid assignment of other centroids (a near-tie-heavy case: the
    # centroids of a shifted copy sit close together)
    cen2 = (art.centroids + np.float32(1e-3)).astype(np.float32)
    assert np.array_equal(IVFFlatIndex.assign(store, cen2), orc.nearest_centroid(data, cen2))


def test_ivf_concurrent_lanes(small):
    """Batches in flight on several streams (one library workspace per stream)
    and host threads driving one stream each give the single-stream results."""
    import threading

    import torch

    g, data, idx = small
    g = {key: g[key] for key in g.files}  # NpzFile reads lazily and is not thread-safe
    qs = gen_matrix(40, 32, 7).astype(np.float64)  # device / host-buffer APIs take float64 queries
    ks, nps = g["ks"], g["nprobes"]
    streams = [torch.cuda.Stream() for _ in range(5)]  # > the 4 lanes: forces lane recycling
    q_dev = torch.from_numpy(qs).cuda()
    outs = [(torch.empty((40, 100), dtype=torch.int64, device="cuda"),
             torch.empty((40, 100), dtype=torch.float64, device="cuda")) for _ in streams]
    torch.cuda.synchronize()
    for rep in range(3):
        for st, (oi, od) in zip(streams, outs):
            idx.search_device(q_dev, ks, nps, oi, od, st)
    torch.cuda.synchronize()
    for oi, od in outs:
        _check_rows(oi.cpu().numpy(), od.cpu().numpy(), g, ks)

    errs = []

    def worker(j):
        try:
            ids = np.empty((40, 100), np.int64)
            d = np.empty((40, 100), np.float64)
            for _ in range(4):
                idx.search_into(qs, ks, nps, ids, d, stream=streams[j])
                _check_rows(ids, d, g, ks)
        except Exception as e:  # surfaced below
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(j,)) for j in range(3)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errs, errs


@pytest.mark.parametrize("scale", [2.0 ** 25, 2.0 ** -25, 1.0])
def test_ivf_scaled_data_and_extreme_queries(scale):
    """fp16 candidate copy is power-of-two scaled: large / tiny data stay exact;
    queries the fp16 scan cannot scale (max element > 2^60), overflowing
    approximate distances and all-zero queries are answered exactly too."""
    base = gen_matrix(6000, 40, 61)
    data = (base.astype(np.float64) * scale).astype(np.float32)
    art = orc.kmeans(data, 24, 3, 6)
    idx = IVFFlatIndex.from_artifact(VectorStore(data=data), art.centroids, art.assign)
    qs = gen_matrix(12, 40, 62).astype(np.float64) * scale
    qs[3] *= 2.0 ** 70
    qs[5] = 0.0
    qs[7] *= 2.0 ** -80
    k, npb = 9, 5
    ids, d = idx.search(qs, k, npb)
    for i, q in enumerate(qs):
        oi, od = orc.ivf_search(data, art, q, k, npb)
        assert np.array_equal(ids[i, : oi.size], oi), i
        assert np.array_equal(d[i, : od.size], od), i


def test_ivf_graph_replay_tracks_inputs(small):
    """Repeated shapes run eagerly, then captured, then replayed as CUDA graphs:
    every call must see the CURRENT query contents (device and pinned-host
    paths), and a new shape or a scratch reallocation must not replay a stale
    graph."""
    import torch

    g, data, idx = small
    art = orc.IVFArtifact(g["centroids"], g["assign"])
    ks = np.array([10, 100] * 8)
    nps = np.array([4, 16] * 8)
    q_dev = torch.empty((16, 32), dtype=torch.float64, device="cuda")
    ids_dev = torch.empty((16, 100), dtype=torch.int64, device="cuda")
    d_dev = torch.empty((16, 100), dtype=torch.float64, device="cuda")
    q_pin = torch.empty((16, 32), dtype=torch.float64).pin_memory()
    ids_pin = torch.empty((16, 100), dtype=torch.int64).pin_memory()
    d_pin = torch.empty((16, 100), dtype=torch.float64).pin_memory()
    st = torch.cuda.Stream()
    for rep in range(5):
        qs = gen_matrix(16, 32, 100 + rep).astype(np.float64)
        q_dev.copy_(torch.from_numpy(qs))
        q_pin.copy_(torch.from_numpy(qs))
        torch.cuda.synchronize()
        idx.search_device(q_dev, ks, nps, ids_dev, d_dev, st)
        st.synchronize()
        idx.search_into(q_pin, ks, nps, ids_pin, d_pin, stream=st)
        for out_ids, out_d in ((ids_dev.cpu().numpy(), d_dev.cpu().numpy()), (ids_pin.numpy(), d_pin.numpy())):
            for i in range(16):
                oi, od = orc.ivf_search(data, art, qs[i], int(ks[i]), int(nps[i]))
                assert np.array_equal(out_ids[i, :oi.size], oi), (rep, i)
                assert np.array_equal(out_d[i, :oi.size], od), (rep, i)
        if rep == 2:  # a different, larger shape on the same lane reallocates scratch
            big = gen_matrix(64, 32, 9).astype(np.float64)
            bi, bd = idx.search(big, 100, 32)
            oi, od = orc.ivf_search(data, art, big[5], 100, 32)
            assert np.array_equal(bi[5, :oi.size], oi)


def test_c3_scale_ragged_parity(scan_kernel):
    """BASELINE C3 at full scale: prefill (k=100, nprobe=64) and decode (k=10,
    nprobe=16) retrievals in ONE ragged batch over the C2 index; exercises the
    cross-item threshold and the fp16 over-fetch at k=100.  Every one of the 256
    rows equals the oracle (process pool)."""
    if scan_kernel != "auto":
        pytest.skip("full-scale ragged case runs on the default path only")
    data = gen_vectors_chunked(1_000_000, 768, seed=3)
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=1024, iters=5, seed=4)
    qs = gen_matrix(256, 768, 77)
    pre = np.arange(256) % 3 == 0
    ks = np.where(pre, 100, 10)
    nps = np.where(pre, 64, 16)
    ids, d = idx.search(qs, ks, nps)
    cen, asg = idx.export()
    art = orc.IVFArtifact(cen, asg)
    from oracle.pool import assert_rows_equal, ivf_oracle_batch

    assert_rows_equal(ids, d, ivf_oracle_batch(data, art, qs.astype(np.float64), ks, nps), ks)


def test_ivf_save_load_same_results(small, tmp_path):
    g, data, idx = small
    path = str(tmp_path / "small.ivf")
    idx.save(path)
    idx2 = IVFFlatIndex.load(VectorStore(data=data), path)
    qs = gen_matrix(40, 32, 7)
    a = idx.search(qs, g["ks"], g["nprobes"])
    b = idx2.search(qs, g["ks"], g["nprobes"])
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("d", [3, 33, 130, 1100])
def test_ivf_odd_and_wide_dims(d, scan_kernel):
    """Row widths off the fast paths: odd d (scalar exact distances), d not a
    multiple of 16 or 64 (padding), d > 1024 (no tensor-core scan / split
    coarse copies: SIMT paths)."""
    if scan_kernel not in ("auto", "simt"):
        pytest.skip("one accelerated and one SIMT configuration are enough here")
    n = 6000
    data = gen_matrix(n, d, 900 + d)
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=48, iters=3, seed=2)
    cen, asg = idx.export()
    art = orc.IVFArtifact(cen, asg)
    qs = gen_matrix(20, d, 901 + d)
    ks = np.array([1, 10, 50, 7] * 5)
    nps = np.array([1, 4, 12, 48] * 5)
    ids, dist = idx.search(qs, ks, nps)
    for i in range(20):
        oi, od = orc.ivf_search(data, art, qs[i], int(ks[i]), int(nps[i]))
        assert np.array_equal(ids[i, :oi.size], oi), (d, i)
        assert np.array_equal(dist[i, :oi.size], od), (d, i)


def test_ivf_duplicate_rows_tie_break(scan_kernel):
    """Every vector stored four times: equal float64 distances everywhere, so the
    order is decided by the (dist, id) tie rule alone (ann_graph.py:136) and the
    certificate's strict inequality must route boundary ties to the exact path."""
    base = gen_matrix(1500, 24, 31)
    data = np.concatenate([base, base, base, base])  # ids i, i+1500, i+3000, i+4500 identical
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=32, iters=3, seed=3)
    cen, asg = idx.export()
    art = orc.IVFArtifact(cen, asg)
    qs = np.concatenate([gen_matrix(12, 24, 32), base[:4].astype(np.float64)])  # the last 4 hit exact copies
    ks = np.array([10, 3, 40, 9] * 4)
    nps = np.array([4, 32, 8, 1] * 4)
    ids, dist = idx.search(qs, ks, nps)
    for i in range(qs.shape[0]):
        oi, od = orc.ivf_search(data, art, qs[i], int(ks[i]), int(nps[i]))
        assert np.array_equal(ids[i, :oi.size], oi), i
        assert np.array_equal(dist[i, :oi.size], od), i


_SCAN_OPTS = [
    {"scan_abufs": 2},
    {"scan_l2hint": 0},
    {"scan_l2hint": 2},
    {"scan_reserve": 16},
    {"scan_reserve": 0},
    {"scan_qbufs": 1, "tc_stages": 4},
    {"pack_mixed": 0},
    {"scan_pool": 0},
    {"scan_pool_pub": 1},
    {"rerank_wide_slab": 0, "rerank_lpt": 0},
    {"rerank_split": 0},
    {"merge_split": 0},
    {"dense_fold": 0},
]
_SCAN_DEFAULTS = {"scan_abufs": 1, "scan_l2hint": 1, "scan_reserve": -1, "scan_qbufs": 2, "tc_stages": 0,
                  "pack_mixed": 1, "scan_pool": 1024, "scan_pool_pub": 2, "rerank_wide_slab": 80, "rerank_lpt": 1,
                  "rerank_split": 1, "merge_split": 1, "dense_fold": 1}


@pytest.mark.parametrize("opts", _SCAN_OPTS, ids=lambda o: ",".join(f"{k}={v}" for k, v in o.items()))
def test_ivf_scan_options_parity(small, opts):
    """Scan tuning options (append buffers, L2 policy, reserved SMs, ring depth,
    per-class instead of mixed-k list groups) change scheduling only: results stay equal to the golden vectors, also with
    batches on several streams (the automatic SM reservation)."""
    import torch

    g, data, idx = small
    qs = gen_matrix(40, 32, 7)
    try:
        for k, v in opts.items():
            _lib.set_option(k, v)
        streams = [torch.cuda.Stream() for _ in range(3)]
        for st in streams:
            ids = np.full((40, int(g["ks"].max())), -1, np.int64)
            d = np.full(ids.shape, np.inf)
            idx.search_into(qs.astype(np.float64), g["ks"], g["nprobes"], ids, d, stream=st)
            _check_rows(ids, d, g, g["ks"])
    finally:
        for k, v in _SCAN_DEFAULTS.items():
            _lib.set_option(k, v)


@pytest.mark.parametrize("pool", [(1024, 2), (1024, 1), (64, 2), (0, 2)])
def test_pooled_bound_wide_members(pool, scan_kernel):
    """kp >= 128 members (k = 100 -> kp 256) tighten their cross-item bound
    from a pool of finished items' (and first chunks') best keys; the bound
    only prunes, so results equal the oracle with the pool on, off, one
    publish per item, or too small to ever reach kp keys.  Rows are stored
    twice (equal distances, distinct ids) so the pool's distinct-row count is
    exercised on exact ties."""
    base = gen_matrix(6000, 32, 41)
    data = np.concatenate([base, base])
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=48, iters=3, seed=5)
    cen, asg = idx.export()
    art = orc.IVFArtifact(cen, asg)
    qs = np.concatenate([gen_matrix(20, 32, 42), base[:4].astype(np.float64)])
    ks = np.array([100, 10, 150, 100, 30, 100] * 4)
    nps = np.array([24, 8, 48, 12, 16, 6] * 4)
    try:
        _lib.set_option("scan_pool", pool[0])
        _lib.set_option("scan_pool_pub", pool[1])
        for _ in range(3):  # eager, captured, replayed
            ids, dist = idx.search(qs, ks, nps)
    finally:
        _lib.set_option("scan_pool", 1024)
        _lib.set_option("scan_pool_pub", 2)
    for i in range(qs.shape[0]):
        oi, od = orc.ivf_search(data, art, qs[i], int(ks[i]), int(nps[i]))
        assert np.array_equal(ids[i, : oi.size], oi), i
        assert np.array_equal(dist[i, : oi.size], od), i


def test_device_path_non_finite_query_rows(small):
    """search_device skips the host finiteness check: a NaN / inf query row comes
    back as id -1 / NaN (never garbage) and leaves the other rows exact."""
    import torch

    g, data, idx = small
    qs = gen_matrix(40, 32, 7).astype(np.float64)
    qs[3, 5] = np.nan
    qs[17, 0] = np.inf
    q = torch.from_numpy(qs).cuda()
    kmax = int(g["ks"].max())
    ids = torch.empty((40, kmax), dtype=torch.int64, device="cuda")
    d = torch.empty((40, kmax), dtype=torch.float64, device="cuda")
    idx.search_device(q, g["ks"], g["nprobes"], ids, d)
    torch.cuda.synchronize()
    hi, hd = ids.cpu().numpy(), d.cpu().numpy()
    for i in (3, 17):
        k = int(g["ks"][i])
        assert (hi[i, :k] == -1).all() and np.isnan(hd[i, :k]).all()
    keep = [i for i in range(40) if i not in (3, 17)]
    _check_rows(hi[keep], hd[keep], {"ids": g["ids"][keep], "dists": g["dists"][keep]}, g["ks"][keep])
    with pytest.raises(ValueError):  # the host entry point rejects it up front
        idx.search(qs, g["ks"], g["nprobes"])


@pytest.mark.gpu
def test_coarse_set_semantics_on_tied_centroids():
    """Duplicated centroids tie exactly: the coarse step's top-nprobe set must
    still be the reference's (dist, id) prefix (nprobe splits tie pairs)."""
    rng = np.random.Generator(np.random.Philox(23))
    data = rng.standard_normal((4000, 16)).astype(np.float32)
    cen = rng.standard_normal((32, 16)).astype(np.float32)
    cen[16:] = cen[:16]  # exact duplicates: ids 16..31 tie with 0..15
    idx = IVFFlatIndex.from_centroids(VectorStore(data=data), cen)
    art = orc.IVFArtifact(cen, idx.export()[1])
    qs = rng.standard_normal((24, 16))
    for npb in (1, 5, 17):
        ids, d = idx.search(qs, 10, npb)
        probes = idx.last_probes(24, npb)
        for i in range(24):
            assert sorted(probes[i].tolist()) == sorted(orc.coarse_probe(art, qs[i], npb).tolist())
            oi, od = orc.ivf_search(data, art, qs[i], 10, npb)
            assert np.array_equal(ids[i, :oi.size], oi) and np.array_equal(d[i, :od.size], od)


@pytest.mark.gpu
def test_native_comm_sharded_search_world_one():
    """tri_comm_init / tri_ivf_search_sharded with a one-rank NCCL communicator:
    local search -> packed all-gather -> device merge equals the plain search."""
    import torch

    from paper_2512_02281_b200.sharded import ShardedIVF

    data = gen_matrix(20_000, 32, 41)
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=64, iters=3, seed=2)
    qs = torch.from_numpy(gen_matrix(40, 32, 42).astype(np.float64)).cuda()
    st = torch.cuda.Stream()
    ref_i = torch.empty((40, 10), dtype=torch.int64, device="cuda")
    ref_d = torch.empty((40, 10), dtype=torch.float64, device="cuda")
    idx.search_device(qs, 10, 8, ref_i, ref_d, st)
    sh = ShardedIVF(idx, 10, transport="native")
    try:
        for _ in range(3):  # the second call captures a graph, the third replays it
            out_i = torch.full((40, 12), 7, dtype=torch.int64, device="cuda")
            out_d = torch.zeros((40, 12), dtype=torch.float64, device="cuda")
            sh.search_device(qs, 8, out_i, out_d, st)
            st.synchronize()
            assert torch.equal(out_i[:, :10], ref_i) and torch.equal(out_d[:, :10], ref_d)
            assert (out_i[:, 10:] == -1).all()
    finally:
        sh.close()
    with pytest.raises(ValueError):
        ShardedIVF(idx, 10, transport="mpi")


@pytest.mark.slow
@pytest.mark.gpu
def test_c4_scale_parity(scan_kernel):
    """BASELINE C4 (10M x 768): the whole database on one GPU and one rank's
    share at G = 8 (rows [3.75M, 5M), global ids through id_offset), both
    built like bench.py's C4 (centroids trained on rows [0, 1M), every row
    listed under its exact nearest centroid); 64 queries of each compared with
    the oracle over the same rows."""
    if scan_kernel != "auto":
        pytest.skip("one scan arithmetic is enough at this size")
    from oracle.pool import assert_rows_equal, ivf_oracle_batch
    from paper_2512_02281_b200.ann_graph import _DeviceStore
    from paper_2512_02281_b200.sharded import shard_bounds
    from paper_2512_02281_b200.workload import gen_rows_chunked

    n, seed = 10_000_000, 100
    tr = _DeviceStore(gen_rows_chunked(0, 1_000_000, 768, seed))
    cen, _ = IVFFlatIndex.train(tr, nlist=1024, iters=5, seed=4).export()
    tr.close()
    qs = gen_matrix(256, 768, 4).astype(np.float64)[::4]
    for lo, hi in [(0, n), shard_bounds(n, 8, 3)]:
        data = gen_rows_chunked(lo, hi, 768, seed)
        store = _DeviceStore(data)
        idx = IVFFlatIndex.from_centroids(store, cen, id_offset=lo)
        store.close()
        ids, d = idx.search(qs, 10, 32)
        art = orc.IVFArtifact(cen, idx.export()[1])
        ref = [(i + lo, dd) for i, dd in ivf_oracle_batch(data, art, qs, 10, 32)]
        assert_rows_equal(ids, d, ref)
        idx.close()
        del data
