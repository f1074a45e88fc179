"""Fixed-shape padded batches: ragged prefill/decode mixes and odd batch sizes
replay a few captured graphs keyed by (bucket(B), max k, max nprobe) -- the
paper's fixed-shape step -- and return exactly what the
exact-shape path and the oracle return."""

import numpy as np
import pytest
import torch

from oracle import trinity_oracle as orc
from paper_2512_02281_b200 import _lib
from paper_2512_02281_b200.ann_graph import VectorStore, brute_force_knn_batch
from paper_2512_02281_b200.ivf import IVFFlatIndex
from paper_2512_02281_b200.workload import gen_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def index():
    data = gen_matrix(30_000, 48, 5)
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=64, iters=3, seed=2)
    cen, asg = idx.export()
    return data, idx, orc.IVFArtifact(cen, asg)


def _mix(rng, B):
    pre = rng.random(B) < 0.35
    return np.where(pre, 100, 10).astype(np.int32), np.where(pre, 64, 16).astype(np.int32)


def _exact_path(fn):
    _lib.set_option("ragged_graphs", 0)
    try:
        return fn()
    finally:
        _lib.set_option("ragged_graphs", 1)


def test_padded_ivf_equals_exact_path_and_oracle(index):
    data, idx, art = index
    rng = np.random.default_rng(3)
    for B in (1, 3, 16, 17, 100, 200, 256, 300):
        q = rng.standard_normal((B, 48))
        ks, nps = _mix(rng, B)
        got_i, got_d = idx.search(q, ks, nps)  # pageable numpy: padded graph path
        ref_i, ref_d = _exact_path(lambda: idx.search(q, ks, nps))
        assert np.array_equal(got_i, ref_i) and np.array_equal(got_d, ref_d), f"B={B}"
        for i in range(0, B, max(1, B // 5)):
            oi, od = orc.ivf_search(data, art, q[i], int(ks[i]), int(nps[i]))
            assert np.array_equal(got_i[i, :oi.size], oi) and np.array_equal(got_d[i, :od.size], od)


def test_padded_replays_track_new_mixes(index):
    """Within one bucket every call after the capture is a replay, and each
    replay answers its own queries, k and nprobe (device and pinned-host API)."""
    data, idx, art = index
    rng = np.random.default_rng(4)
    st = torch.cuda.Stream()
    q_dev = torch.empty((32, 48), dtype=torch.float64, device="cuda")
    ids = torch.empty((32, 100), dtype=torch.int64, device="cuda")
    d = torch.empty((32, 100), dtype=torch.float64, device="cuda")
    qp = torch.empty((32, 48), dtype=torch.float64).pin_memory()
    ip = torch.empty((32, 100), dtype=torch.int64).pin_memory()
    dp = torch.empty((32, 100), dtype=torch.float64).pin_memory()
    c0 = _lib.graph_counters()
    n = 12
    for t in range(n):
        B = int(rng.integers(17, 33))  # bucket 32
        q = rng.standard_normal((B, 48))
        ks, nps = _mix(rng, B)
        ks[0], nps[0] = 100, 64  # same profile (max k, max nprobe) every call
        q_dev[:B].copy_(torch.from_numpy(q))
        idx.search_device(q_dev[:B], ks, nps, ids[:B], d[:B], st)
        qp[:B].copy_(torch.from_numpy(q))
        idx.search_into(qp[:B], ks, nps, ip[:B], dp[:B], stream=st)
        st.synchronize()
        ref_i, ref_d = _exact_path(lambda: idx.search(q, ks, nps))
        for gi, gd in ((ids[:B].cpu().numpy(), d[:B].cpu().numpy()), (ip[:B].numpy(), dp[:B].numpy())):
            for i in range(B):
                kk = int(ks[i])
                assert np.array_equal(gi[i, :kk], ref_i[i, :kk]) and np.array_equal(gi[i, :kk], ref_i[i, :kk])
                assert np.array_equal(gd[i, :kk], ref_d[i, :kk])
    c1 = _lib.graph_counters()
    # two padded shapes (device, host) x (eager, capture) at most outside the replays
    assert c1["replayed"] - c0["replayed"] >= 2 * n - 4


def test_padded_bruteforce(index):
    data = gen_matrix(5_000, 40, 9)
    store = VectorStore(data=data)
    rng = np.random.default_rng(5)
    for B in (3, 50, 100, 50):
        q = rng.standard_normal((B, 40))
        gi, gd = brute_force_knn_batch(store, q, 5)
        ri, rd = _exact_path(lambda: brute_force_knn_batch(store, q, 5))
        assert np.array_equal(gi, ri) and np.array_equal(gd, rd)
        for i in range(0, B, 7):
            oi, od = orc.exact_knn(data, q[i], 5)
            assert np.array_equal(gi[i], oi) and np.array_equal(gd[i], od)
