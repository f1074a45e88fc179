"""Concurrency stress: host threads, each driving its own CUDA stream, mix
ragged IVF batches (random size, per-query k / nprobe: padded fixed-shape
graphs, pooled wide-member bounds) and brute-force batches (dense and
tensor-core paths) on shared handles.  Every result row is checked against
the CPU oracle, so a workspace, graph-cache or plan race shows up as a
mismatch."""

import threading

import numpy as np
import pytest

from oracle import trinity_oracle as orc
from paper_2512_02281_b200.ann_graph import VectorStore
from paper_2512_02281_b200.ivf import IVFFlatIndex
from paper_2512_02281_b200.workload import gen_matrix

pytestmark = pytest.mark.gpu


def test_mixed_apis_many_streams():
    import torch

    rng0 = np.random.Generator(np.random.Philox(123))
    data = gen_matrix(12_000, 48, 11)
    store = VectorStore(data=data)
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=40, iters=3, seed=2)
    art = orc.IVFArtifact(*idx.export())
    small = gen_matrix(3_000, 48, 12)  # dense small-store brute force
    sstore = VectorStore(data=small)
    dev = store.device()
    sdev = sstore.device()
    streams = [torch.cuda.Stream() for _ in range(4)]
    seeds = rng0.integers(0, 2**31, size=4)
    errs = []

    def worker(j):
        try:
            rng = np.random.Generator(np.random.Philox(int(seeds[j])))
            for it in range(25):
                B = int(rng.integers(1, 70))
                qs = rng.standard_normal((B, 48))
                kind = (it + j) % 3
                if kind == 0:  # ragged IVF
                    ks = rng.choice([1, 10, 100, 150], size=B).astype(np.int32)
                    nps = rng.integers(1, 41, size=B).astype(np.int32)
                    ids = np.full((B, 150), -7, np.int64)
                    d = np.full((B, 150), np.nan)
                    idx.search_into(qs, ks, nps, ids, d, stream=streams[j])
                    for i in rng.choice(B, size=min(B, 4), replace=False):
                        oi, od = orc.ivf_search(data, art, qs[i], int(ks[i]), int(nps[i]))
                        assert np.array_equal(ids[i, : oi.size], oi), ("ivf", j, it, i)
                        assert np.array_equal(d[i, : od.size], od), ("ivf", j, it, i)
                else:  # brute force: tensor-core store or dense small store
                    X, h = (data, dev) if kind == 1 else (small, sdev)
                    ks = rng.choice([1, 10, 64, 200], size=B).astype(np.int32)
                    ids = np.full((B, 200), -7, np.int64)
                    d = np.full((B, 200), np.nan)
                    h.knn_into(qs, ks, ids, d, stream=streams[j])
                    for i in rng.choice(B, size=min(B, 4), replace=False):
                        oi, od = orc.exact_knn(X, qs[i], int(ks[i]))
                        assert np.array_equal(ids[i, : oi.size], oi), ("bf", kind, j, it, i)
                        assert np.array_equal(d[i, : od.size], od), ("bf", kind, j, it, i)
        except Exception as e:  # surfaced below
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(j,)) for j in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errs, errs[:3]
