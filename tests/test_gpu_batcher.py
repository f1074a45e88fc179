"""Continuous batching of heterogeneous retrievals (C3) and sharded search (C4) on one GPU."""

import os

import numpy as np
import pytest
import torch

from oracle import trinity_oracle as orc
from paper_2512_02281_b200.ann_graph import VectorStore
from paper_2512_02281_b200.batcher import RetrievalBatcher
from paper_2512_02281_b200.ivf import IVFFlatIndex
from paper_2512_02281_b200.sharded import device_merge, pad_results, shard_bounds
from paper_2512_02281_b200.workload import gen_matrix

pytestmark = pytest.mark.gpu


def test_batcher_matches_reference_primitives(golden_dir):
    g = np.load(os.path.join(golden_dir, "ivf_small.npz"))
    store = VectorStore(data=gen_matrix(20_000, 32, 5))
    idx = IVFFlatIndex.from_artifact(store, g["centroids"], g["assign"])
    b = RetrievalBatcher(idx, max_batch=16)  # several steps, mixed stages per step
    qs = gen_matrix(40, 32, 7)
    rids = [b.submit(qs[i], k=int(g["ks"][i]), nprobe=int(g["nprobes"][i]),
                     stage="prefill" if g["ks"][i] == 100 else "decode") for i in range(40)]
    out = {r.request_id: r for r in b.run_to_completion()}
    assert b.steps == 3
    for i, rid in enumerate(rids):
        n = int((g["ids"][i] >= 0).sum())
        m = min(int(g["ks"][i]), n)
        assert np.array_equal(out[rid].ids[:m], g["ids"][i, :m])
        assert np.array_equal(out[rid].dists[:m], g["dists"][i, :m])


def test_c3_ragged_prefill_decode_mix():
    """C3 shapes on a scaled database: prefill k=100/nprobe=64 and decode
    k=10/nprobe=16 (1:2, the reference's default trace mix) in one launch."""
    data = gen_matrix(60_000, 64, 31)
    store = VectorStore(data=data)
    idx = IVFFlatIndex.train(store, nlist=256, iters=5, seed=2)
    cen, asg = idx.export()
    art = orc.IVFArtifact(cen, asg)
    b = RetrievalBatcher(idx, max_batch=256)
    qs = gen_matrix(48, 64, 32)
    stages = ["prefill" if i % 3 == 0 else "decode" for i in range(48)]
    rids = [b.submit(q, stage=s) for q, s in zip(qs, stages)]
    res = {r.request_id: r for r in b.step()}
    assert idx.last_fixups() == 0
    for i, rid in enumerate(rids):
        k, npb = (100, 64) if stages[i] == "prefill" else (10, 16)
        oi, od = orc.ivf_search(data, art, qs[i], k, npb)
        assert np.array_equal(res[rid].ids, oi) and np.array_equal(res[rid].dists, od)


def test_simulated_shards_device_merge():
    """C4 on one GPU: 3 id-range shards with the shared artifact, per-shard
    search, device (dist, id) merge == the global oracle."""
    data = gen_matrix(9000, 24, 41)
    art = orc.kmeans(data, 32, 3, 4)
    qs = gen_matrix(16, 24, 42)
    k, npb = 12, 6
    parts_i, parts_d = [], []
    for r in range(3):
        lo, hi = shard_bounds(data.shape[0], 3, r)
        idx = IVFFlatIndex.from_artifact(VectorStore(data=data[lo:hi]), art.centroids, art.assign[lo:hi],
                                         id_offset=lo)
        ids, d = idx.search(qs, k, npb)
        ids, d = pad_results(ids, d, k)
        parts_i.append(ids)
        parts_d.append(d)
    gi = torch.from_numpy(np.stack(parts_i)).cuda()
    gd = torch.from_numpy(np.stack(parts_d)).cuda()
    mi, md = device_merge(gd, gi, k)
    for j, q in enumerate(qs):
        oi, od = orc.ivf_search(data, art, q, k, npb)
        assert np.array_equal(mi[j, : oi.size], oi) and np.array_equal(md[j, : od.size], od)
