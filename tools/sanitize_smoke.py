"""Small runs of every device kernel family, for compute-sanitizer.

memcheck / racecheck / synccheck / initcheck over: the tensor-core brute force
(TF32 tcgen05 scan, wide 64-query items with the TMEM seed pass, select, fp64
re-rank with the fused compact merge), the IVF pipeline (split-fp16 tcgen05
coarse GEMM, dense select, coarse set kernel, device packer, fp16 tcgen05
list scan, merge, re-rank) on a ragged padded batch (device-built plan), the
forced fix-up path, the graph engine step kernel, the exhaustive large-k
brute force, the native NCCL sharded search (one rank) and the shard merge.  Each result is checked against the CPU oracle; exit code 1 on a
mismatch.  CUDA graphs are off (TRI_GRAPHS=0) so every kernel is launched
directly under the tool.

usage: TRI_GRAPHS=0 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle import trinity_oracle as orc
    from paper_2512_02281_b200 import _lib
    from paper_2512_02281_b200.ann_graph import VectorStore, brute_force_knn_batch, build_knn_graph
    from paper_2512_02281_b200.engine import ContinuousBatchEngine, EngineConfig
    from paper_2512_02281_b200.ivf import IVFFlatIndex, merge_topk_device

    rng = np.random.Generator(np.random.Philox(77))
    bad = 0
    # 1. brute force on tensor cores (store large enough for the scan kernels)
    data = rng.standard_normal((20_000, 128)).astype(np.float32)
    qs = rng.standard_normal((64, 128))
    ids, d = brute_force_knn_batch(VectorStore(data=data), qs, 10)
    for i in range(0, 64, 9):
        oi, od = orc.exact_knn(data, qs[i], 10)
        bad += not (np.array_equal(ids[i], oi) and np.array_equal(d[i], od))
    print("brute force", "ok" if not bad else "MISMATCH", flush=True)
    # 2. IVF ragged batch (prefill k=100 nprobe=16 + decode k=10 nprobe=4)
    x = rng.standard_normal((30_000, 96)).astype(np.float32)
    idx = IVFFlatIndex.train(VectorStore(data=x), nlist=64, iters=2, seed=3)
    art = orc.IVFArtifact(*idx.export())
    q = rng.standard_normal((24, 96))
    ks = np.array([100, 10, 10] * 8)
    nps = np.array([16, 4, 4] * 8)
    ids, d = idx.search(q, ks, nps)
    for i in range(0, 24, 5):
        oi, od = orc.ivf_search(x, art, q[i], int(ks[i]), int(nps[i]))
        bad += not (np.array_equal(ids[i, :oi.size], oi) and np.array_equal(d[i, :od.size], od))
    print("ivf", "ok" if not bad else "MISMATCH", flush=True)
    # 3. forced fix-up path (every query uncertified)
    _lib.set_option("force_fixup", 1)
    ids, d = idx.search(q[:6], 10, 8)
    _lib.set_option("force_fixup", 0)
    for i in range(6):
        oi, od = orc.ivf_search(x, art, q[i], 10, 8)
        bad += not (np.array_equal(ids[i, :oi.size], oi) and np.array_equal(d[i, :od.size], od))
    print("fix-up", "ok" if not bad else "MISMATCH", flush=True)
    # 4. graph engine
    g = rng.standard_normal((2000, 16)).astype(np.float32)
    gs = VectorStore(data=g)
    graph = build_knn_graph(gs, 8)
    gq = rng.standard_normal((12, 16))
    eng = ContinuousBatchEngine(gs, graph, EngineConfig(m=32, p=2, entry_count=4, batch_capacity=64))
    rids = eng.submit_many(gq, 5)
    eng.run_to_completion()
    ref_ids, ref_d, ref_ext, _, _ = orc.engine_run(g, graph.adjacency, gq, np.full(12, 5), np.zeros(12, np.int64),
                                                   m=32, p=2, entry_count=4, batch_capacity=64)
    for i, rid in enumerate(rids):
        r = eng.result(int(rid))
        bad += [n.id for n in r.neighbors] != ref_ids[i].tolist()
    print("engine", "ok" if not bad else "MISMATCH", flush=True)
    # 4b. exhaustive large-k brute force (k > TRI_MAX_K: exact distances + radix sort)
    big = rng.standard_normal((3000, 16)).astype(np.float32)
    bq = rng.standard_normal((2, 16))
    ids, d = brute_force_knn_batch(VectorStore(data=big), bq, 2000)
    for i in range(2):
        oi, od = orc.exact_knn(big, bq[i], 2000)
        bad += not (np.array_equal(ids[i], oi) and np.array_equal(d[i], od))
    print("exhaustive", "ok" if not bad else "MISMATCH", flush=True)
    # 4c. native sharded search (one-rank NCCL communicator): search, all-gather, strided merge
    from paper_2512_02281_b200.sharded import ShardedIVF

    sh = ShardedIVF(idx, 10, transport="native")
    qd = torch.from_numpy(q).cuda()
    si = torch.empty((24, 10), dtype=torch.int64, device="cuda")
    sd = torch.empty((24, 10), dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    sh.search_device(qd, 8, si, sd, st)
    st.synchronize()
    ri, rd = idx.search(q, 10, 8)
    bad += not (np.array_equal(si.cpu().numpy(), ri) and np.array_equal(sd.cpu().numpy(), rd))
    sh.close()
    print("native sharded", "ok" if not bad else "MISMATCH", flush=True)
    # 5. shard merge
    dd = torch.from_numpy(np.sort(rng.random((3, 5, 7)), axis=2)).cuda()
    ii = torch.from_numpy(rng.integers(0, 10_000, (3, 5, 7))).cuda()
    od = torch.empty((5, 7), dtype=torch.float64, device="cuda")
    oi = torch.empty((5, 7), dtype=torch.int64, device="cuda")
    merge_topk_device(dd, ii, 7, od, oi)
    torch.cuda.synchronize()
    for b in range(5):
        mi, md = orc.merge_shards([(ii[gg, b].cpu().numpy(), dd[gg, b].cpu().numpy()) for gg in range(3)], 7)
        bad += not np.array_equal(oi[b].cpu().numpy(), mi)
    print("merge", "ok" if not bad else "MISMATCH", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
