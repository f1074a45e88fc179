"""C4 on one B200: the 10M x 768 IVF database and each rank's share of it.

BASELINE config 4 shards IVF-Flat 10M x 768 across 2/4/8 GPUs.  Only one GPU
is available here, so this measures, on that GPU:

* the whole 10M database (G = 1): QPS of C2-shaped batches (256 queries,
  nlist 1024, nprobe 32, k 10) and the scan's HBM rate at that scale;
* the per-rank workload at G = 2, 4, 8: rows [0, 10M/G) of the same
  database with the SAME k-means artifact (how bench.py --gpus G shards), i.e.
  exactly what one rank scans per batch.  The NCCL gather of the per-shard
  top-k (B*k*(8+8) bytes per rank) and the device merge are not in these numbers.

Parity: a few queries of every run against the CPU oracle (composed from the
reference's primitives over the shard's rows).

usage: python tools/bench_c4.py [--n 10000000] [--shards 1,2,4,8] [--steps 60]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle import trinity_oracle as orc
    from paper_2512_02281_b200.ann_graph import _DeviceStore
    from paper_2512_02281_b200.ivf import IVFFlatIndex
    from paper_2512_02281_b200.workload import gen_matrix, gen_vectors_chunked

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--shards", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--lanes", type=int, default=3)
    a = ap.parse_args()
    N, D, NLIST, NPROBE, B, K = a.n, 768, 1024, 32, 256, 10
    t0 = time.perf_counter()
    data = gen_vectors_chunked(N, D, 100)
    t_gen = time.perf_counter() - t0
    queries = gen_matrix(B, D, 4).astype(np.float64)
    t0 = time.perf_counter()
    full = _DeviceStore(data)
    idx = IVFFlatIndex.train(full, NLIST, 5, 4)
    cen, asg = idx.export()
    idx.close()
    full.close()
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    out = {"workload": f"C4 on one GPU: gen_vectors_chunked({N}, 768, seed=100), nlist {NLIST} (5 Lloyd iters), "
                       f"nprobe {NPROBE}, batch {B}, k {K}; shard g of G = rows [0, N/G) with the full-database "
                       f"k-means artifact", "gen_s": t_gen, "build_s": t_build, "runs": {}}
    q_dev = torch.from_numpy(queries).cuda()
    for G in [int(x) for x in a.shards.split(",")]:
        n = N // G
        store = _DeviceStore(data[:n])
        sidx = IVFFlatIndex.from_artifact(store, cen, asg[:n])
        L = a.lanes
        lanes = [torch.cuda.Stream() for _ in range(L)]
        ids = [torch.empty((B, K), dtype=torch.int64, device="cuda") for _ in range(L)]
        ds = [torch.empty((B, K), dtype=torch.float64, device="cuda") for _ in range(L)]
        for j in range(3 * L):
            sidx.search_device(q_dev, K, NPROBE, ids[j % L], ds[j % L], lanes[j % L])
        torch.cuda.synchronize()
        art = orc.IVFArtifact(cen, asg[:n])
        ok = True
        hid, hd = ids[0].cpu().numpy(), ds[0].cpu().numpy()
        for i in (0, 131, 255):
            oi, od = orc.ivf_search(data[:n], art, queries[i], K, NPROBE)
            ok = ok and np.array_equal(hid[i], oi) and np.array_equal(hd[i], od)
        sidx.set_profiling(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(lanes[0])
        for ls in lanes[1:]:
            ls.wait_event(e0)
        for j in range(a.steps):
            sidx.search_device(q_dev, K, NPROBE, ids[j % L], ds[j % L], lanes[j % L])
        for ls in lanes[1:]:
            lanes[0].wait_stream(ls)
        e1.record(lanes[0])
        torch.cuda.synchronize()
        scan_ms, scan_n = sidx.scan_time()
        sidx.set_profiling(False)
        ms = e0.elapsed_time(e1) / a.steps
        scan_bytes, _ = sidx.last_scan_bytes()
        out["runs"][f"G={G}"] = {
            "rows": n, "qps": B / (ms / 1e3), "ms_per_batch": ms, "scan_ms": scan_ms / max(scan_n, 1),
            "scan_bytes": scan_bytes, "scan_gbs": scan_bytes / (scan_ms / max(scan_n, 1) / 1e3) / 1e9,
            "fixups": sidx.last_fixups(),
            "parity": f"{'ok' if ok else 'MISMATCH'}: queries 0, 131, 255 == CPU oracle over the shard",
        }
        print(json.dumps({f"G={G}": out["runs"][f"G={G}"]}), flush=True)
        sidx.close()
        store.close()
        torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
