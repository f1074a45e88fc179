"""C4 on one B200: the 10M x 768 IVF database and each rank's share of it.

BASELINE config 4 shards IVF-Flat 10M x 768 across 2/4/8 GPUs.  Only one GPU
is available, so this measures, on that GPU, what one rank of
`bench.py --gpus G` (config C4) holds and scans per batch: rows
[0, 10M / G) of the C4 database (gen_vectors_chunked(10M, 768, seed=100)),
listed under the same centroids (k-means on rows [0, 1M), every row's exact
nearest centroid), searched with C2-shaped batches (256 queries, nprobe 32,
k 10) on `--lanes` streams.  The per-batch gather of B*k*16 bytes per rank and
the device merge are not in these numbers.

Parity: `--check` queries of every run against the CPU oracle over the shard.

usage: python tools/bench_c4.py [--shards 1,2,4,8] [--steps 40] [--out gpurun_out/c4.json]
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

    import bench
    from oracle import trinity_oracle as orc
    from oracle.pool import ivf_oracle_batch
    from paper_2512_02281_b200.ann_graph import _DeviceStore
    from paper_2512_02281_b200.ivf import IVFFlatIndex
    from paper_2512_02281_b200.workload import gen_rows_chunked

    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--lanes", type=int, default=4)
    ap.add_argument("--check", type=int, default=8)
    ap.add_argument("--out", default=None)
    ap.add_argument("--opt", action="append", default=[], help="library option name=value")
    a = ap.parse_args()
    from paper_2512_02281_b200 import _lib

    for kv in a.opt:
        name, val = kv.split("=")
        _lib.set_option(name, int(val))
    cfg = bench.IVF_CONFIGS["C4"]
    N, D, B, K, NPROBE = cfg["n"], bench.DIM, bench.BATCH, bench.K, bench.NPROBE
    t0 = time.perf_counter()
    train = gen_rows_chunked(0, cfg["n_train"], D, cfg["seed"])
    ts = _DeviceStore(train)
    ti = IVFFlatIndex.train(ts, bench.NLIST, bench.ITERS, bench.KM_SEED)
    cen, _ = ti.export()
    ti.close()
    ts.close()
    del train
    queries = bench.queries_f64()
    q_dev = torch.from_numpy(queries).cuda()
    out = {"workload": cfg["workload"] + "; shard g of G = rows [0, N/G) on one GPU", "train_s": time.perf_counter() - t0,
           "runs": {}}
    for G in [int(x) for x in a.shards.split(",")]:
        n = N // G
        data = gen_rows_chunked(0, n, D, cfg["seed"])
        store = _DeviceStore(data)
        idx = IVFFlatIndex.from_centroids(store, cen)
        store.close()
        L = a.lanes
        lanes = [torch.cuda.Stream() for _ in range(L)]
        ids = [torch.empty((B, K), dtype=torch.int64, device="cuda") for _ in range(L)]
        ds = [torch.empty((B, K), dtype=torch.float64, device="cuda") for _ in range(L)]
        for j in range(3 * L):
            idx.search_device(q_dev, K, NPROBE, ids[j % L], ds[j % L], lanes[j % L])
        torch.cuda.synchronize()
        rows = list(range(0, B, max(1, B // a.check)))[: a.check]
        art = orc.IVFArtifact(cen, idx.export()[1])
        ref = ivf_oracle_batch(data, art, queries[rows], K, NPROBE)
        hid, hd = ids[0].cpu().numpy(), ds[0].cpu().numpy()
        bad = sum(1 for j, i in enumerate(rows)
                  if not (np.array_equal(hid[i], ref[j][0]) and np.array_equal(hd[i], ref[j][1])))
        idx.set_profiling(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(lanes[0])
        for ls in lanes[1:]:
            ls.wait_event(e0)
        for j in range(a.steps):
            idx.search_device(q_dev, K, NPROBE, ids[j % L], ds[j % L], lanes[j % L])
        for ls in lanes[1:]:
            lanes[0].wait_stream(ls)
        e1.record(lanes[0])
        torch.cuda.synchronize()
        scan_ms, scan_n = idx.scan_time()
        stages, ns = idx.stage_times()
        idx.set_profiling(False)
        ms = e0.elapsed_time(e1) / a.steps
        scan_bytes, _ = idx.last_scan_bytes()
        rec = {"rows": n, "qps": B / (ms / 1e3), "ms_per_batch": ms, "scan_ms": scan_ms / max(scan_n, 1),
               "scan_bytes": scan_bytes, "scan_gbs": scan_bytes / (scan_ms / max(scan_n, 1) / 1e3) / 1e9,
               "stage_ms": {k: v / max(ns, 1) for k, v in stages.items()}, "fixups_last_batch": idx.last_fixups(),
               "parity": f"{'ok' if not bad else 'FAIL'}: {len(rows)} queries == CPU oracle over the shard"}
        out["runs"][f"G={G}"] = rec
        print(json.dumps({f"G={G}": rec}), flush=True)
        idx.close()
        del data
        torch.cuda.synchronize()
    g1 = out["runs"].get("G=1", {}).get("qps")
    if g1:
        out["ideal_scaling_from_shares"] = {k: v["qps"] / g1 for k, v in out["runs"].items()}
    txt = json.dumps(out, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
