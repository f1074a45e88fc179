"""A/B of the coarse (dense) select variants on the bench's C2 index: same
results (ids and distances equal) and the per-search device time with each
option value.  usage: python tools/dense_ab.py [--option dense_fold]"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--option", default="dense_fold")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--values", default="0,1", help="two option values, alternated twice")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2512_02281_b200 import _lib

    b = bench.build_ivf(bench.IVF_CONFIGS["C2"], bench.Ctx(0, 1, 0, None))
    idx = b["idx"]
    q = torch.from_numpy(bench.queries_f64()).cuda()
    st = torch.cuda.Stream()
    out = {}
    res = {}
    v0, v1 = (int(x) for x in a.values.split(","))
    for val in (v0, v1, v0, v1):
        _lib.set_option(a.option, val)
        ids = torch.empty((256, 10), dtype=torch.int64, device="cuda")
        d = torch.empty((256, 10), dtype=torch.float64, device="cuda")
        for _ in range(10):
            idx.search_device(q, 10, 32, ids, d, st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.iters):
            idx.search_device(q, 10, 32, ids, d, st)
        e1.record(st)
        torch.cuda.synchronize()
        out.setdefault(val, []).append(round(e0.elapsed_time(e1) * 1e3 / a.iters, 2))
        res[val] = (ids.cpu(), d.cpu())
    same = bool(torch.equal(res[v0][0], res[v1][0]) and torch.equal(res[v0][1], res[v1][1]))
    print(json.dumps({"option": a.option, "us_per_search": out, "identical": same}))


if __name__ == "__main__":
    main()
