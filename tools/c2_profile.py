"""C2 search steps for ncu: builds the bench's C2 index, warms up, then runs
``--steps`` searches (one lane, 256 queries) between cudaProfilerStart/Stop,
so `ncu --profile-from-start off` sees exactly those steps' kernels.
``--c3`` runs the first ragged C3 batch (prefill k100/np64 + decode k10/np16)
over the same index instead.

usage: TRI_GRAPHS=0 ncu --profile-from-start off ... python tools/c2_profile.py [--steps 3] [--c3] [--opt k=v,...]
       python tools/c2_profile.py --c3 --opt scan_debug=16   (scan append / fold counters per step)
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--c3", action="store_true")
    ap.add_argument("--opt", default="", help="library options k=v,k=v set before the warm-up")
    a = ap.parse_args()
    import torch

    import bench

    from paper_2512_02281_b200 import _lib

    for kv in filter(None, a.opt.split(",")):
        _lib.set_option(kv.split("=")[0], int(kv.split("=")[1]))
    b = bench.build_ivf(bench.IVF_CONFIGS[a.config], bench.Ctx(0, 1, 0, None))
    idx = b["idx"]
    q = torch.from_numpy(bench.queries_f64()).cuda()
    k, npb, kmax = 10, 32, 10
    if a.c3:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_configs as bc

        qs, _, ks, nps = bc.c3_workload(b["data"].shape[0], b["data"].shape[1])
        q = torch.from_numpy(qs[:256]).cuda()
        k, npb, kmax = ks[:256], nps[:256], 100
    ids = torch.empty((256, kmax), dtype=torch.int64, device="cuda")
    d = torch.empty((256, kmax), dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    for _ in range(5):
        idx.search_device(q, k, npb, ids, d, st)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(a.steps):
        idx.search_device(q, k, npb, ids, d, st)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    if "scan_debug=16" in a.opt:
        import ctypes as C

        import numpy as np

        cnt = np.zeros(4, np.uint64)
        _lib.check(_lib.gpu().tri_debug_scan_ts(cnt.ctypes.data_as(C.c_void_p), 4))
        print(f"per step: appended {cnt[0] / (a.steps + 5):.0f} in {cnt[1] / (a.steps + 5):.0f} folds; "
              f"kp>=128 members {cnt[2] / (a.steps + 5):.0f} in {cnt[3] / (a.steps + 5):.0f} folds")
    print("done", a.steps, "steps of", a.config)


if __name__ == "__main__":
    main()
