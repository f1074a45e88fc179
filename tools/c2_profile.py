"""C2 search steps for ncu: builds the bench's C2 index, warms up, then runs
``--steps`` searches (one lane, 256 queries) between cudaProfilerStart/Stop,
so `ncu --profile-from-start off` sees exactly those steps' kernels.

usage: TRI_GRAPHS=0 ncu --profile-from-start off ... python tools/c2_profile.py [--steps 3]
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
    a = ap.parse_args()
    import torch

    import bench

    b = bench.build_ivf(bench.IVF_CONFIGS[a.config], bench.Ctx(0, 1, 0, None))
    idx = b["idx"]
    q = torch.from_numpy(bench.queries_f64()).cuda()
    ids = torch.empty((256, 10), dtype=torch.int64, device="cuda")
    d = torch.empty((256, 10), dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    for _ in range(5):
        idx.search_device(q, 10, 32, ids, d, st)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(a.steps):
        idx.search_device(q, 10, 32, ids, d, st)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("done", a.steps, "steps of", a.config)


if __name__ == "__main__":
    main()
