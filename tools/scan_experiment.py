"""Timing experiments for the list-scan kernel on the C2 workload (not a benchmark of record).

python tools/scan_experiment.py [--n 1000000] [--modes 0,1,2,3]
mode bits: 1 = skip selection, 2 = skip MMA (results invalid, timing only)
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2512_02281_b200 import _lib  # noqa: E402
from paper_2512_02281_b200.ann_graph import _DeviceStore  # noqa: E402
from paper_2512_02281_b200.ivf import IVFFlatIndex  # noqa: E402
from paper_2512_02281_b200.workload import gen_matrix, gen_vectors_chunked  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=768)
ap.add_argument("--nlist", type=int, default=1024)
ap.add_argument("--nprobe", type=int, default=32)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--modes", default="0,1,2,3")
ap.add_argument("--kernels", default="0,1")
ap.add_argument("--stages", default="0", help="tensor-core ring depth caps to try (0 = deepest)")
ap.add_argument("--reserve", default="0", help="SMs left out of the scan grid")
ap.add_argument("--box-rows", type=int, default=128)
args = ap.parse_args()

data = gen_vectors_chunked(args.n, args.d, 3)
qs = gen_matrix(args.B, args.d, 4).astype(np.float64)
_lib.set_option("tc_box_rows", args.box_rows)
store = _DeviceStore(data)
t = time.time()
idx = IVFFlatIndex.train(store, args.nlist, 5, 4)
print(f"train {time.time() - t:.2f}s", flush=True)
for kern, stg, rsv in [(int(x), int(y), int(z)) for x in args.kernels.split(",") for y in args.stages.split(",")
                       for z in args.reserve.split(",")]:
    _lib.set_option("scan_kernel", kern)
    _lib.set_option("tc_stages", stg)
    _lib.set_option("scan_reserve", rsv)
    for mode in [int(x) for x in args.modes.split(",")]:
        _lib.set_option("scan_debug", mode)
        for _ in range(3):
            idx.search(qs, args.k, args.nprobe)
        idx.set_profiling(True)
        t = time.perf_counter()
        for _ in range(20):
            idx.search(qs, args.k, args.nprobe)
        wall = (time.perf_counter() - t) / 20
        st, n = idx.stage_times()
        ms = st["scan"]
        idx.set_profiling(False)
        b, pairs = idx.last_scan_bytes()
        print(f"kernel={kern} stages={stg} reserve={rsv} mode={mode} scan {ms / n:.3f} ms ({b / (ms / n) / 1e6:.0f} GB/s)  "
              f"call {wall * 1e3:.3f} ms  fixups={idx.last_fixups()}  stages(us)="
              + " ".join(f"{k}={v / n * 1e3:.0f}" for k, v in st.items()), flush=True)
_lib.set_option("scan_debug", 0)
