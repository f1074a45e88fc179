"""Per-stage timings of the C2 search pipeline under library option sets (not a benchmark of record).

python tools/stage_experiment.py --opts "gthr=0" "gthr=1" [--n 1000000] [--k 10 --nprobe 32]

Each option set: 3 warm-up searches, then 20 profiled ones (CUDA events per
stage), parity of 4 queries against the CPU oracle, fix-up count.
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import trinity_oracle as orc  # noqa: E402
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
ap.add_argument("--opts", nargs="*", default=[""])
args = ap.parse_args()

data = gen_vectors_chunked(args.n, args.d, 3)
qs = gen_matrix(args.B, args.d, 4).astype(np.float64)
store = _DeviceStore(data)
idx = IVFFlatIndex.train(store, args.nlist, 5, 4)
cen, asg = idx.export()
art = orc.IVFArtifact(cen, asg)
check = [0, 1, args.B // 2, args.B - 1]
ref = {i: orc.ivf_search(data, art, qs[i], args.k, args.nprobe) for i in check}
for spec in args.opts:
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    for _ in range(3):
        idx.search(qs, args.k, args.nprobe)
    idx.set_profiling(True)
    t = time.perf_counter()
    for _ in range(20):
        ids, d = idx.search(qs, args.k, args.nprobe)
    wall = (time.perf_counter() - t) / 20
    st, n = idx.stage_times()
    idx.set_profiling(False)
    ok = all(np.array_equal(ids[i], ref[i][0]) and np.array_equal(d[i], ref[i][1]) for i in check)
    print(f"[{spec or 'defaults'}] call {wall * 1e3:.3f} ms parity={'ok' if ok else 'MISMATCH'} "
          f"fixups={idx.last_fixups()} stages(us)=" + " ".join(f"{k}={v / n * 1e3:.1f}" for k, v in st.items()),
          flush=True)
