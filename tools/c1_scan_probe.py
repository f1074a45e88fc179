"""C1 brute-force batches under one option set, for ncu captures of the scan kernel (not a benchmark of record).

python tools/c1_scan_probe.py "opt=v,opt2=v" [batches]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02281_b200 import _lib  # noqa: E402
from paper_2512_02281_b200.ann_graph import _DeviceStore  # noqa: E402
from paper_2512_02281_b200.workload import gen_matrix  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else ""
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
B = int(os.environ.get("C1_B", "64"))
data = gen_matrix(100_000, 128, 1)
qs = gen_matrix(B, 128, 2).astype(np.float64)
lib = _lib.gpu()
q = torch.from_numpy(qs).cuda()
ks = np.full(B, 10, np.int32)
ids = torch.empty((B, 10), dtype=torch.int64, device="cuda")
d = torch.empty((B, 10), dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
for kv in filter(None, spec.split(",")):
    k, v = kv.split("=")
    _lib.set_option(k, int(v))
store = _DeviceStore(data)
for _ in range(n):
    _lib.check(lib.tri_knn_bruteforce_dev(store.handle, _lib.ptr(q), B, ks.ctypes.data, 10, _lib.ptr(ids),
                                          _lib.ptr(d), C.c_void_p(st.cuda_stream)))
st.synchronize()
print("done", spec)
if "scan_debug" in spec and int(dict(kv.split("=") for kv in spec.split(",") if kv).get("scan_debug", 0)) & 8:
    ts = np.zeros(256 * 16, np.uint64)
    _lib.check(lib.tri_debug_scan_ts(ts.ctypes.data, ts.size))
    ts = ts.reshape(256, 16).astype(np.int64)
    live = ts[:, 0] > 0
    t0 = ts[live, 0].min()
    rel = (ts[live] - t0) / 1e3
    names = ["entry", "setup", "item", "qtile", "mma0", "epi0", "lastTMA", "epi_end", "seedA", "publish", "spun",
             "seeded", "B_loop", "B_sync", "B_rel", "B_out"]
    for i, nm in enumerate(names):
        col = rel[:, i]
        print(f"{nm:8s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us")
if "scan_debug" in spec and int(dict(kv.split("=") for kv in spec.split(",") if kv).get("scan_debug", 0)) & 16:
    cnt = np.zeros(4, np.uint64)
    _lib.check(lib.tri_debug_scan_ts(cnt.ctypes.data, 4))
    print(f"per batch: appended {cnt[0] / n:.0f}, folds {cnt[1] / n:.0f}, seeds open {cnt[2] / n:.0f}, set {cnt[3] / n:.0f}")
