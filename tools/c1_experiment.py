"""C1 brute-force timing under library option sets (not a benchmark of record).

python tools/c1_experiment.py "opt=v,opt2=v" ...   (options apply cumulatively; tc_box_rows needs a new store)
C1_SAME_STORE=1 keeps one store for every spec (placement held fixed: the A/B of an option alone)
"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02281_b200 import _lib  # noqa: E402
from paper_2512_02281_b200.ann_graph import _DeviceStore  # noqa: E402
from paper_2512_02281_b200.workload import gen_matrix  # noqa: E402

g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "bf_c1.npz"))
data = gen_matrix(100_000, 128, 1)
qs = gen_matrix(64, 128, 2).astype(np.float64)
lib = _lib.gpu()
q = torch.from_numpy(qs).cuda()
ks = np.full(64, 10, np.int32)
ids = torch.empty((64, 10), dtype=torch.int64, device="cuda")
d = torch.empty((64, 10), dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
same = os.environ.get("C1_SAME_STORE") == "1"
shared = _DeviceStore(data) if same else None
for spec in sys.argv[1:] or [""]:
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    store = shared if same else _DeviceStore(data)

    def one():
        _lib.check(lib.tri_knn_bruteforce_dev(store.handle, _lib.ptr(q), 64, ks.ctypes.data, 10, _lib.ptr(ids),
                                              _lib.ptr(d), C.c_void_p(st.cuda_stream)))

    for _ in range(60):  # the first tens of batches after a store's creation run slower
        one()
    st.synchronize()
    ok = np.array_equal(ids.cpu().numpy(), g["ids"]) and np.array_equal(d.cpu().numpy(), g["dists"])
    reps, host = [], []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        t0 = time.perf_counter()
        for _ in range(200):
            one()
        host.append((time.perf_counter() - t0) / 200 * 1e6)
        e1.record(st)
        e1.synchronize()
        reps.append(e0.elapsed_time(e1) / 200 * 1e3)
    reps.sort()
    print(f"[{spec or 'defaults'}] {reps[3]:.1f} us/batch (min {reps[0]:.1f}, max {reps[-1]:.1f}) "
          f"host enqueue {sorted(host)[3]:.1f} us/call parity={'ok' if ok else 'MISMATCH'}", flush=True)
    if not same:
        store.close()
