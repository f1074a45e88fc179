"""C1 brute-force time per batch for several allocations of the same store (not a benchmark of record).

python tools/c1_placement.py   (TRI_DEBUG_ALLOC=1 prints each store's device addresses)

Each store: 100 + 300 batches per L2 policy of the scan loads (scan_l2hint 0, 1, 2, 0).
Shows the per-allocation fast / slow modes described in DESIGN.md section 9.
"""
import ctypes as C, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2512_02281_b200 import _lib
from paper_2512_02281_b200.ann_graph import _DeviceStore
from paper_2512_02281_b200.workload import gen_matrix
data = gen_matrix(100_000, 128, 1)
qs = gen_matrix(64, 128, 2).astype(np.float64)
lib = _lib.gpu()
q = torch.from_numpy(qs).cuda()
ks = np.full(64, 10, np.int32)
ids = torch.empty((64, 10), dtype=torch.int64, device="cuda")
d = torch.empty((64, 10), dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
def run(store, tag):
    def one():
        _lib.check(lib.tri_knn_bruteforce_dev(store.handle, _lib.ptr(q), 64, ks.ctypes.data, 10, _lib.ptr(ids), _lib.ptr(d), C.c_void_p(st.cuda_stream)))
    res = {}
    for h in (0, 1, 2, 0):
        _lib.set_option("scan_l2hint", h)
        for _ in range(100): one()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(300): one()
        e1.record(st); e1.synchronize()
        res.setdefault(h, []).append(round(e0.elapsed_time(e1) / 300 * 1e3, 1))
    _lib.set_option("scan_l2hint", 0)
    print(tag, res, flush=True)
if len(sys.argv) > 1:
    for kv in sys.argv[1:]:
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
A = _DeviceStore(data); run(A, "A")
B = _DeviceStore(data); run(B, "B (A alive)")
run(A, "A again")
Cs = _DeviceStore(data); run(Cs, "C")
A.close(); B.close(); Cs.close()
D = _DeviceStore(data); run(D, "D (after closing all)")
E = _DeviceStore(data); run(E, "E")
