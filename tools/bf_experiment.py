"""Brute-force kNN timing on a few shapes (device buffers, CUDA events; not a benchmark of record)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02281_b200 import _lib  # noqa: E402
from paper_2512_02281_b200.ann_graph import _DeviceStore  # noqa: E402

SHAPES = [(1024, 768, 256, 32), (4096, 768, 256, 32), (100_000, 128, 64, 10), (100_000, 128, 1024, 10)]
if len(sys.argv) > 1:
    SHAPES = [SHAPES[int(i)] for i in sys.argv[1].split(",")]
KERNELS = (1, 2) if len(sys.argv) <= 2 else tuple(int(x) for x in sys.argv[2].split(","))
lib = _lib.gpu()
for n, d, B, k in SHAPES:
    rng = np.random.Generator(np.random.Philox(n + d))
    data = rng.standard_normal((n, d)).astype(np.float32)
    st = _DeviceStore(data)
    q = torch.from_numpy(rng.standard_normal((B, d))).cuda()
    ids = torch.empty((B, k), dtype=torch.int64, device="cuda")
    dd = torch.empty((B, k), dtype=torch.float64, device="cuda")
    ks = np.full(B, k, np.int32)
    s = torch.cuda.Stream()
    for kern in KERNELS:
        _lib.set_option("scan_kernel", kern)
        def run():
            _lib.check(lib.tri_knn_bruteforce_dev(st.handle, q.data_ptr(), B, ks.ctypes.data, k, ids.data_ptr(),
                                                  dd.data_ptr(), s.cuda_stream))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            run()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"n={n} d={d} B={B} k={k} kernel={'simt' if kern == 1 else 'tc'}: {ms * 1e3:.1f} us/batch "
              f"({n * d * 4 / ms / 1e6:.0f} GB/s of rows) fixups={st.last_fixups()}", flush=True)
_lib.set_option("scan_kernel", 0)
