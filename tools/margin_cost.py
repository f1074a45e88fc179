"""Cost of the certificate's safety margin: C2 and C3-like ragged batches over
the C2 index at bound_margin 1 and 2 -- fix-ups per batch and device ms."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2512_02281_b200 import _lib
from paper_2512_02281_b200.ann_graph import _DeviceStore
from paper_2512_02281_b200.ivf import IVFFlatIndex
from paper_2512_02281_b200.workload import gen_matrix, gen_vectors_chunked

data = gen_vectors_chunked(1_000_000, 768, 3)
idx = IVFFlatIndex.train(_DeviceStore(data), 1024, 5, 4)
nb = 24
qs = gen_matrix(256 * nb, 768, 77).astype(np.float64)
pre = np.arange(256) % 3 == 0
for margin, div in ((100, 4), (125, 4), (150, 4), (175, 4), (200, 4), (200, 2), (200, 1), (150, 2)):
    _lib.set_option("bound_margin", margin)
    _lib.set_option("f16_div", div)
    for name, ks, nps in (("C2", np.full(256, 10), np.full(256, 32)),
                          ("C3", np.where(pre, 100, 10), np.where(pre, 64, 16))):
        fx = 0
        t = time.perf_counter()
        for b in range(nb):
            idx.search(qs[256 * b: 256 * (b + 1)], ks, nps)
            fx += idx.last_fixups()
        ms = (time.perf_counter() - t) * 1e3 / nb
        print(f"margin={margin}% f16_div={div} {name}: fixups {fx} in {nb * 256} queries ({fx / nb:.2f}/batch), {ms:.3f} ms/batch host-timed",
              flush=True)
