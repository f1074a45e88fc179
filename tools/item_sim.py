"""C2 work-item statistics: list sizes, probes per list, and the makespan of the
persistent scan's longest-first schedule on 148 SMs (cost = rows scanned).

python tools/item_sim.py   (GPU box; builds the C2 index like bench.py)
"""
import heapq
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2512_02281_b200.ann_graph import _DeviceStore  # noqa: E402
from paper_2512_02281_b200.ivf import IVFFlatIndex  # noqa: E402
from paper_2512_02281_b200.workload import gen_matrix, gen_vectors_chunked  # noqa: E402

data = gen_vectors_chunked(1_000_000, 768, 3)
qs = gen_matrix(256, 768, 4).astype(np.float64)
idx = IVFFlatIndex.train(_DeviceStore(data), 1024, 5, 4)
sizes = idx.list_sizes()
idx.search(qs, 10, 32)
pr = idx.last_probes(256, 32)
cnt = np.bincount(pr.ravel(), minlength=1024)
print("list sizes: min %d median %d mean %.0f max %d p99 %d" % (sizes.min(), np.median(sizes), sizes.mean(),
                                                                 sizes.max(), np.percentile(sizes, 99)))
print("probes per list: mean %.1f max %d  lists probed %d" % (cnt.mean(), cnt.max(), (cnt > 0).sum()))
items = []
for l in np.argsort(-sizes, kind="stable"):
    g = (cnt[l] + 15) // 16
    items += [int(sizes[l])] * int(g)
print("items %d, rows scanned %d (unique %d)" % (len(items), sum(items), int(sizes[cnt > 0].sum())))
for ovh in (0, 64, 256):
    sm = [(0, i) for i in range(148)]
    heapq.heapify(sm)
    for r in items:
        t, i = heapq.heappop(sm)
        heapq.heappush(sm, (t + r + ovh, i))
    ts = sorted(t for t, _ in sm)
    print("overhead %3d rows/item: makespan %d, mean %.0f, min %d -> efficiency %.3f" %
          (ovh, ts[-1], np.mean(ts), ts[0], np.mean(ts) / ts[-1]))
