"""Per-batch fix-up counts and device times of the C3 batches on one stream (diagnostic).

python tools/c3_fixups.py [opt=value ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02281_b200 import _lib  # noqa: E402
from paper_2512_02281_b200.ann_graph import _DeviceStore  # noqa: E402
from paper_2512_02281_b200.ivf import IVFFlatIndex  # noqa: E402
from paper_2512_02281_b200.workload import WorkloadSpec, gen_trace, gen_vectors_chunked  # noqa: E402

for kv in sys.argv[1:]:
    k, v = kv.split("=")
    _lib.set_option(k, int(v))
data = gen_vectors_chunked(1_000_000, 768, 3)
idx = IVFFlatIndex.train(_DeviceStore(data), 1024, 5, 4)
spec = WorkloadSpec(n_db=data.shape[0], dim=data.shape[1], n_requests=1200, arrival_rate=1e4, seed=7)
items = []
for r in gen_trace(spec):
    for j in range(r.queries.shape[0]):
        items.append((r.queries[j], j == 0))
qs = np.stack([q for q, _ in items]).astype(np.float64)
pre = np.array([p for _, p in items])
ks = np.where(pre, 100, 10).astype(np.int32)
nps = np.where(pre, 64, 16).astype(np.int32)
n = qs.shape[0]
q_dev = torch.from_numpy(qs).cuda()
ids = torch.empty((n, 100), dtype=torch.int64, device="cuda")
d = torch.empty((n, 100), dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
for rep in range(2):
    out = []
    for s in range(0, n, 256):
        e = min(n, s + 256)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        idx.search_device(q_dev[s:e], ks[s:e], nps[s:e], ids[s:e], d[s:e], st)
        e1.record(st)
        e1.synchronize()
        out.append((s, int(pre[s:e].sum()), idx.last_fixups(), round(e0.elapsed_time(e1), 3)))
    print(rep, out, flush=True)
