"""C3 per-stage timings and fix-up counts under library option sets (diagnostic)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_configs as b  # noqa: E402
from oracle import trinity_oracle as orc  # noqa: E402
from paper_2512_02281_b200 import _lib  # noqa: E402
from paper_2512_02281_b200.ann_graph import _DeviceStore  # noqa: E402
from paper_2512_02281_b200.ivf import IVFFlatIndex  # noqa: E402
from paper_2512_02281_b200.workload import gen_vectors_chunked  # noqa: E402

data = gen_vectors_chunked(1_000_000, 768, 3)
idx = IVFFlatIndex.train(_DeviceStore(data), 1024, 5, 4)
cen, asg = idx.export()
art = orc.IVFArtifact(cen, asg)
for spec in sys.argv[1:] or [""]:
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    idx.set_profiling(True)
    r = b.c3(idx, data, art)
    st, n = idx.stage_times()
    idx.set_profiling(False)
    print(f"[{spec or 'defaults'}] qps {r['qps']:.0f} ms/batch(1 stream) {r['ms_per_batch_one_stream']:.3f} fixups(last) {idx.last_fixups()} "
          + json.dumps({k: round(v / n * 1e3, 1) for k, v in st.items()}) + " " + r["parity"], flush=True)
