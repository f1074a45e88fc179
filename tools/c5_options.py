"""C5 scheduled-trace GPU time per policy under library option sets (diagnostic).

python tools/c5_options.py "" "pack_mixed=0" ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_configs as b  # noqa: E402
from paper_2512_02281_b200 import _lib  # noqa: E402
from paper_2512_02281_b200.ann_graph import _DeviceStore  # noqa: E402
from paper_2512_02281_b200.ivf import IVFFlatIndex  # noqa: E402
from paper_2512_02281_b200.workload import gen_vectors_chunked  # noqa: E402

data = gen_vectors_chunked(1_000_000, 768, 3)
idx = IVFFlatIndex.train(_DeviceStore(data), 1024, 5, 4)
for spec in sys.argv[1:] or [""]:
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    r = b.c5(idx)
    out = {p: (v["batches"], round(v["gpu_ms"], 1), round(v["latency"]["prefill"]["p50_ms"], 2))
           for p, v in r["policies"].items()}
    print(f"[{spec or 'defaults'}] (batches, gpu_ms, prefill p50 ms) {out}", flush=True)
