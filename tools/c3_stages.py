"""C3 per-stage timings and fix-up counts under library option sets (diagnostic).

usage: python tools/c3_stages.py "opt=v,..." ...   (options apply cumulatively)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench  # noqa: E402
import bench_configs as bc  # noqa: E402
from paper_2512_02281_b200 import _lib  # noqa: E402

b = bench.build_ivf(bench.IVF_CONFIGS["C2"], bench.Ctx(0, 1, 0, None))
idx = b["idx"]
for spec in sys.argv[1:] or [""]:
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    r = bc.c3(b, bench.load_peaks()[0])
    print(f"[{spec or 'defaults'}] qps {r['value']:.0f} e2e {r['e2e']['value']:.0f} scan_ms/launch "
          f"{r['roofline']['scan_ms_per_launch']:.3f} frac {r['roofline']['frac']:.3f} fixups(last) {idx.last_fixups()} "
          + r["parity"], flush=True)
