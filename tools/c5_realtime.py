"""C5 repeatability: the real-time pool (bench_configs.c5) over the C2 index,
both policies at two arrival rates, ``--repeats`` runs each.

usage: python tools/c5_realtime.py [--repeats 3] [--out gpurun_out/c5.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import bench
    import bench_configs as bc

    b = bench.build_ivf(bench.IVF_CONFIGS["C2"], bench.Ctx(0, 1, 0, None))
    r = bc.c5(b, bench.load_peaks()[0], repeats=a.repeats)
    txt = json.dumps(r, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt)
    for name, reps in r["runs"].items():
        reps = reps if isinstance(reps, list) else [reps]
        print(name, [{s: round(v["p99_ms"], 2) for s, v in x["latency"].items()} for x in reps])
    print("cpu", {s: round(v["p99_ms"], 1) for s, v in r["cpu_baseline"]["latency_ms"].items()})


if __name__ == "__main__":
    main()
