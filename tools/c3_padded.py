"""C3 with and without fixed-shape padded graphs (option ragged_graphs), more
batches than the bench's configs pass: device QPS (4 lanes) and e2e through
search_into (pinned, one host thread per lane).

usage: python tools/c3_padded.py [--requests 4800]
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=4800)
    a = ap.parse_args()
    import bench
    import bench_configs as bc
    from paper_2512_02281_b200 import _lib

    b = bench.build_ivf(bench.IVF_CONFIGS["C2"], bench.Ctx(0, 1, 0, None))
    orig = bc.c3_workload
    bc.c3_workload = lambda n, d, n_requests=0: orig(n, d, a.requests)
    for rg in (1, 0, 1):
        _lib.set_option("ragged_graphs", rg)
        c0 = _lib.graph_counters()
        r = bc.c3(b, bench.load_peaks()[0])
        c1 = _lib.graph_counters()
        print(f"ragged_graphs={rg}: qps {r['value']:.0f} e2e {r['e2e']['value']:.0f} batches {r['batches']} "
              f"scan frac {r['roofline']['frac']:.3f} graphs {dict((k, c1[k] - c0[k]) for k in c1)} {r['parity']}",
              flush=True)


if __name__ == "__main__":
    main()
