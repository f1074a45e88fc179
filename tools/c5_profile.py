"""Host-side profile of the C5 real-time pool (diagnostic, not a benchmark of record):
one decode_priority run at 10K requests/s under cProfile, plus the device
time of its IVF searches (stage timers) beside the batches' wall time.

usage: python tools/c5_profile.py [rate]
"""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_02281_b200.ann_graph import VectorStore  # noqa: E402
from paper_2512_02281_b200.pool import GpuBackend, RealtimePool  # noqa: E402
from paper_2512_02281_b200.scheduler import SchedulerConfig  # noqa: E402
from paper_2512_02281_b200.workload import WorkloadSpec, gen_matrix, gen_trace  # noqa: E402

rate = float(sys.argv[1]) if len(sys.argv) > 1 else 10_000.0
b = bench.build_ivf(bench.IVF_CONFIGS["C2"], bench.Ctx(0, 1, 0, None))
idx = b["idx"]
cache = VectorStore(data=gen_matrix(10_000, idx.dim, 62))
cfg = SchedulerConfig(slots_n=256, r=0.25, tau_pre=2e-4, tau_global=1e-3, policy="decode_priority")
be = GpuBackend(idx, cache, slots=256, stream=torch.cuda.Stream())
warm = gen_trace(WorkloadSpec(n_db=idx.count, dim=idx.dim, n_requests=2000, arrival_rate=rate, seed=8))
RealtimePool(be, cfg, tpot=5e-3, prefill_chunk=64).run(warm)
trace = gen_trace(WorkloadSpec(n_db=idx.count, dim=idx.dim, n_requests=int(rate), arrival_rate=rate, seed=7))
idx.set_profiling(True)
pr = cProfile.Profile()
pr.enable()
r = RealtimePool(be, cfg, tpot=5e-3, prefill_chunk=64).run(trace)
pr.disable()
st, n = idx.stage_times()
idx.set_profiling(False)
print(f"batches {r.batches} launches {r.launches} busy {r.busy_s:.3f} s wall {r.wall_s:.3f} s "
      f"busy/batch {r.busy_s / r.batches * 1e3:.3f} ms; IVF device ms per search: "
      + " ".join(f"{k}={v / max(n, 1):.3f}" for k, v in st.items()) + f" (n={n})")
print({s: (round(v["p50_ms"], 3), round(v["p99_ms"], 3)) for s, v in r.percentiles().items()})
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
