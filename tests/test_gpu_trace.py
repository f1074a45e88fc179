"""Scheduled retrieval trace (C5): every retrieval served, results exact, latencies reported."""

import numpy as np
import pytest

from oracle import trinity_oracle as orc
from paper_2512_02281_b200.ann_graph import VectorStore
from paper_2512_02281_b200.ivf import IVFFlatIndex
from paper_2512_02281_b200.scheduler import SchedulerConfig
from paper_2512_02281_b200.trace import run_trace
from paper_2512_02281_b200.workload import LengthDist, WorkloadSpec, gen_matrix, gen_trace

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("policy", ["prefill_reserved", "decode_priority"])
def test_trace_serves_everything_exactly(policy):
    data = gen_matrix(20_000, 32, 61)
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=128, iters=4, seed=1)
    cen, asg = idx.export()
    art = orc.IVFArtifact(cen, asg)
    cache = VectorStore(data=gen_matrix(500, 32, 62))
    spec = WorkloadSpec(n_db=20_000, dim=32, n_requests=60, arrival_rate=3000.0,
                        output_len_dist=LengthDist.fixed(64), delta=32, seed=7)
    cfg = SchedulerConfig(slots_n=64, r=0.25, tau_pre=5e-5, tau_global=2e-4, policy=policy)
    res = run_trace(idx, cache, spec, cfg, tpot=1e-3, keep_results=True)
    pct = res.percentiles()
    assert pct["prefill"]["n"] == 60 and pct["decode"]["n"] == 120 and pct["cache"]["n"] == 60
    for st in pct.values():
        assert 0 < st["p50_ms"] <= st["p95_ms"] <= st["p99_ms"]
    trace = gen_trace(spec)
    for r in trace[::7]:
        for j in range(r.queries.shape[0]):
            k, npb = (100, 64) if j == 0 else (10, 16)
            oi, _ = orc.ivf_search(data, art, r.queries[j], k, npb)
            assert np.array_equal(res.results[(r.id, j)], oi)
