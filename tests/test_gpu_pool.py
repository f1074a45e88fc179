"""Real-time pool (C5) on the GPU: every retrieval and cache lookup served on
the wall clock through the scheduler, results exact against the oracle."""

import numpy as np
import pytest

from oracle import trinity_oracle as orc
from paper_2512_02281_b200.ann_graph import VectorStore
from paper_2512_02281_b200.ivf import IVFFlatIndex
from paper_2512_02281_b200.pool import GpuBackend, RealtimePool
from paper_2512_02281_b200.scheduler import SchedulerConfig
from paper_2512_02281_b200.workload import LengthDist, WorkloadSpec, gen_matrix, gen_trace

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("policy,chunk", [("prefill_reserved", None), ("decode_priority", None),
                                          ("decode_priority", 8)])
def test_pool_serves_everything_exactly(policy, chunk):
    data = gen_matrix(20_000, 32, 61)
    idx = IVFFlatIndex.train(VectorStore(data=data), nlist=128, iters=4, seed=1)
    cen, asg = idx.export()
    art = orc.IVFArtifact(cen, asg)
    cdata = gen_matrix(500, 32, 62)
    cache = VectorStore(data=cdata)
    spec = WorkloadSpec(n_db=20_000, dim=32, n_requests=200, arrival_rate=20000.0,
                        output_len_dist=LengthDist.fixed(64), delta=32, seed=7)
    cfg = SchedulerConfig(slots_n=64, r=0.25, tau_pre=5e-5, tau_global=2e-4, policy=policy)
    pool = RealtimePool(GpuBackend(idx, cache, slots=64), cfg, tpot=1e-4, prefill_chunk=chunk)
    trace = gen_trace(spec)
    res = pool.run(trace, keep_results=True)
    pct = res.percentiles()
    assert pct["prefill"]["n"] == 200 and pct["decode"]["n"] == 400 and pct["cache"]["n"] == 200
    for st in pct.values():
        assert 0 < st["p50_ms"] <= st["p95_ms"] <= st["p99_ms"]
    for r in trace[::9]:
        for j in range(r.queries.shape[0]):
            k, npb = (100, 64) if j == 0 else (10, 16)
            oi, _ = orc.ivf_search(data, art, r.queries[j], k, npb)
            assert np.array_equal(res.results[(r.id, j)][:oi.size], oi)
        ci, _ = orc.exact_knn(cdata, r.queries[0], 1)
        assert np.array_equal(res.results[(r.id, "cache")], ci)
