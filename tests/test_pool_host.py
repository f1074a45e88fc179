"""Real-time pool driver (pool.py) on the CPU with a stand-in backend.

The loop itself (producer thread, single-owner stepper, scheduler policies,
decode probes released after their prefill, prefill chunking with in-flight
preemption, cache lookups through the scheduler) is backend-agnostic; a
backend that sleeps a fixed time per call checks its accounting and timing
without a GPU.
"""

import time

import numpy as np
import pytest

from paper_2512_02281_b200.pool import RealtimePool
from paper_2512_02281_b200.scheduler import SchedulerConfig
from paper_2512_02281_b200.workload import WorkloadSpec, gen_trace


class SleepBackend:
    def __init__(self, per_call=2e-4, per_query=2e-6):
        self.per_call, self.per_query = per_call, per_query
        self.calls = []

    def search(self, qs, ks, nps):
        self.calls.append(("ivf", len(qs), sorted(set(ks.tolist()))))
        time.sleep(self.per_call + self.per_query * len(qs))
        return np.zeros((len(qs), int(ks.max())), np.int64)

    def cache(self, qs):
        self.calls.append(("cache", len(qs), [1]))
        time.sleep(self.per_call)
        return np.zeros((len(qs), 1), np.int64)


def _trace(n=300, rate=5000.0):
    return gen_trace(WorkloadSpec(n_db=1000, dim=8, n_requests=n, arrival_rate=rate, seed=7))


@pytest.mark.parametrize("policy", ["prefill_reserved", "decode_priority"])
def test_pool_serves_every_entry_in_real_time(policy):
    tr = _trace()
    be = SleepBackend()
    pool = RealtimePool(be, SchedulerConfig(slots_n=64, r=0.25, tau_pre=2e-4, tau_global=1e-3, policy=policy),
                        tpot=1e-4)
    res = pool.run(tr)
    n_dec = sum(r.queries.shape[0] - 1 for r in tr)
    assert len(res.latencies["prefill"]) == len(tr) and len(res.latencies["cache"]) == len(tr)
    assert len(res.latencies["decode"]) == n_dec
    assert res.retrievals == 2 * len(tr) + n_dec
    lat = np.concatenate([np.asarray(v) for v in res.latencies.values()])
    assert (lat > 0).all()  # results come back after their release time
    # the trace spans len/rate seconds of arrivals; the run cannot finish before
    assert res.wall_s >= tr[-1].arrival_time
    assert res.busy_s <= res.wall_s
    # every IVF launch carries at most slots_n entries
    assert max(c[1] for c in be.calls) <= 64


def test_decode_probes_wait_for_their_prefill():
    tr = _trace(n=40, rate=2000.0)
    tpot = 2e-3
    pool = RealtimePool(SleepBackend(), SchedulerConfig(slots_n=64, tau_pre=2e-4, tau_global=1e-3), tpot=tpot)
    res = pool.run(tr, keep_results=True)
    # each request's decode probes are released probe_interval * tpot after its prefill returned
    assert {(r.id, j) for r in tr for j in range(r.queries.shape[0])} <= set(res.results)
    assert res.wall_s >= tr[-1].arrival_time + (tr[-1].queries.shape[0] - 1) * tr[-1].probe_interval * tpot


def test_prefill_chunks_yield_to_waiting_decode():
    tr = _trace(n=400, rate=40000.0)  # a burst: many prefill entries per batch
    be = SleepBackend(per_call=5e-4)
    cfg = SchedulerConfig(slots_n=256, r=0.25, tau_pre=2e-4, tau_global=1e-3, policy="decode_priority")
    res = RealtimePool(be, cfg, tpot=1e-4, prefill_chunk=16).run(tr)
    assert res.launches > res.batches  # prefill batches ran in chunks
    assert res.preemptions > 0  # and decode / cache work ran between chunks
    assert all(c[1] <= 256 for c in be.calls)
    with pytest.raises(ValueError):
        RealtimePool(be, cfg, prefill_chunk=0)
