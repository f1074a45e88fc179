"""Stage-aware scheduled retrieval trace (BASELINE.json config C5).

Replaces the reference's modeled pool step (cluster_sim.py:399-410,
``batches * extend_time * contention``) with real searches: a discrete-event
loop over a ``gen_trace`` workload (workload.py:118-151) in which

* each request issues one prefill retrieval at arrival (IVF, k=100,
  nprobe=64), one prompt-cache lookup (k=1 exact search on a separate cache
  store) and one decode probe every ``delta`` generated tokens after its
  prefill completes (IVF, k=10, nprobe=16);
* the ``TwoQueueScheduler`` (scheduler.py mirror, reference policy or
  ``decode_priority``) decides when to launch and which entries ride in each
  ragged batch; the batch runs on the GPU and the simulated clock advances by
  its MEASURED device time (CUDA events), which is also fed back through
  ``record_extend_latency``;
* latency = completion - enqueue, reported per stage as p50/p95/p99.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np

from .scheduler import QueueEntry, SchedulerConfig, TwoQueueScheduler
from .workload import WorkloadSpec, gen_trace

STAGE_KNP = {"prefill": (100, 64), "decode": (10, 16)}


@dataclass
class TraceResult:
    latencies: dict = field(default_factory=lambda: {"prefill": [], "decode": [], "cache": []})
    batches: int = 0
    gpu_ms: float = 0.0
    sim_seconds: float = 0.0
    retrievals: int = 0
    results: dict = field(default_factory=dict)  # (request, probe) -> ids (for parity sampling)

    def percentiles(self) -> dict:
        out = {}
        for stage, v in self.latencies.items():
            if v:
                a = np.asarray(v) * 1e3
                out[stage] = {"n": int(a.size), "p50_ms": float(np.percentile(a, 50)),
                              "p95_ms": float(np.percentile(a, 95)), "p99_ms": float(np.percentile(a, 99))}
        return out


class _Timer:
    def __init__(self):
        import torch

        self.torch = torch
        self.stream = torch.cuda.Stream()
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e1 = torch.cuda.Event(enable_timing=True)

    def run(self, fn):
        with self.torch.cuda.stream(self.stream):
            self.e0.record(self.stream)
            out = fn(self.stream)
            self.e1.record(self.stream)
        self.e1.synchronize()
        return out, self.e0.elapsed_time(self.e1) / 1e3


def run_trace(index, cache_store, spec: WorkloadSpec, sched: SchedulerConfig, tpot: float = 0.02,
              l_pre_max: float = 2e-3, keep_results: bool = False) -> TraceResult:
    """Drive ``spec``'s trace through the scheduler and the GPU; see module doc."""
    import torch

    trace = gen_trace(spec)
    sch = TwoQueueScheduler(sched)
    timer = _Timer()
    res = TraceResult()
    events = []  # (time, seq, kind, payload)
    seq = 0
    for r in trace:
        events.append((r.arrival_time, seq, "arrive", r))
        seq += 1
    heapq.heapify(events)
    cache_pending = []
    t = 0.0
    dev_q = torch.empty((sched.slots_n, index.dim), dtype=torch.float64, device="cuda")
    dev_ids = torch.empty((sched.slots_n, 100), dtype=torch.int64, device="cuda")
    dev_d = torch.empty((sched.slots_n, 100), dtype=torch.float64, device="cuda")

    def admit_until(now):
        while events and events[0][0] <= now:
            te, _, kind, obj = heapq.heappop(events)
            if kind == "arrive":
                sch.enqueue(QueueEntry(request_id=obj.id, stage="prefill", t_arrival=te, deadline=te + l_pre_max,
                                       est_remaining_extends=1.0, payload=(obj, 0)))
                cache_pending.append((te, obj))
            else:  # decode probe j of a request
                req, j = obj
                sch.enqueue(QueueEntry(request_id=req.id, stage="decode", t_arrival=te, payload=(req, j)))

    while events or sch.backlog() or cache_pending:
        admit_until(t)
        if not sch.backlog() and not cache_pending:
            t = events[0][0]
            continue
        if cache_pending:  # prompt-cache lookups: one exact k=1 launch for all waiting
            qs = np.stack([o.queries[0] for _, o in cache_pending]).astype(np.float64)
            (ids, _), dt = timer.run(lambda st: cache_store.device().knn(qs, np.ones(len(qs), np.int32)))
            t += dt
            res.gpu_ms += dt * 1e3
            for te, _ in cache_pending:
                res.latencies["cache"].append(t - te)
            cache_pending = []
            res.batches += 1
        if not sch.backlog():
            continue
        if not sch.should_launch(t) and events:
            # next instant anything can change: an arrival, the oldest prefill
            # aging past tau_pre, or the oldest entry reaching tau_global
            cands = [events[0][0], min(e.t_arrival for e in sch.q_pre + list(sch.q_dec)) + sched.tau_global]
            if sch.q_pre:
                cands.append(min(e.t_arrival for e in sch.q_pre) + sch.tau_pre)
            later = [c for c in cands if c > t]
            if later:
                t = min(later)
                continue
        # launch (timeouts reached, buffer full, or nothing else can happen)
        plan = sch.preempt(sch.build_batch(t), t)
        entries = plan.picked_prefill + plan.picked_decode
        if not entries:
            continue
        B = len(entries)
        qs = np.stack([e.payload[0].queries[e.payload[1]] for e in entries]).astype(np.float64)
        ks = [STAGE_KNP[e.stage][0] for e in entries]
        nps = [STAGE_KNP[e.stage][1] for e in entries]
        dev_q[:B].copy_(torch.from_numpy(qs))

        def launch(st):
            index.search_device(dev_q[:B], ks, nps, dev_ids[:B], dev_d[:B], st)

        _, dt = timer.run(launch)
        t += dt
        res.gpu_ms += dt * 1e3
        res.batches += 1
        res.retrievals += B
        sch.record_extend_latency(dt)
        ids_host = dev_ids[:B].cpu().numpy() if keep_results else None
        for i, e in enumerate(entries):
            res.latencies[e.stage].append(t - e.t_arrival)
            obj, j = e.payload
            if keep_results:
                res.results[(obj.id, j)] = ids_host[i, : ks[i]].copy()
            if e.stage == "prefill":
                for jj in range(1, obj.queries.shape[0]):
                    heapq.heappush(events, (t + jj * obj.probe_interval * tpot, seq, "probe", (obj, jj)))
                    seq += 1
    res.sim_seconds = t
    return res
