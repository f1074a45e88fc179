"""Real-time driver of the shared vector-search pool (BASELINE.json config C5).

Replaces the reference's modeled pool step (cluster_sim.py:399-410, where a
pool batch costs ``batches * extend_time * contention`` on a simulated clock)
with searches served on the wall clock:

* a **producer thread** releases each request at its trace arrival time
  (``gen_trace``, workload.py:118-151): one prefill retrieval (IVF, k=100,
  nprobe=64) and one prompt-cache lookup (k=1 exact search on the cache
  store), and later the request's decode probes (IVF, k=10, nprobe=16), due
  ``j * probe_interval * tpot`` seconds after its prefill result came back;
* the **stepper** (the caller's thread, the single owner of the scheduler, as
  the reference's SPEC.md:308 prescribes) drains the inbox at every step,
  asks the ``TwoQueueScheduler`` (scheduler.py:206-248 mirror; reference
  policy or ``decode_priority``) whether and what to launch, runs the batch
  through the backend -- prefill and decode entries as one ragged IVF
  search, cache entries as one k=1 search -- and feeds the batch's measured
  wall time to ``record_extend_latency``;
* **in-flight prefill preemption** (``prefill_chunk``): a batch's prefill
  entries run in chunks; between chunks the stepper drains the inbox and, when
  decode or cache entries are waiting, serves them first (decode_priority);
* latency = host time the result is back - the entry's scheduled release
  time, per stage, so time the stepper spent busy before noticing an arrival
  counts against the pool.

The backend is injected (``search(queries, ks, nprobes)`` and
``cache(queries)``, both blocking): ``GpuBackend`` calls the library through
pinned host buffers; the CPU reference loop (bench's C5 ``cpu_baseline``) plugs
the numpy oracle in from outside the package.
"""

from __future__ import annotations

import gc
import heapq
import threading
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .scheduler import CACHE, DECODE, PREFILL, QueueEntry, SchedulerConfig, TwoQueueScheduler

STAGE_KNP = {PREFILL: (100, 64), DECODE: (10, 16)}


@dataclass
class PoolResult:
    latencies: dict = field(default_factory=lambda: {PREFILL: [], DECODE: [], CACHE: []})
    batches: int = 0          # scheduler launches
    launches: int = 0         # backend calls (chunks and cache searches included)
    preemptions: int = 0      # prefill chunks that yielded to waiting decode / cache entries
    retrievals: int = 0
    busy_s: float = 0.0       # wall time inside backend calls
    wall_s: float = 0.0
    results: dict = field(default_factory=dict)  # (request, probe) -> ids, when keep_results

    def percentiles(self) -> dict:
        out = {}
        for stage, v in self.latencies.items():
            if v:
                a = np.asarray(v) * 1e3
                out[stage] = {"n": int(a.size), "p50_ms": float(np.percentile(a, 50)),
                              "p95_ms": float(np.percentile(a, 95)), "p99_ms": float(np.percentile(a, 99))}
        return out


class GpuBackend:
    """Blocking searches on one CUDA stream through pinned host buffers."""

    def __init__(self, index, cache_store, slots: int, stream=None, kmax: int = 100):
        import torch

        self.index = index
        self.cache_store = cache_store.device() if hasattr(cache_store, "device") and callable(
            getattr(cache_store, "device")) else cache_store
        self.stream = stream or torch.cuda.Stream()
        d = index.dim
        self.q = torch.empty((slots, d), dtype=torch.float64).pin_memory()
        self.ids = torch.empty((slots, kmax), dtype=torch.int64).pin_memory()
        self.dists = torch.empty((slots, kmax), dtype=torch.float64).pin_memory()
        self.cq = torch.empty((slots, self.cache_store.d), dtype=torch.float64).pin_memory()
        self.cids = torch.empty((slots, 1), dtype=torch.int64).pin_memory()
        self.cd = torch.empty((slots, 1), dtype=torch.float64).pin_memory()
        self.ones = np.ones(slots, dtype=np.int32)
        self.kmax = kmax
        self._s2 = None  # second stream for the cache lookups (search_and_cache), made on first use

    def search(self, queries: np.ndarray, ks, nps) -> np.ndarray:
        B = queries.shape[0]
        self.q.numpy()[:B] = queries
        self.index.search_into(self.q[:B], ks, nps, self.ids[:B], self.dists[:B], stream=self.stream)
        return self.ids.numpy()[:B]

    def cache(self, queries: np.ndarray) -> np.ndarray:
        B = queries.shape[0]
        self.cq.numpy()[:B] = queries
        self.cache_store.knn_into(self.cq[:B], self.ones[:B], self.cids[:B], self.cd[:B], stream=self.stream)
        return self.cids.numpy()[:B]

    def search_and_cache(self, queries: np.ndarray, ks, nps, cqueries: np.ndarray):
        """One batch's IVF search and prompt-cache lookups side by side: the
        lookups are enqueued on a second stream (H2D, exact kNN on the device
        store, D2H), the IVF search runs blocking on the first, then the second
        is awaited -- the batch takes the longer of the two, not their sum."""
        import torch

        from . import _lib

        if self._s2 is None:
            self._s2 = torch.cuda.Stream()
            n, d = self.cq.shape
            self._cq_dev = torch.empty((n, d), dtype=torch.float64, device="cuda")
            self._cids_dev = torch.empty((n, 1), dtype=torch.int64, device="cuda")
            self._cd_dev = torch.empty((n, 1), dtype=torch.float64, device="cuda")
            self._ev = torch.cuda.Event()
        Bc = cqueries.shape[0]
        self.cq.numpy()[:Bc] = cqueries
        with torch.cuda.stream(self._s2):
            self._cq_dev[:Bc].copy_(self.cq[:Bc], non_blocking=True)
            _lib.check(_lib.gpu().tri_knn_bruteforce_dev(
                self.cache_store.handle, _lib.ptr(self._cq_dev), Bc, self.ones.ctypes.data, 1,
                _lib.ptr(self._cids_dev), _lib.ptr(self._cd_dev), _lib.C.c_void_p(self._s2.cuda_stream)))
            self.cids[:Bc].copy_(self._cids_dev[:Bc], non_blocking=True)
            self._ev.record(self._s2)
        ids = self.search(queries, ks, nps)
        self._ev.synchronize()
        return ids, self.cids.numpy()[:Bc]


class RealtimePool:
    """Wall-clock serving loop: producer thread + single-owner stepper (see module doc)."""

    def __init__(self, backend, sched: SchedulerConfig, tpot: float = 5e-3, l_pre_max: float = 2e-3,
                 prefill_chunk: int | None = None, stage_knp: dict | None = None):
        if prefill_chunk is not None and prefill_chunk < 1:
            raise ValueError("prefill_chunk must be >= 1")
        self.backend = backend
        self.sched_cfg = sched
        self.tpot = tpot
        self.l_pre_max = l_pre_max
        self.prefill_chunk = prefill_chunk
        self.stage_knp = stage_knp or STAGE_KNP

    # -- producer ------------------------------------------------------------
    def _producer(self):
        """Release every entry whose time has come (all of them at once), then
        sleep until the next one is due or a new one is scheduled."""
        with self._cv:
            while not self._stop:
                now = self._clock()
                moved = False
                while self._due and self._due[0][0] <= now:
                    self._inbox.append(heapq.heappop(self._due)[2])
                    moved = True
                if moved:
                    self._cv.notify_all()
                wait = self._due[0][0] - now if self._due else 0.05
                self._cv.wait(min(max(wait, 0.0), 0.05))

    def _schedule(self, t_due: float, entry: QueueEntry) -> None:
        with self._cv:
            heapq.heappush(self._due, (t_due, self._seq, entry))
            self._seq += 1
            self._cv.notify_all()

    # -- stepper --------------------------------------------------------------
    def _drain(self, sch: TwoQueueScheduler) -> None:
        while self._inbox:
            sch.enqueue(self._inbox.popleft())

    def _launch(self, sch, entries, res: PoolResult, keep: bool) -> None:
        ivf = [e for e in entries if e.stage != CACHE]
        cch = [e for e in entries if e.stage == CACHE]
        t0 = time.perf_counter()
        if ivf:
            qs = np.stack([e.payload[0].queries[e.payload[1]] for e in ivf]).astype(np.float64)
            ks = np.array([self.stage_knp[e.stage][0] for e in ivf], np.int32)
            nps = np.array([self.stage_knp[e.stage][1] for e in ivf], np.int32)
        if cch:
            cq = np.stack([e.payload[0].queries[0] for e in cch]).astype(np.float64)
        if ivf and cch and hasattr(self.backend, "search_and_cache"):
            ids, cids = self.backend.search_and_cache(qs, ks, nps, cq)  # both on the device at once
            res.launches += 2
        else:
            if ivf:
                ids = self.backend.search(qs, ks, nps)
                res.launches += 1
            if cch:
                cids = self.backend.cache(cq)
                res.launches += 1
        t_done = self._clock()
        dt = time.perf_counter() - t0
        res.busy_s += dt
        sch.record_extend_latency(max(dt, 1e-9))
        for i, e in enumerate(ivf):
            res.latencies[e.stage].append(t_done - e.t_arrival)
            req, j = e.payload
            if keep:
                res.results[(req.id, j)] = ids[i, : self.stage_knp[e.stage][0]].copy()
            if e.stage == PREFILL:  # the request's decode probes become due as it generates
                for jj in range(1, req.queries.shape[0]):
                    self._schedule(t_done + jj * req.probe_interval * self.tpot,
                                   QueueEntry(request_id=req.id, stage=DECODE,
                                              t_arrival=t_done + jj * req.probe_interval * self.tpot,
                                              payload=(req, jj)))
        for i, e in enumerate(cch):
            res.latencies[CACHE].append(t_done - e.t_arrival)
            if keep:
                res.results[(e.payload[0].id, "cache")] = cids[i, :1].copy()
        res.retrievals += len(entries)

    def _execute(self, sch, plan, res: PoolResult, keep: bool) -> None:
        pre, dec = plan.picked_prefill, plan.picked_decode
        res.batches += 1
        chunk = self.prefill_chunk
        if not chunk or len(pre) <= chunk:
            self._launch(sch, pre + dec, res, keep)
            return
        # in-flight preemption: the first chunk rides with the batch's decode
        # entries; before every later chunk, decode / cache entries that
        # arrived meanwhile are served first
        self._launch(sch, pre[:chunk] + dec, res, keep)
        for s in range(chunk, len(pre), chunk):
            self._drain(sch)
            if sch.config.policy == "decode_priority" and sch.q_dec:
                urgent = sch.pop_decode(sch.config.slots_n)
                self._launch(sch, urgent, res, keep)
                res.preemptions += 1
            self._launch(sch, pre[s:s + chunk], res, keep)

    def run(self, trace: list, keep_results: bool = False, time_scale: float = 1.0) -> PoolResult:
        """Serve ``trace`` (``gen_trace`` requests) in real time; returns latencies."""
        sch = TwoQueueScheduler(self.sched_cfg)
        res = PoolResult()
        self._cv = threading.Condition()
        self._due = []
        self._seq = 0
        self._inbox = deque()
        self._stop = False
        expected = sum(2 + r.queries.shape[0] - 1 for r in trace)  # prefill + cache + decode probes
        # the whole arrival schedule is built before the clock starts (pushing
        # it entry by entry would eat into the first arrivals' latency)
        for r in trace:
            ta = r.arrival_time * time_scale
            self._due.append((ta, self._seq, QueueEntry(request_id=r.id, stage=PREFILL, t_arrival=ta,
                                                        deadline=ta + self.l_pre_max, est_remaining_extends=1.0,
                                                        payload=(r, 0))))
            self._due.append((ta, self._seq + 1, QueueEntry(request_id=r.id, stage=CACHE, t_arrival=ta,
                                                            payload=(r, 0))))
            self._seq += 2
        heapq.heapify(self._due)
        # no cyclic-GC pauses inside the timed loop (the loop allocates steadily)
        gc_was = gc.isenabled()
        gc.collect()
        gc.disable()
        t_start = time.perf_counter()
        self._clock = lambda: time.perf_counter() - t_start
        prod = threading.Thread(target=self._producer, daemon=True)
        prod.start()
        try:
            while True:
                self._drain(sch)
                now = self._clock()
                if sch.backlog() and sch.should_launch(now):
                    self._execute(sch, sch.preempt(sch.build_batch(now), now), res, keep_results)
                    continue
                if res.retrievals >= expected:
                    break
                with self._cv:
                    if not self._inbox:
                        # sleep until an arrival or the next launch timeout
                        wake = 0.01
                        if sch.backlog():
                            oldest = min([e.t_arrival for e in sch.q_pre] + [e.t_arrival for e in sch.q_dec])
                            nxt = oldest + sch.config.tau_global
                            if sch.q_pre:
                                nxt = min(nxt, min(e.t_arrival for e in sch.q_pre) + sch.tau_pre)
                            wake = max(0.0, min(wake, nxt - now))
                        if wake > 0:
                            self._cv.wait(wake)
        finally:
            with self._cv:
                self._stop = True
                self._cv.notify_all()
            prod.join()
            if gc_was:
                gc.enable()
        res.wall_s = self._clock()
        return res
