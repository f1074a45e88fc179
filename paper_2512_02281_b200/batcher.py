"""Continuous batching of heterogeneous retrievals over one IVF index (config C3).

Prefill retrievals (large k, large nprobe), decode probes (small k, small
nprobe) and prompt-cache lookups share ONE device launch sequence per step:
``tri_ivf_search`` takes a per-query k and nprobe, the device packer turns the
ragged probe sets into list-major work items, and no query is padded to the
largest request (the reference pads fixed-shape *slots*, engine.py:208-226;
here only the candidate capacity is rounded, per query).

The batcher is host-side and single-owner like the reference's engine
(engine.py:313-319): ``submit`` appends, ``step`` drains up to ``max_batch``
pending queries in arrival order, runs them, and returns the finished ones.
"""

from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass

import numpy as np

from .ivf import IVFFlatIndex

STAGE_PARAMS = {"prefill": (100, 64), "decode": (10, 16)}


@dataclass(frozen=True)
class Retrieval:
    request_id: int
    stage: str
    ids: np.ndarray
    dists: np.ndarray
    t_submit: float
    t_done: float

    @property
    def latency(self) -> float:
        return self.t_done - self.t_submit


@dataclass
class _Pending:
    rid: int
    query: np.ndarray
    k: int
    nprobe: int
    stage: str
    t_submit: float


class RetrievalBatcher:
    """Ragged continuous batcher: one fused device launch sequence per step."""

    def __init__(self, index: IVFFlatIndex, max_batch: int = 256, clock=time.perf_counter):
        self.index = index
        self.max_batch = max_batch
        self.clock = clock
        self._queue: deque = deque()
        self._next = 0
        self.steps = 0

    def submit(self, query, k: int | None = None, nprobe: int | None = None, stage: str = "decode",
               t_submit: float | None = None) -> int:
        # validated here, so one bad submission cannot fail a whole batch in step()
        dk, dnp = STAGE_PARAMS.get(stage, (10, 16))
        q = np.asarray(query, dtype=np.float64).ravel()
        if q.shape[0] != self.index.dim:
            raise ValueError(f"query dim {q.shape[0]} != index dim {self.index.dim}")
        if not np.isfinite(q).all():
            raise ValueError("query must be finite")
        k = dk if k is None else int(k)
        nprobe = dnp if nprobe is None else int(nprobe)
        if k < 1:
            raise ValueError(f"k must be >= 1, got {k}")
        if not 1 <= nprobe <= self.index.nlist:
            raise ValueError(f"nprobe must be in [1, {self.index.nlist}], got {nprobe}")
        rid = self._next
        self._next += 1
        self._queue.append(_Pending(rid, q, k, nprobe, stage, self.clock() if t_submit is None else t_submit))
        return rid

    @property
    def pending(self) -> int:
        return len(self._queue)

    def step(self) -> list:
        if not self._queue:
            return []
        take = [self._queue.popleft() for _ in range(min(self.max_batch, len(self._queue)))]
        qs = np.stack([p.query for p in take])
        ks = np.array([p.k for p in take])
        nps = np.array([p.nprobe for p in take])
        ids, dists = self.index.search(qs, ks, nps)
        t = self.clock()
        self.steps += 1
        return [Retrieval(p.rid, p.stage, ids[i, : p.k].copy(), dists[i, : p.k].copy(), p.t_submit, t)
                for i, p in enumerate(take)]

    def run_to_completion(self) -> list:
        out = []
        while self._queue:
            out.extend(self.step())
        return out
