"""Full-batch oracle parity at BASELINE sizes: the numpy oracle (oracle/) for
every query of a batch, fanned out over the host cores.  Test infrastructure
(tests/ and bench.py's untimed parity checks), like the rest of oracle/.

The oracle costs about 0.2 s per C2 query on one core, so a whole 256-query
batch takes seconds on a process pool.  Workers are forked and read the
database copy-on-write; they only run numpy (no CUDA, no BLAS)."""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_STATE = None


def _one(i):
    from oracle import trinity_oracle as orc

    data, art, qs, ks, nps = _STATE
    return orc.ivf_search(data, art, qs[i], int(ks[i]), int(nps[i]))


def ivf_oracle_batch(data, art, qs, ks, nps, procs: int | None = None):
    """[(ids, dists)] of orc.ivf_search for every row of qs (per-row k / nprobe)."""
    global _STATE
    B = qs.shape[0]
    ks = np.broadcast_to(np.asarray(ks), (B,))
    nps = np.broadcast_to(np.asarray(nps), (B,))
    _STATE = (data, art, qs, ks, nps)
    procs = procs or min(B, os.cpu_count() or 1)
    try:
        if procs <= 1:
            return [_one(i) for i in range(B)]
        with mp.get_context("fork").Pool(procs) as pool:
            return pool.map(_one, range(B), chunksize=1)
    finally:
        _STATE = None


def assert_rows_equal(ids, d, ref, ks=None):
    """Every row equals the oracle: ids and float64 distances bit-exact, -1 past the results."""
    for i, (oi, od) in enumerate(ref):
        n = oi.size
        assert np.array_equal(ids[i, :n], oi), f"ids differ on query {i}"
        assert np.array_equal(d[i, :n], od), f"distances differ on query {i}"
        if ks is not None:
            assert (ids[i, n:int(np.broadcast_to(ks, (len(ref),))[i])] == -1).all()
