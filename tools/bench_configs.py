"""Secondary BASELINE.json configurations, measured beside the bench headline.

bench.py (N=1, rank 0) calls these after its own timed region.  Each returns a
complete record -- ``value`` (device-resident throughput), ``roofline``,
``cpu_baseline`` (the numpy oracle on one core, bounded sample), ``e2e``
(through the public host API, copies inside the timed region) and ``parity``
(against the oracle or the reference-generated golden vectors).  ``compact``
keeps the headline numbers of a record for bench's one JSON line; the full
record goes to ``--full-out``.

* c1  brute-force exact kNN, 100K x 128 fp32, B=64, k=10 (BASELINE config 1)
* c3  continuous batching of heterogeneous retrievals over the C2 index:
      prefill (k=100, nprobe=64) and decode (k=10, nprobe=16) probes of a
      ``gen_trace`` workload, ragged batches of 256 in arrival order
* c5  stage-aware scheduled trace (RAG retrievals + prompt-cache lookups)
      on the wall clock (paper_2512_02281_b200/pool.py)
* engine  graph search engine (tools/bench_engine.py)
"""

from __future__ import annotations

import os
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = "queries/s"


def _pct(a):
    a = np.asarray(a, dtype=np.float64)
    return {"p50_ms": float(np.percentile(a, 50)), "p95_ms": float(np.percentile(a, 95)),
            "p99_ms": float(np.percentile(a, 99))}


def _r(x, n=4):
    return None if x is None else float(f"{x:.{n}g}")


def compact(r: dict) -> dict:
    """The headline numbers of a config record (bench's line keeps these)."""
    if "error" in r:
        return {"error": r["error"][:160]}
    out = {"value": _r(r.get("value")), "unit": r.get("unit", UNIT)}
    if r.get("ms_per_step") is not None:
        out["ms_per_step"] = _r(r["ms_per_step"])
    rf = r.get("roofline")
    if rf:
        out["roofline"] = {"bound": rf.get("bound"), "frac": _r(rf.get("frac"), 3)}
        if rf.get("tensor_frac") is not None:
            out["roofline"]["tensor_frac"] = _r(rf["tensor_frac"], 3)
    cb = r.get("cpu_baseline")
    if cb:
        out["cpu_baseline"] = {"value": _r(cb["value"]), "cores": cb["cores"]}
    e = r.get("e2e")
    if e:
        out["e2e"] = _r(e["value"])
    if r.get("latency_ms"):
        out["p99_ms"] = {s: _r(v["p99_ms"], 3) for s, v in r["latency_ms"].items()}
    if r.get("parity"):
        out["parity"] = r["parity"].split(":")[0]
    return out


# ----------------------------------------------------------------------------
# C1


def c1(peak_gbs: float, steps: int = 200, cpu_sample: int = 16, lanes: int = 4) -> dict:
    """Brute force 100K x 128, 64 queries, k=10 (store L2-resident: 51 MB)."""
    import ctypes as C

    import torch

    from oracle import trinity_oracle as orc
    from paper_2512_02281_b200 import _lib
    from paper_2512_02281_b200.ann_graph import VectorStore, _DeviceStore, brute_force_knn_batch
    from paper_2512_02281_b200.workload import gen_matrix

    N, D, B, K = 100_000, 128, 64, 10
    g = np.load(os.path.join(ROOT, "tests", "golden", "bf_c1.npz"))
    data = gen_matrix(N, D, 1)
    qs = gen_matrix(B, D, 2).astype(np.float64)
    store = _DeviceStore(data)
    lib = _lib.gpu()
    q = torch.from_numpy(qs).cuda()
    ks = np.full(B, K, np.int32)
    L = lanes  # batches in flight (one stream + library workspace each), as C2
    ids = [torch.empty((B, K), dtype=torch.int64, device="cuda") for _ in range(L)]
    d = [torch.empty((B, K), dtype=torch.float64, device="cuda") for _ in range(L)]
    sts = [torch.cuda.Stream() for _ in range(L)]
    st = sts[0]

    def one(j=0):
        _lib.check(lib.tri_knn_bruteforce_dev(store.handle, _lib.ptr(q), B, ks.ctypes.data, K, _lib.ptr(ids[j]),
                                              _lib.ptr(d[j]), C.c_void_p(sts[j].cuda_stream)))

    for i in range(50):  # the first tens of batches after a store's creation run slower
        one(i % L)
    torch.cuda.synchronize()
    ok = all(np.array_equal(ids[j].cpu().numpy(), g["ids"]) and np.array_equal(d[j].cpu().numpy(), g["dists"])
             for j in range(L))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)  # one stream: the per-batch latency
    for _ in range(steps):
        one()
    e1.record(st)
    e1.synchronize()
    lat_ms = e0.elapsed_time(e1) / steps
    e0.record(st)  # L lanes: throughput
    for ls in sts[1:]:
        ls.wait_event(e0)
    for i in range(steps):
        one(i % L)
    for ls in sts[1:]:
        st.wait_stream(ls)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    fixups = store.last_fixups()
    store.close()
    # e2e: host queries in, host results out.  (a) the reference-shaped batch
    # call, one at a time (pageable numpy); (b) knn_into on pinned buffers, one
    # host thread per lane (4 lanes), as the C2 / C3 e2e figures are taken
    vs = VectorStore(data=data)
    for _ in range(5):
        brute_force_knn_batch(vs, qs, K)
    n_e2e = 100
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        brute_force_knn_batch(vs, qs, K)
    single_ms = (time.perf_counter() - t0) * 1e3 / n_e2e
    dev = vs.device()
    # (lanes: the host threads, one per device lane)
    qp = torch.from_numpy(qs).pin_memory()
    outs = [(torch.empty((B, K), dtype=torch.int64).pin_memory(), torch.empty((B, K), dtype=torch.float64).pin_memory())
            for _ in range(lanes)]
    sts = [torch.cuda.Stream() for _ in range(lanes)]
    gate = threading.Barrier(lanes + 1)
    t_end = [0.0] * lanes

    def lane_loop(j):
        for _ in range(5):
            dev.knn_into(qp, K, *outs[j], stream=sts[j])
        gate.wait()
        for _ in range(n_e2e):
            dev.knn_into(qp, K, *outs[j], stream=sts[j])
        t_end[j] = time.perf_counter()

    ths = [threading.Thread(target=lane_loop, args=(j,)) for j in range(lanes)]
    for th in ths:
        th.start()
    gate.wait()
    te0 = time.perf_counter()
    for th in ths:
        th.join()
    e2e_ms = (max(t_end) - te0) * 1e3 / (lanes * n_e2e)
    ok = ok and np.array_equal(outs[0][0].numpy(), g["ids"]) and np.array_equal(outs[0][1].numpy(), g["dists"])
    # CPU: the reference's brute_force_knn (restated by the oracle), one query at a time
    t0 = time.perf_counter()
    for i in range(cpu_sample):
        orc.exact_knn(data, qs[i], K)
    cpu_s = time.perf_counter() - t0
    store_bytes = N * (D * 4 + 4)
    flops = 2.0 * B * N * D
    tf32_peak = _tf32_peak_tflops()
    return {
        "workload": "C1: brute-force exact kNN, gen_vectors(100000,128,seed=1), 64 queries (seed=2), k=10",
        "value": B / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "lanes": L,
        "batch_latency_ms_one_stream": lat_ms,
        "roofline": {
            "bound": "hbm", "unit": "GB/s", "achieved": store_bytes / (ms / 1e3) / 1e9, "peak": peak_gbs,
            "frac": store_bytes / (ms / 1e3) / 1e9 / peak_gbs, "algorithmic_bytes_per_launch": store_bytes,
            "tensor_tflops": flops / (ms / 1e3) / 1e12, "tensor_peak_tflops": tf32_peak,
            "tensor_frac": flops / (ms / 1e3) / 1e12 / tf32_peak,
            "note": "bytes / step time with 4 batches in flight (TF32 tcgen05 scan + select + fp64 re-rank); "
                    "the 51.6 MB store stays L2-resident between batches, so HBM is not the binding limit; "
                    "tensor peak = TF32 = half the measured dense bf16 peak",
        },
        "cpu_baseline": {"value": cpu_sample / cpu_s, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"oracle exact_knn (ann_graph.py:124-137) on the first {cpu_sample} queries, "
                                   f"{cpu_s:.1f} s"},
        "e2e": {"value": B / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": B * D * 8,
                "d2h_bytes_per_step": B * K * 16,
                "api": "_DeviceStore.knn_into on pinned host buffers, one host thread per lane (4 lanes)",
                "single_call_qps": B / (single_ms / 1e3),
                "single_call_api": "brute_force_knn_batch(VectorStore, numpy queries), one call at a time"},
        "parity": f"{'ok' if ok else 'FAIL'}: 64 x 10 ids and f64 dists == reference golden (tests/golden/bf_c1.npz)",
        "fixups": fixups,
    }


def _tf32_peak_tflops() -> float:
    import json

    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        for key in ("bf16_tflops", "dense_bf16_tflops", "bf16_dense_tflops"):
            if key in p:
                return float(p[key]) / 2
    except Exception:
        pass
    return 1125.0


# ----------------------------------------------------------------------------
# C3


def c3_workload(n_db: int, dim: int, n_requests: int = 1200):
    """gen_trace(seed=7) retrievals in arrival order: (queries f64, stage, k, nprobe)."""
    from paper_2512_02281_b200.workload import WorkloadSpec, gen_trace

    spec = WorkloadSpec(n_db=n_db, dim=dim, n_requests=n_requests, arrival_rate=1e4, seed=7)
    items = []
    for r in gen_trace(spec):
        for j in range(r.queries.shape[0]):
            items.append((r.queries[j], "prefill" if j == 0 else "decode"))
    qs = np.stack([it[0] for it in items]).astype(np.float64)
    stage = np.array([it[1] for it in items])
    ks = np.where(stage == "prefill", 100, 10).astype(np.int32)
    nps = np.where(stage == "prefill", 64, 16).astype(np.int32)
    return qs, stage, ks, nps


def c3(b: dict, peak_gbs: float, batch: int = 256, lanes: int = 4, cpu_sample: int = 12) -> dict:
    """Ragged prefill/decode batches from a gen_trace workload over the C2 index.

    Consecutive batches go round-robin to ``lanes`` streams (the continuous
    pipeline a serving loop runs); ``value`` is the whole run's throughput,
    the per-class latency that of the batch carrying the retrieval."""
    import torch

    from oracle import trinity_oracle as orc
    from oracle.pool import ivf_oracle_batch

    idx, data = b["idx"], b["data"]
    art = orc.IVFArtifact(b["cen"], b["asg"])
    qs, stage, ks, nps = c3_workload(data.shape[0], data.shape[1])
    n = qs.shape[0]
    q_dev = torch.from_numpy(qs).cuda()
    ids = torch.empty((n, 100), dtype=torch.int64, device="cuda")
    d = torch.empty((n, 100), dtype=torch.float64, device="cuda")
    starts = list(range(0, n, batch))
    streams = [torch.cuda.Stream() for _ in range(lanes)]

    def run_all(times=None):
        for bi, s in enumerate(starts):
            st = streams[bi % lanes]
            e = min(n, s + batch)
            if times is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record(st)
            idx.search_device(q_dev[s:e], ks[s:e], nps[s:e], ids[s:e], d[s:e], st)
            if times is not None:
                ev[1].record(st)
                times.append(ev)

    # algorithmic scan bytes of every batch (one untimed pass, one stream)
    scan_bytes = 0
    for s in starts:
        e = min(n, s + batch)
        idx.search_device(q_dev[s:e], ks[s:e], nps[s:e], ids[s:e], d[s:e], streams[0])
        streams[0].synchronize()
        scan_bytes += idx.last_scan_bytes()[0]
    # the shapes of every lane captured and replayed, with the stage-timer event
    # nodes the timed pass uses (profiling is part of a graph's key)
    idx.set_profiling(True)
    for _ in range(2):
        run_all()
    torch.cuda.synchronize()
    idx.set_profiling(True)  # reset the timers
    times = []
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(streams[0])
    for st in streams[1:]:
        st.wait_event(t0)
    run_all(times)
    for st in streams[1:]:
        streams[0].wait_stream(st)
    t1.record(streams[0])
    t1.synchronize()
    scan_ms, scan_n = idx.scan_time()
    idx.set_profiling(False)
    total_ms = t0.elapsed_time(t1)
    lat = {"prefill": [], "decode": []}
    for bi, (a, bb) in enumerate(times):
        ms = a.elapsed_time(bb)
        for i in range(starts[bi], min(n, starts[bi] + batch)):
            lat[stage[i]].append(ms)
    # parity: every 25th retrieval (prefill and decode) against the oracle, on the host cores
    hid, hd = ids.cpu().numpy(), d.cpu().numpy()
    rows = list(range(0, n, 25))
    ref = ivf_oracle_batch(data, art, qs[rows], ks[rows], nps[rows])
    bad = sum(1 for j, i in enumerate(rows)
              if not (np.array_equal(hid[i, :ref[j][0].size], ref[j][0]) and
                      np.array_equal(hd[i, :ref[j][1].size], ref[j][1])))
    # e2e: the host API (pinned buffers), one host thread per lane
    q_pin = torch.from_numpy(qs).pin_memory()
    outs = [(torch.empty((batch, 100), dtype=torch.int64).pin_memory(),
             torch.empty((batch, 100), dtype=torch.float64).pin_memory()) for _ in range(lanes)]
    gate = threading.Barrier(lanes + 1)
    t_end = [0.0] * lanes

    def lane_loop(j):
        mine = starts[j::lanes]
        for s in mine:  # warm-up: one untimed pass over the lane's batches (every shape it will see)
            e = min(n, s + batch)
            idx.search_into(q_pin[s:e], ks[s:e], nps[s:e], outs[j][0][:e - s], outs[j][1][:e - s], stream=streams[j])
        gate.wait()
        for s in mine:
            e = min(n, s + batch)
            idx.search_into(q_pin[s:e], ks[s:e], nps[s:e], outs[j][0][:e - s], outs[j][1][:e - s], stream=streams[j])
        t_end[j] = time.perf_counter()

    ths = [threading.Thread(target=lane_loop, args=(j,)) for j in range(lanes)]
    for th in ths:
        th.start()
    gate.wait()
    te0 = time.perf_counter()
    for th in ths:
        th.join()
    e2e_s = max(t_end) - te0
    # CPU: the oracle per retrieval (its own k and nprobe), one core
    crow = [i for i in range(n) if stage[i] == "prefill"][: cpu_sample // 3] + \
           [i for i in range(n) if stage[i] == "decode"][: cpu_sample - cpu_sample // 3]
    tc0 = time.perf_counter()
    for i in crow:
        orc.ivf_search(data, art, qs[i], int(ks[i]), int(nps[i]))
    cpu_s = time.perf_counter() - tc0
    n_pre = int((stage == "prefill").sum())
    per_launch = scan_ms / max(scan_n, 1)
    bytes_per_launch = scan_bytes / len(starts)
    return {
        "workload": f"C3: gen_trace(seed=7) over the C2 index, {n} retrievals ({n_pre} prefill k=100 nprobe=64, "
                    f"{n - n_pre} decode k=10 nprobe=16), ragged batches of {batch} in arrival order, {lanes} lanes",
        "value": n / (total_ms / 1e3), "unit": UNIT, "ms_per_step": total_ms / len(starts), "batches": len(starts),
        "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": bytes_per_launch / (per_launch / 1e3) / 1e9,
                     "peak": peak_gbs, "frac": bytes_per_launch / (per_launch / 1e3) / 1e9 / peak_gbs,
                     "algorithmic_bytes_per_launch": bytes_per_launch, "scan_ms_per_launch": per_launch},
        "cpu_baseline": {"value": len(crow) / cpu_s, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"oracle ivf_search on {len(crow)} retrievals (1:2 prefill:decode), {cpu_s:.1f} s"},
        "e2e": {"value": n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": batch * (qs.shape[1] * 8 + 8),
                "d2h_bytes_per_step": batch * 100 * 16,
                "api": "IVFFlatIndex.search_into (pinned host buffers, per-query k / nprobe), one thread per lane"},
        "batch_latency_ms": {k: _pct(v) for k, v in lat.items()},
        "parity": f"{'ok' if not bad else 'FAIL'}: {len(rows)} retrievals (every 25th) == oracle (ids, f64 dists)",
    }


# ----------------------------------------------------------------------------
# C5


class OracleBackend:
    """The CPU reference in the pool's real-time loop: the numpy oracle
    (reference primitives) for IVF retrievals and cache lookups, each batch
    fanned out over a process pool of the host cores."""

    def __init__(self, data, art, cache_data, procs):
        import multiprocessing as mp

        global _ORC
        _ORC = (data, art, cache_data)
        self.pool = mp.get_context("fork").Pool(procs)

    def search(self, qs, ks, nps):
        res = self.pool.map(_orc_ivf, [(q, int(k), int(n)) for q, k, n in zip(qs, ks, nps)], chunksize=1)
        out = np.full((len(qs), int(np.max(ks))), -1, np.int64)
        for i, ids in enumerate(res):
            out[i, :ids.size] = ids
        return out

    def cache(self, qs):
        return np.stack(self.pool.map(_orc_cache, list(qs), chunksize=1))

    def close(self):
        self.pool.terminate()


_ORC = None


def _orc_ivf(a):
    from oracle import trinity_oracle as orc

    data, art, _ = _ORC
    return orc.ivf_search(data, art, a[0], a[1], a[2])[0]


def _orc_cache(q):
    from oracle import trinity_oracle as orc

    return orc.exact_knn(_ORC[2], q, 1)[0]


def c5(b: dict, peak_gbs: float, rates=(5_000.0, 10_000.0), seconds: float = 1.0, repeats: int = 3,
       cpu_rate: float = 10.0, cpu_requests: int = 40) -> dict:
    """Stage-aware scheduled trace on the wall clock (pool.py): RAG retrievals
    (prefill k=100 nprobe=64, decode k=10 nprobe=16) + one prompt-cache lookup
    per request, both scheduler policies at two arrival rates, latency from
    release to host result; the CPU reference runs in the same loop."""
    import torch

    from oracle import trinity_oracle as orc
    from paper_2512_02281_b200 import _lib
    from paper_2512_02281_b200.ann_graph import VectorStore
    from paper_2512_02281_b200.pool import GpuBackend, RealtimePool
    from paper_2512_02281_b200.scheduler import SchedulerConfig
    from paper_2512_02281_b200.workload import WorkloadSpec, gen_matrix, gen_trace

    idx = b["idx"]
    cdata = gen_matrix(10_000, idx.dim, 62)
    cache = VectorStore(data=cdata)
    tpot = 5e-3
    policies = {"prefill_reserved": None, "decode_priority": 64}  # policy -> prefill chunk (in-flight preemption)

    def cfg(policy):
        return SchedulerConfig(slots_n=256, r=0.25, tau_pre=2e-4, tau_global=1e-3, policy=policy)

    be = GpuBackend(idx, cache, slots=256, stream=torch.cuda.Stream())
    # warm-up on the same backend (lane, workspace, graphs) that is measured
    warm = gen_trace(WorkloadSpec(n_db=idx.count, dim=idx.dim, n_requests=2000, arrival_rate=rates[-1], seed=8))
    for policy, chunk in policies.items():
        RealtimePool(be, cfg(policy), tpot=tpot, prefill_chunk=chunk).run(warm)
    out = {"workload": f"C5: gen_trace(Poisson, output 64, delta 32, seed 7) over the C2 index + 10K x {idx.dim} "
                       f"prompt cache (k=1, one lookup per request through the scheduler); wall-clock release of "
                       f"arrivals and decode probes (tpot {tpot * 1e3:g} ms), latency = host result - release; "
                       f"{seconds:g} s of arrivals per run", "runs": {}}
    for rate in rates:
        trace = gen_trace(WorkloadSpec(n_db=idx.count, dim=idx.dim, n_requests=int(rate * seconds),
                                       arrival_rate=rate, seed=7))
        for policy, chunk in policies.items():
            reps = []
            for _ in range(repeats):
                g0 = _lib.graph_counters()
                r = RealtimePool(be, cfg(policy), tpot=tpot, prefill_chunk=chunk).run(trace)
                g1 = _lib.graph_counters()
                reps.append({"latency": r.percentiles(), "batches": r.batches, "launches": r.launches,
                             "preemptions": r.preemptions, "retrievals": r.retrievals, "wall_s": r.wall_s,
                             "busy_s": r.busy_s, "graphs": {k: g1[k] - g0[k] for k in g1}})
            out["runs"][f"{policy}@{rate:g}/s"] = reps if repeats > 1 else reps[0]
    # CPU reference (scheduler + oracle) in the same real-time loop, bounded
    art = orc.IVFArtifact(b["cen"], b["asg"])
    cores = os.cpu_count() or 1
    ob = OracleBackend(b["data"], art, cdata, cores)
    try:
        ctrace = gen_trace(WorkloadSpec(n_db=idx.count, dim=idx.dim, n_requests=cpu_requests, arrival_rate=cpu_rate,
                                        seed=7))
        cr = RealtimePool(ob, cfg("prefill_reserved"), tpot=tpot).run(ctrace)
    finally:
        ob.close()
    cpu_lat = cr.percentiles()
    # the headline run: with repeats, the one with the median prefill p99 (every
    # run's latencies stay in "runs"; at 10K requests/s the pool is ~97% busy,
    # so a single run's p99 can jump on a host hiccup)
    hi = out["runs"][f"decode_priority@{rates[-1]:g}/s"]
    if isinstance(hi, list):
        hi = sorted(hi, key=lambda x: x["latency"]["prefill"]["p99_ms"])[len(hi) // 2]
    out["headline_run"] = "median prefill p99 of the repeats" if repeats > 1 else "single run"
    out["value"] = hi["retrievals"] / hi["wall_s"]
    out["unit"] = "retrievals/s served"
    out["latency_ms"] = hi["latency"]
    out["cpu_baseline"] = {"value": cr.retrievals / cr.wall_s, "unit": "retrievals/s served", "cores": cores,
                           "kind": "port", "latency_ms": cpu_lat,
                           "sample": f"{cpu_requests} requests at {cpu_rate:g}/s, reference scheduler + numpy oracle "
                                     f"on a {cores}-process pool, same loop"}
    out["e2e"] = {"value": out["value"], "unit": out["unit"], "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                  "api": "RealtimePool + GpuBackend: IVFFlatIndex.search_into / knn_into on pinned host buffers"}
    return out


# ----------------------------------------------------------------------------
# graph engine


def engine(peak_gbs: float) -> dict:
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from bench_engine import run

    r = run(n=100_000, d=128, nq=4096, reps=3)
    r["value"] = r["qps"]
    r["e2e"] = {"value": r["e2e_batched_qps"], "unit": UNIT, "api": "submit_many + run_to_completion + result_arrays"}
    return r
