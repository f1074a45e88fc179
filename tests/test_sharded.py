"""Vector-sharded search protocol over torch.distributed gloo, world size 2 (CPU).

Each rank searches its id-range shard with the CPU oracle (standing in for the
device IVF shard), the same ShardedSearch gather/merge code path used with NCCL
on GPUs merges the per-shard lists, and the result must equal the global IVF
oracle bit-for-bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import trinity_oracle as orc
from paper_2512_02281_b200.sharded import ShardedSearch, pad_results, shard_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cpu_merge(dists, ids, k):
    d, i = dists.numpy(), ids.numpy()
    out_i = np.full((d.shape[1], k), -1, np.int64)
    out_d = np.full((d.shape[1], k), np.inf)
    for q in range(d.shape[1]):
        mi, md = orc.merge_shards([(i[g, q], d[g, q]) for g in range(d.shape[0])], k)
        out_i[q, : mi.size], out_d[q, : md.size] = mi, md
    return out_i, out_d


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.Generator(np.random.Philox(77))
    data = rng.standard_normal((3000, 12)).astype(np.float32)
    art = orc.kmeans(data, 24, 3, 5)  # shared artifact (deterministic on every rank)
    lo, hi = shard_bounds(data.shape[0], world, rank)
    shard_art = orc.IVFArtifact(art.centroids, art.assign[lo:hi])
    queries = rng.standard_normal((9, 12))

    def local(qs, k, nprobe):
        ids = np.full((qs.shape[0], k), -1, np.int64)
        ds = np.full((qs.shape[0], k), np.inf)
        for j, q in enumerate(qs):
            i, d = orc.ivf_search(data[lo:hi], shard_art, q, k, nprobe)
            ids[j, : i.size], ds[j, : d.size] = i + lo, d
        return ids, ds

    ss = ShardedSearch(local, _cpu_merge)
    ids, ds = ss.search(queries, 7, 5)
    if rank == 0:
        np.savez(out_path, ids=ids, ds=ds)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_cover():
    for n, w in [(10, 3), (1_000_000, 8), (7, 7)]:
        parts = [shard_bounds(n, w, r) for r in range(w)]
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_pad_results():
    i, d = pad_results(np.array([[3, 4]]), np.array([[1.0, 2.0]]), 4)
    assert i.tolist() == [[3, 4, -1, -1]] and np.isinf(d[0, 2:]).all()


def test_two_rank_gloo_sharded_equals_global(tmp_path):
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    rng = np.random.Generator(np.random.Philox(77))
    data = rng.standard_normal((3000, 12)).astype(np.float32)
    art = orc.kmeans(data, 24, 3, 5)
    queries = rng.standard_normal((9, 12))
    for j, q in enumerate(queries):
        i, d = orc.ivf_search(data, art, q, 7, 5)
        assert np.array_equal(got["ids"][j, : i.size], i) and np.array_equal(got["ds"][j, : d.size], d)


def test_reference_arm_c4_small():
    """bench.py --impl reference on a reduced C4: CPU oracle only (no GPU)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BENCH_C4_N="20000")
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C4", "--steps", "2",
                          "--warmup", "1"], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["config"]["n_db"] == 20000
    assert line["e2e"]["h2d_bytes_per_step"] == 0
