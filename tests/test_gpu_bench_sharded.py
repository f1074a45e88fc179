"""bench.py's own sharded (N > 1) step, run as two ranks on one GPU.

The driver launches ``bench.py --gpus N`` under torchrun with NCCL, one GPU
per rank.  Here both ranks share cuda:0 over gloo (BENCH_DEVICE / BENCH_BACKEND
test hooks; NCCL refuses two ranks on one device) on a reduced C4 database
(BENCH_C4_N), which runs the same code: per-rank row draw, centroids trained on
rank 0 and broadcast, per-rank exact list assignment, packed all-gather,
device merge, e2e through ShardedIVF.search_into.  ``--parity full`` compares
every query of lane 0 with the global oracle (per-shard oracle lists merged
by (dist, id)), so a missed neighbour on any shard fails the run.
"""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
def test_bench_sharded_step_two_ranks_full_parity():
    env = dict(os.environ, BENCH_DEVICE="0", BENCH_BACKEND="gloo", BENCH_C4_N="300000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "4", "--warmup", "3", "--lanes", "2", "--parity", "full"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    keep = [ln for ln in res.stderr.splitlines() if "[rank0]" in ln or "parity" in ln or "Error" in ln]
    assert res.returncode == 0, "\n".join(keep)[-4000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["parallelism"] == "vector-shard x2"
    assert line["config"]["n_db"] == 300000 and line["config"]["workload"].startswith("C4")
    assert line["parity"].startswith("ok: 259 queries"), line["parity"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    # the reference arm (CPU oracle) builds the same index artifact on its own
    ref = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C4", "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert ref.returncode == 0, ref.stderr[-2000:]
    rline = json.loads(ref.stdout.strip().splitlines()[-1])
    assert rline["config"] == line["config"], (rline["config"], line["config"])
