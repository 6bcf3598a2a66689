"""bench.py's N > 1 path on one GPU: two ranks under torchrun with SRO_BENCH_EMULATE_RANKS=1 (gloo
process group, both ranks on cuda:0, the sharded legs exchanging through the library's host
all-gather instead of NCCL). Checks the JSON line rank 0 prints: the replicas' headline, and the
column-sharded FW-ELS (config [3]) and batched B = 1024 (config [4]) legs reaching g <= 1e-6 in
the iteration counts of the unsharded runs (the sharded trajectory is the unsharded one, R19/R26)."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_rank_emulation():
    env = dict(os.environ, SRO_BENCH_EMULATE_RANKS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "1",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["replicas"] == 2
    sh = line["sharded"]
    assert sh["config3"]["converged"] and sh["config3"]["iterations"] == 6 and sh["config3"]["gap"] <= 1e-6
    assert sh["config4"]["converged"] and sh["config4"]["iterations"] == 1024 and sh["config4"]["gap"] <= 1e-6
    assert all(v["shards"] == 2 for v in sh.values())
