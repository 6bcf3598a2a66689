"""The multi-process sharded path (one shard per process, nranks = G) on ONE GPU.

G processes join a gloo process group and each builds a sharded Solver for its own column
shard, exactly as bench.py's and dist.sharded_solver's ranks do on a multi-GPU box; the per-step
exchanges go through sro_params.exchange (a host all-gather over gloo) instead of NCCL, since
NCCL will not put two ranks on one device. Everything else is the nranks == G code path: rank-
local cost shards and hash generation, phase A / exchange / phase B / exchange / apply per block
step, the all-gathered gap and objective, GA block sampling with every process holding its
replica of the tree. The ranks' kernels never wait on one another (the exchange is a host round
trip between launches). Rank 0's per-step trace and every rank's held columns of the plan, row sums,
gap and objective equal the UNSHARDED oracle's bit for bit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from oracle import BATCHED, ELS, FW, GA, P, Oracle
from sro_inputs import instance

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name):
    """(problem dict, solver kwargs, solve args) of one case."""
    if name == "fw-hash":
        m, n = 1024, 512
        d = dict(a=np.full(m, 1.0 / m), b=np.full(n, 1.0 / n), lam=1.0)
        return d, dict(cost="hash", hash_seed=0x5EED0003), (FW, 10, dict(step=ELS, epsilon=1e-12)), 0
    if name == "fw-dense":
        d = instance(1, m=300, n=256, seed=21)
        d["C32"] = (((d["X"][:, None, :] - d["Y"][None, :, :]) ** 2).sum(-1)).astype(np.float32)
        return d, dict(C=d["C32"], prec="f32"), (FW, 30, dict(step=ELS, epsilon=1e-9)), 0
    if name == "batched-colour":
        d = instance(4, m=512, n=8192, seed=3)
        return d, dict(X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32"), \
            (BATCHED, 60, dict(step=ELS, sampling=P, block_size=1024, epsilon=1e-9)), 1024
    if name == "batched-ga":
        d = instance(1, m=257, n=512, seed=22)
        d["C32"] = (((d["X"][:, None, :] - d["Y"][None, :, :]) ** 2).sum(-1)).astype(np.float32)
        return d, dict(C=d["C32"], prec="f32"), \
            (BATCHED, 90, dict(step=ELS, sampling=GA, ga_M=2, ga_inner=1, ga_post_update=1, block_size=64,
                               epsilon=1e-9)), 64
    raise KeyError(name)


def _worker(rank, world, port, name, q, reset_first=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2103_05857_b200 as sro
        from paper_2103_05857_b200.dist import sharded_solver
        d, skw, (variant, iters, opts), Bo = _case(name)
        C = skw.pop("C", None)
        Y = skw.pop("Y", None)
        X = skw.pop("X", None)
        g = sharded_solver(d["a"], d["b"], d["lam"], shard_block=Bo, C=C, X=X, Y=Y, transport="host", **skw)
        gv = {FW: sro.SRO_FW, BATCHED: sro.SRO_BATCHED}[variant]
        if reset_first:   # a whole solve, then sro_reset: the second solve must be the first one again
            g.solve(gv, iters, seed=5, **opts)
            g.reset()
        r = g.solve(gv, iters, seed=5, trace=True, **opts)
        total, gcol, jcol = g.gap()
        q.put((rank, dict(held=g.held, trace=r["trace"], gap=r["gap"], converged=r["converged"],
                          iters=r["iters_done"], T=g.plan(), r=g.rowsums(), f=g.objective(), g=total, gcol=gcol,
                          jcol=jcol)))
        g.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G,reset_first", [(2, False), (4, False), (2, True)], ids=["G2", "G4", "G2-after-reset"])
@pytest.mark.parametrize("name", ["fw-hash", "fw-dense", "batched-colour", "batched-ga"])
def test_multiprocess_sharded_bitexact(name, G, reset_first):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, G, port, name, q, reset_first)) for r in range(G)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(G):
        rank, res = q.get(timeout=600)
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
    for r in range(G):
        assert isinstance(out[r], dict), out[r]
    d, skw, (variant, iters, opts), _ = _case(name)
    if "C" in skw:
        o = Oracle(d["a"], d["b"], d["lam"], C=np.asarray(skw["C"], dtype=np.float64), cap=31)
    elif skw.get("cost") == "hash":
        o = Oracle(d["a"], d["b"], d["lam"], cost="hash", hash_seed=skw["hash_seed"], cap=31)
    else:
        o = Oracle(d["a"], d["b"], d["lam"], X=d["X"], Y=d["Y"], cost=skw["cost"], prec=skw["prec"], cap=31)
    ro = o.solve(variant, iters, seed=5, trace=True, **opts)
    To = o.plan()
    ro_tot, ro_g, ro_j, _ = o.gap()
    held_all = np.sort(np.concatenate([out[r]["held"] for r in range(G)]))
    assert np.array_equal(held_all, np.arange(o.n))
    for r in range(G):
        res = out[r]
        if r == 0:   # the per-step record is written by the rank holding U's first column (sro.h)
            for f in ("k", "i", "j", "gamma", "num", "den", "minval"):
                assert np.array_equal(res["trace"][f], ro["trace"][f]), (r, f)
        assert res["iters"] == ro["iters_done"] and res["gap"] == ro["gap"] and res["converged"] == ro["converged"]
        assert np.array_equal(res["T"], To[:, res["held"]])
        assert np.array_equal(res["r"], o.r())
        assert res["f"] == o.objective()
        assert res["g"] == ro_tot
        assert np.array_equal(res["gcol"], ro_g[res["held"]]) and np.array_equal(res["jcol"], ro_j[res["held"]])
