"""GPU parity of the column-sharded path: G shards held by one
process (nranks = 1: every phase runs per shard on one stream and the
exchange slots are filled in place — the same kernels and exchange layout as
one shard per GPU, minus the NCCL all-gather). The reductions are subtrees of
the fixed 256-chunk tree (R19), so every G must reproduce the UNSHARDED oracle
bit for bit: argmin rows, step sizes, plan, row sums, gap and objective.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import BATCHED, DEC, ELS, FW, GA, P, U, Oracle
from sro_inputs import instance

pytestmark = pytest.mark.gpu

sro = pytest.importorskip("paper_2103_05857_b200")


def _pair(d, G, shard_block=0, prec="f32", cap=31, cost="dense"):
    if cost == "dense":
        C = d["C32"] if prec == "f32" else d["C64"]
        g = sro.Solver(d["a"], d["b"], d["lam"], C=C, prec=prec, slab_cap=cap, shards=G, shard_block=shard_block)
        o = Oracle(d["a"], d["b"], d["lam"], C=np.asarray(C, dtype=np.float64), cap=cap)
    else:
        g = sro.Solver(d["a"], d["b"], d["lam"], X=d["X"], Y=d["Y"], cost=cost, prec=prec, slab_cap=cap, shards=G,
                       shard_block=shard_block)
        o = Oracle(d["a"], d["b"], d["lam"], X=d["X"], Y=d["Y"], cost=cost, prec=prec, cap=cap)
    return g, o


def _dense(m, n, seed):
    d = instance(1, m=m, n=n, seed=seed)
    if d["C32"] is None:
        C = ((d["X"][:, None, :] - d["Y"][None, :, :]) ** 2).sum(-1)
        d["C32"] = C.astype(np.float32)
    d["C64"] = d["C32"].astype(np.float64)
    return d


def _same_trace(tg, to):
    assert len(tg) == len(to)
    for f in ("k", "i", "j", "gamma", "num", "den", "minval"):
        bad = np.nonzero(tg[f] != to[f])[0]
        assert len(bad) == 0, f"{f} differs first at step {bad[0]}: gpu {tg[bad[0]]} oracle {to[bad[0]]}"


def _same_state(g, o):
    assert g.n_held == o.n
    assert np.array_equal(g.held, np.arange(o.n))
    assert np.array_equal(g.plan(), o.plan())
    assert np.array_equal(g.rowsums(), o.r())
    assert g.objective() == o.objective()
    tg, gg, jg = g.gap()
    to, go, jo, _ = o.gap()
    assert tg == to and np.array_equal(gg, go) and np.array_equal(jg, jo)


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("step", [ELS, DEC])
@pytest.mark.parametrize("tail", [True, False], ids=["tail", "multikernel"])
def test_sharded_fw_bitexact(G, step, tail, monkeypatch):
    """Full FW (Alg. A.1) over G contiguous column shards == the unsharded oracle."""
    if not tail:
        monkeypatch.setenv("SRO_NO_TAIL", "1")
    d = _dense(300, 256, seed=21)
    g, o = _pair(d, G)
    ro = o.solve(FW, 30, trace=True, step=step, epsilon=1e-9)
    rg = g.solve(sro.SRO_FW, 30, trace=True, step=step, epsilon=1e-9)
    _same_trace(rg["trace"], ro["trace"])
    assert rg["converged"] == ro["converged"] and rg["gap"] == ro["gap"]
    _same_state(g, o)


@pytest.mark.parametrize("G,B", [(2, 64), (4, 64), (8, 32), (8, 256)])
@pytest.mark.parametrize("tail", [True, False], ids=["tail", "multikernel"])
def test_sharded_batched_bitexact(G, B, tail, monkeypatch):
    """Batched BCFW (R18) with block_size == shard_block over G interleaved shards
    == the unsharded oracle (P block order, ELS, gap checks every epoch)."""
    if not tail:
        monkeypatch.setenv("SRO_NO_TAIL", "1")
    d = _dense(257, 512, seed=22)
    g, o = _pair(d, G, shard_block=B)
    iters = 6 * (512 // B)
    ro = o.solve(BATCHED, iters, seed=5, trace=True, step=ELS, sampling=P, block_size=B, epsilon=1e-9)
    rg = g.solve(sro.SRO_BATCHED, iters, seed=5, trace=True, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=B,
                 epsilon=1e-9)
    _same_trace(rg["trace"], ro["trace"])
    assert rg["gap"] == ro["gap"]
    _same_state(g, o)


def test_sharded_rectangular_colours_to_gap():
    """Config [4] shape at reduced size (m = 512, n = 8192, fused fp32 colour cost,
    B = 1024 over G = 8 shards) to g <= 1e-6: every step bit-exact vs the oracle."""
    d = instance(4, m=512, n=8192, seed=3)
    g, o = _pair(d, 8, shard_block=1024, cost="sqeuclid")
    ro = o.solve(BATCHED, 400, seed=2, trace=True, step=ELS, sampling=P, block_size=1024, epsilon=1e-6)
    rg = g.solve(sro.SRO_BATCHED, 400, seed=2, trace=True, step=sro.STEP_ELS, sampling=sro.SAMPLE_P,
                 block_size=1024, epsilon=1e-6)
    assert ro["converged"] == 1 and rg["converged"] == 1
    _same_trace(rg["trace"], ro["trace"])
    _same_state(g, o)


def test_sharded_hash_cost_gap_and_fw():
    """HASH_UNIFORM (config [3] cost) generated per shard for its global columns:
    gap sweep and FW-ELS steps identical to the oracle at G = 4."""
    m, n = 1024, 512
    seed = 0x5EED0003
    a = np.full(m, 1.0 / m)
    b = np.full(n, 1.0 / n)
    g = sro.Solver(a, b, 1.0, cost="hash", hash_seed=seed, shards=4)
    o = Oracle(a, b, 1.0, cost="hash", hash_seed=seed, cap=31)
    _same_state(g, o)
    ro = o.solve(FW, 12, trace=True, step=ELS, epsilon=1e-12)
    rg = g.solve(sro.SRO_FW, 12, trace=True, step=sro.STEP_ELS, epsilon=1e-12)
    _same_trace(rg["trace"], ro["trace"])
    _same_state(g, o)


def test_sharded_capacity_error_leaves_state_before_step():
    """A support overflow on some shard (slab_cap = 2, FW-DEC grows supports) is
    reported by every shard as ERR_CAPACITY at the oracle's step, and the columns
    already updated on the other shards are rolled back: plan == oracle's."""
    d = _dense(64, 64, seed=23)
    g, o = _pair(d, 4, cap=2)
    err_o = err_g = None
    try:
        o.solve(FW, 50, step=DEC, epsilon=-1.0)
    except Exception as e:  # noqa: BLE001
        err_o = e
    try:
        g.solve(sro.SRO_FW, 50, step=sro.STEP_DEC, epsilon=-1.0)
    except sro.SroError as e:
        err_g = e
    assert err_o is not None and err_g is not None and err_g.status == 6
    assert np.array_equal(g.plan(), o.plan())
    assert np.array_equal(g.rowsums(), o.r())


def test_sharded_handle_rejects_sequential_variants():
    d = _dense(32, 64, seed=24)
    g, _ = _pair(d, 2)
    with pytest.raises(sro.SroError) as e:
        g.solve(sro.SRO_BCFW, 10, step=sro.STEP_ELS)
    assert e.value.status == 2
    with pytest.raises(sro.SroError):
        g.solve(sro.SRO_BATCHED, 2, block_size=32)   # block_size != shard_block (n)
    with pytest.raises(sro.SroError):
        sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32", shards=3)
    with pytest.raises(sro.SroError):
        sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32", shards=4, shard_block=6)


def test_sharded_nccl_single_rank_path():
    """The NCCL branch itself on one GPU: G = 1 process per shard is not possible on
    one device, so this checks the unique-id call and that an NCCL-mode handle with
    a bad rank is refused before any communicator is built."""
    uid = sro.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128
    d = _dense(32, 64, seed=25)
    with pytest.raises(sro.SroError):
        sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32", shards=2, nranks=2, rank=5, nccl_id=uid)


@pytest.mark.parametrize("G,B,post", [(2, 64, 1), (4, 64, 0), (8, 32, 1)])
def test_sharded_batched_ga_bitexact(G, B, post):
    """GA block sampling (R31) over G column shards: the lead's tree over all n columns, the
    block's gaps gathered from the shards in global position order, the global refresh from
    the exchanged gap sweep == the unsharded oracle step for step (G-invariance)."""
    d = _dense(257, 512, seed=23)
    g, o = _pair(d, G, shard_block=B)
    iters = 5 * (512 // B) + 3
    kw = dict(step=ELS, sampling=GA, ga_M=1, ga_inner=1, ga_post_update=post, block_size=B)
    ro = o.solve(BATCHED, iters, seed=9, trace=True, epsilon=-1.0, **kw)
    rg = g.solve(sro.SRO_BATCHED, iters, seed=9, trace=True, epsilon=-1.0, **kw)
    _same_trace(rg["trace"], ro["trace"])
    assert rg["gap"] == ro["gap"]
    assert rg["entries_scanned"] == ro["entries_scanned"]
    _same_state(g, o)


@pytest.mark.parametrize("G", [2, 8])
def test_sharded_solve_after_reset_repeats_first_solve(G):
    """A sharded handle run to convergence, reset (sro_reset) and run again repeats the first
    solve exactly (hash cost FW-ELS, the multi-kernel step path of config [3])."""
    m, n = 1024, 2048 * G
    seed = 0x5EED0003
    a = np.full(m, 1.0 / m)
    b = np.full(n, 1.0 / n)
    g = sro.Solver(a, b, 1.0, cost="hash", hash_seed=seed, shards=G)
    r1 = g.solve(sro.SRO_FW, 60, trace=True, step=sro.STEP_ELS, epsilon=1e-6)
    T1 = g.plan()
    g.reset()
    r2 = g.solve(sro.SRO_FW, 60, trace=True, step=sro.STEP_ELS, epsilon=1e-6)
    assert r1["iters_done"] == r2["iters_done"] and r1["gap"] == r2["gap"] and r1["converged"] == 1
    assert np.array_equal(r1["trace"], r2["trace"]) and np.array_equal(g.plan(), T1)
