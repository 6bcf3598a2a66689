"""Degenerate and ragged inputs through the CUDA path, bit-exact against the oracle
(DESIGN.md §3 fixes every operation, so the bar is equality): a single row (every LMO returns
row 0, the plan is feasible and optimal at T^(0)), a single column (BCFW == FW), both, sizes
that leave ragged 256-chunks and vector tails (fp64 and fp32 costs), rows with a_k = 0, constant costs (every LMO a
full tie -> lowest row), zero costs, and extreme lambda (h dominated by r - a or vanishing).
Every BCFW-family variant, FW and batched run a few epochs with per-step traces compared."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import BATCHED, BCAFW, BCFW, BCPFW, ELS, DEC, FW, GA, P, U, Oracle
from sro_inputs import mixture_colours, sqeuclid_cost

pytestmark = pytest.mark.gpu

sro = pytest.importorskip("paper_2103_05857_b200")

RUNS = [
    ("bcfw-U-ELS", BCFW, sro.SRO_BCFW, dict(step=ELS, sampling=U)),
    ("bcfw-P-DEC", BCFW, sro.SRO_BCFW, dict(step=DEC, sampling=P)),
    ("bcafw-U", BCAFW, sro.SRO_BCAFW, dict(step=ELS, sampling=U)),
    ("bcpfw-P", BCPFW, sro.SRO_BCPFW, dict(step=ELS, sampling=P)),
    ("ga-gad", BCFW, sro.SRO_BCFW, dict(step=ELS, sampling=GA, ga_M=1, ga_inner=1, ga_post_update=1)),
    ("fw-ELS", FW, sro.SRO_FW, dict(step=ELS)),
    ("fw-DEC", FW, sro.SRO_FW, dict(step=DEC)),
    ("batched", BATCHED, sro.SRO_BATCHED, dict(step=ELS, sampling=P)),
]


def _inst(kind, m, n, seed=0):
    X, _, _ = mixture_colours(m, 4, 0.05, 2 * seed + 11)
    Y, _, _ = mixture_colours(n, 4, 0.05, 2 * seed + 12)
    rng = np.random.default_rng(seed)
    a = rng.random(m) + 0.05
    b = rng.random(n) + 0.05
    if kind == "zero_rows" and m > 2:
        a[::3] = 0.0
    a /= a.sum()
    b /= b.sum()
    C = sqeuclid_cost(X, Y)
    if kind == "const":
        C = np.full((m, n), 0.37)
    elif kind == "zero":
        C = np.zeros((m, n))
    return a, b, C


CASES = [
    ("one_row", 1, 37, 1.0), ("one_col", 41, 1, 1.0), ("one_by_one", 1, 1, 1.0), ("ragged", 257, 35, 1.0),
    ("ragged", 5, 3, 1.0), ("ragged", 1031, 13, 1.0), ("zero_rows", 90, 40, 1.0), ("const", 64, 48, 1.0),
    ("zero", 30, 20, 1.0), ("lam_small", 80, 60, 1e-6), ("lam_large", 80, 60, 1e6),
]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("case,m,n,lam", CASES, ids=[f"{c[0]}-{c[1]}x{c[2]}" for c in CASES])
@pytest.mark.parametrize("name,ov,gv,kw", RUNS, ids=[r[0] for r in RUNS])
def test_degenerate_inputs_bitexact(case, m, n, lam, name, ov, gv, kw, prec):
    a, b, C = _inst(case, m, n)
    if prec == "f32":
        C = C.astype(np.float32)
    kw = dict(kw)
    if ov == BATCHED:
        B = next(d for d in (16, 8, 5, 4, 3, 2, 1) if n % d == 0)
        kw["block_size"] = B
        iters = 3 * (n // B)
    elif ov == FW:
        iters = 6
    else:
        iters = 3 * n
    g = sro.Solver(a, b, lam, C=C, prec=prec)
    o = Oracle(a, b, lam, C=C, prec=prec, cap=31)
    ro = o.solve(ov, iters, seed=5, trace=True, epsilon=-1.0, **kw)
    rg = g.solve(gv, iters, seed=5, trace=True, epsilon=-1.0, **kw)
    assert rg["iters_done"] == ro["iters_done"]
    for f in ("k", "i", "j", "gamma", "num", "den", "minval"):
        assert np.array_equal(rg["trace"][f], ro["trace"][f]), f
    assert np.array_equal(g.plan(), o.plan())
    assert np.array_equal(g.rowsums(), o.r())
    tg, gg, jg = g.gap()
    to, go, jo, _ = o.gap()
    assert tg == to and np.array_equal(gg, go) and np.array_equal(jg, jo)
    assert g.objective() == o.objective()
    g.close()


@pytest.mark.parametrize("m,n", [(20000, 48), (3, 9000)])
@pytest.mark.parametrize("name,ov,gv,kw", [RUNS[0], RUNS[2], RUNS[3], RUNS[4]], ids=[RUNS[q][0] for q in (0, 2, 3, 4)])
def test_tall_and_wide_sequential_bitexact(m, n, name, ov, gv, kw):
    """Shapes outside the shared-memory / register-file kernels' limits (m = 20000 rows of h
    and r do not fit next to the GA tree; n = 9000 stored gaps): the fallback kernels
    (global-memory state) give the same trajectories."""
    a, b, C = _inst("ragged", m, n, seed=1)
    C = C.astype(np.float32)
    g = sro.Solver(a, b, 1.0, C=C, prec="f32")
    o = Oracle(a, b, 1.0, C=C, prec="f32", cap=31)
    iters = 2 * n if n < 1000 else 3000
    ro = o.solve(ov, iters, seed=2, trace=True, epsilon=-1.0, **kw)
    rg = g.solve(gv, iters, seed=2, trace=True, epsilon=-1.0, **kw)
    for f in ("i", "j", "gamma", "num", "den", "minval"):
        assert np.array_equal(rg["trace"][f], ro["trace"][f]), f
    assert np.array_equal(g.plan(), o.plan())
    g.close()


def test_explicit_visits_out_of_range_rejected():
    """sro_solve range-checks an explicit visit list (columns in [0, n), blocks in [0, n / B))
    before it reaches the device: INVALID_ARG, state untouched."""
    a, b, C = _inst("plain", 40, 32)
    g = sro.Solver(a, b, 1.0, C=C)
    T0 = g.plan()
    for v in ([0, 5, 32], [-1], [3, 2**31 - 1]):
        with pytest.raises(sro.SroError) as e:
            g.solve(sro.SRO_BCFW, len(v), visit=v, step=sro.STEP_ELS, epsilon=-1.0)
        assert e.value.status == 2
        g.reset()
    with pytest.raises(sro.SroError) as e:
        g.solve(sro.SRO_BATCHED, 2, visit=[0, 4], step=sro.STEP_ELS, block_size=8, epsilon=-1.0)
    assert e.value.status == 2
    assert np.array_equal(g.plan(), T0)


def test_batched_ga_past_4096_steps_bitexact():
    """Batched GA in cursor mode draws the next block after a call's last step into visit slot
    iters: with iters > 4096 (beyond the default visit buffer) the solve stays in bounds and
    bit-exact against the oracle, across two calls."""
    a, b, C = _inst("plain", 48, 64, seed=3)
    g = sro.Solver(a, b, 1.0, C=C)
    o = Oracle(a, b, 1.0, C=C, cap=31)
    kw = dict(step=ELS, sampling=GA, ga_M=2, ga_inner=1, ga_post_update=1, block_size=4)
    for iters in (4200, 300):
        ro = o.solve(BATCHED, iters, seed=6, trace=True, epsilon=-1.0, **kw)
        rg = g.solve(sro.SRO_BATCHED, iters, seed=6, trace=True, epsilon=-1.0, **kw)
        for f in ("k", "i", "j", "gamma", "num", "den"):
            assert np.array_equal(rg["trace"][f], ro["trace"][f]), f
    assert np.array_equal(g.plan(), o.plan())


COLOUR_CASES = [("one_row", 1, 37), ("one_col", 41, 1), ("one_by_one", 1, 1), ("ragged", 257, 35), ("ragged", 5, 3),
                ("ragged", 1031, 13), ("ragged", 929, 300), ("wide", 33, 9476)]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("cost", ["sqeuclid", "euclid"])
@pytest.mark.parametrize("case,m,n", COLOUR_CASES, ids=[f"{c[0]}-{c[1]}x{c[2]}" for c in COLOUR_CASES])
@pytest.mark.parametrize("name,ov,gv,kw", [RUNS[0], RUNS[5], RUNS[7]], ids=[RUNS[q][0] for q in (0, 5, 7)])
def test_degenerate_colour_inputs_bitexact(case, m, n, name, ov, gv, kw, cost, prec):
    """Fused colour costs (the sweeps' packed binary32 paths: row pairs with an odd last row, planar
    slabs of one row, blocks of one column) on ragged and degenerate shapes: bit-exact trajectories,
    plans, gaps and objectives against the oracle."""
    X, _, _ = mixture_colours(m, 4, 0.05, 31)
    Y, _, _ = mixture_colours(n, 4, 0.05, 32)
    rng = np.random.default_rng(7)
    a = rng.random(m) + 0.05
    b = rng.random(n) + 0.05
    a /= a.sum()
    b /= b.sum()
    kw = dict(kw)
    if ov == BATCHED:
        B = next(d for d in (16, 8, 5, 4, 3, 2, 1) if n % d == 0)
        kw["block_size"] = B
        iters = 3 * (n // B)
    elif ov == FW:
        iters = 6
    else:
        iters = 3 * n
    g = sro.Solver(a, b, 1.0, X=X, Y=Y, cost=cost, prec=prec)
    o = Oracle(a, b, 1.0, X=X, Y=Y, cost=cost, prec=prec, cap=31)
    ro = o.solve(ov, iters, seed=5, trace=True, epsilon=-1.0, **kw)
    rg = g.solve(gv, iters, seed=5, trace=True, epsilon=-1.0, **kw)
    assert rg["iters_done"] == ro["iters_done"]
    for f in ("k", "i", "j", "gamma", "num", "den", "minval"):
        assert np.array_equal(rg["trace"][f], ro["trace"][f]), f
    assert np.array_equal(g.plan(), o.plan())
    assert np.array_equal(g.rowsums(), o.r())
    tg, gg, jg = g.gap()
    to, go, jo, _ = o.gap()
    assert tg == to and np.array_equal(gg, go) and np.array_equal(jg, jo)
    assert g.objective() == o.objective()
    g.close()
