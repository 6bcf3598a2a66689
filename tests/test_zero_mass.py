"""Zero-mass target bins (b_i = 0; Eq. 8 / P:136-146 allow b in the closed simplex, SPEC's
problem invariants ask only b >= 0). DESIGN.md R32: column i's block b_i Delta_m is {0}, so
t_i = 0 at every iterate (empty support), its column gap is exactly 0 and a BCFW-family step on
it is a no-op (away / pairwise: dir 3; plain: the d = 0 step of Alg. 1, which leaves T as it is).

CPU: the oracle on such a problem is pinned against the same problem with the zero columns
removed (the two have the same optimum, objective and gap for the same nonzero columns).
GPU: every variant bit-exact against the oracle with zero-mass columns present."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import BATCHED, BCAFW, BCFW, BCPFW, DEC, ELS, FW, GA, P, U, Oracle
from sro_inputs import instance


def _with_zero_columns(m, n, seed, zeros):
    d = instance(1, m=m, n=n, seed=seed)
    b = d["b"].copy()
    b[zeros] = 0.0
    b /= b.sum()
    C = ((d["X"][:, None, :] - d["Y"][None, :, :]) ** 2).sum(-1)
    return d["a"], b, C


def test_oracle_zero_mass_columns_match_reduced_problem():
    """FW (the unit-free variant, so the column count does not enter the step rule) on the
    problem with zero columns follows the trajectory of the problem without them: the same
    objective and gap at every iteration (the zero columns add exact zeros to every sum), the
    zero columns stay empty, and their column gaps are exactly 0."""
    m, n = 9, 12
    zeros = [0, 5, 11]
    a, b, C = _with_zero_columns(m, n, 3, zeros)
    keep = [i for i in range(n) if i not in zeros]
    full = Oracle(a, b, 1.0, C=C, cap=12)
    red = Oracle(a, b[keep], 1.0, C=C[:, keep], cap=12)
    for it in range(6):
        rf = full.solve(FW, 1, step=ELS, epsilon=-1.0)
        rr = red.solve(FW, 1, step=ELS, epsilon=-1.0)
        assert abs(rf["objective"] - rr["objective"]) <= 1e-15 * abs(rr["objective"])
        assert np.abs(full.plan()[:, keep] - red.plan()).max() <= 1e-15
    T = full.plan()
    assert (T[:, zeros] == 0).all()
    _, g, _, _ = full.gap()
    assert (g[zeros] == 0.0).all()
    assert abs(full.gap()[0] - red.gap()[0]) <= 1e-14


@pytest.mark.parametrize("var,kw", [(BCAFW, dict(step=ELS, sampling=U)), (BCPFW, dict(step=ELS, sampling=P)),
                                    (BCFW, dict(step=DEC, sampling=U)),
                                    (BCFW, dict(step=ELS, sampling=GA, ga_M=1, ga_inner=1, ga_post_update=1))],
                         ids=["away", "pairwise", "plain-dec", "ga"])
def test_oracle_zero_mass_steps_are_noops(var, kw):
    """Every visit of a zero-mass column leaves the plan unchanged; feasibility (columns sum to
    b_i, T >= 0) holds throughout; the solve converges; GA's stored gap of a zero column is 0
    after its first refresh, so the sampler stops drawing it."""
    m, n = 8, 10
    zeros = [2, 7]
    a, b, C = _with_zero_columns(m, n, 4, zeros)
    o = Oracle(a, b, 1.0, C=C, cap=10)
    r = o.solve(var, 2000 * n, seed=3, trace=True, epsilon=1e-5 if kw["step"] == ELS else 1e-3, **kw)
    tr = r["trace"]
    z = np.isin(tr["i"], zeros)
    assert z.any() and r["converged"] == 1
    if var in (BCAFW, BCPFW):
        assert (tr["dir"][z] == 3).all() and (tr["gamma"][z] == 0).all()
    T = o.plan()
    assert (T[:, zeros] == 0).all() and T.min() >= 0
    assert np.abs(T.sum(0) - b).max() <= 1e-15
    if kw["sampling"] == GA:
        G, _ = o.ga_state()
        assert (G[zeros] == 0).all()


# --------------------------------------------------------------------------- GPU parity
@pytest.mark.gpu
@pytest.mark.parametrize("var,kw,m", [
    (BCFW, dict(step=ELS, sampling=U), 300), (BCFW, dict(step=DEC, sampling=P), 4096),
    (BCAFW, dict(step=ELS, sampling=U), 300), (BCAFW, dict(step=ELS, sampling=U), 4096),
    (BCPFW, dict(step=ELS, sampling=P), 4096),
    (BCFW, dict(step=ELS, sampling=GA, ga_M=1, ga_inner=1, ga_post_update=1), 4096),
    (BCPFW, dict(step=ELS, sampling=GA, ga_M=2, ga_inner=1, ga_post_update=0), 300),
    (FW, dict(step=ELS), 300), (BATCHED, dict(step=ELS, sampling=P, block_size=16), 300)],
    ids=["bcfw", "bcfw-dec-pipe", "bcafw", "bcafw-pipe", "bcpfw-pipe", "ga-pipe", "ga-pairwise", "fw", "batched"])
def test_gpu_zero_mass_columns_bitexact(var, kw, m):
    sro = pytest.importorskip("paper_2103_05857_b200")
    n = 256
    zeros = [0, 3, 100, 255]
    a, b, C = _with_zero_columns(m, n, 9, zeros)
    C32 = C.astype(np.float32)
    g = sro.Solver(a, b, 1.0, C=C32, prec="f32")
    o = Oracle(a, b, 1.0, C=C32.astype(np.float64), prec="f32", cap=31)
    GV = {BCFW: sro.SRO_BCFW, BCAFW: sro.SRO_BCAFW, BCPFW: sro.SRO_BCPFW, FW: sro.SRO_FW, BATCHED: sro.SRO_BATCHED}
    iters = 40 if var == FW else (6 * n // 16 if var == BATCHED else 6 * n)
    ro = o.solve(var, iters, seed=4, trace=True, epsilon=1e-12, **kw)
    rg = g.solve(GV[var], iters, seed=4, trace=True, epsilon=1e-12, **kw)
    for f in ("k", "i", "j", "v", "dir", "gamma", "num", "den", "minval"):
        assert np.array_equal(rg["trace"][f], ro["trace"][f]), f
    assert np.array_equal(g.plan(), o.plan()) and np.array_equal(g.rowsums(), o.r())
    assert g.objective() == o.objective()
    tg, gg, _ = g.gap()
    to, go, _, _ = o.gap()
    assert tg == to and np.array_equal(gg, go) and (gg[zeros] == 0).all()
