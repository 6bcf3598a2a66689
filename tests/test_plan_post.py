"""The step after the solve: barycentric projection (Eq. 15,
PAPER.md P:427-432) and the evaluation metrics (iii), (iv), (vi).

CPU tests pin the oracle's implementation to closed forms; GPU tests require the
CUDA path (C-ABI sro_barycentric / sro_metrics) to match the oracle bit for bit
(both sides use the fixed 256-chunk sum shape of R19 over the columns).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import BCFW, ELS, P, U, Oracle
from sro_inputs import instance


def _sq(X, Y):
    return ((X[:, None, :] - Y[None, :, :]) ** 2).sum(-1)


# --------------------------------------------------------------------------- oracle pins (CPU)
def test_identity_plan_projects_onto_targets():
    """X = Y, a = b, T = diag(a): each source colour moves exactly to its target
    (up to the rounding of (t y)/t), e_c = 0, sparsity = 1 - 1/n, <T, C> = 0."""
    rng = np.random.default_rng(0)
    n = 40
    X = rng.random((n, 3))
    a = rng.random(n) + 0.1
    a /= a.sum()
    o = Oracle(a, a, 1.0, C=_sq(X, X), cap=8)
    o.set_plan(np.diag(a))
    xh = o.barycentric(X, X)
    assert np.allclose(xh, X, rtol=2e-16 * 4, atol=0)
    e_c, sp, lin = o.metrics()
    assert e_c <= 1e-16 and lin == 0.0
    assert sp == 1.0 - 1.0 / n


def test_product_plan_projects_every_row_to_the_b_mean():
    """T = a b^T (feasible): every row of Eq. 15 is the b-weighted mean of the
    target colours (the P:1367 observation), e_c ~ 0 and sparsity 0."""
    rng = np.random.default_rng(1)
    m, n = 24, 30
    X, Y = rng.random((m, 3)), rng.random((n, 3))
    a, b = rng.random(m) + 0.2, rng.random(n) + 0.2
    a /= a.sum()
    b /= b.sum()
    o = Oracle(a, b, 1.0, C=_sq(X, Y), cap=m)
    o.set_plan(np.outer(a, b))
    xh = o.barycentric(X, Y)
    mean = (b[:, None] * Y).sum(0)
    assert np.abs(xh - mean[None, :]).max() <= 1e-14
    e_c, sp, _ = o.metrics()
    assert e_c <= 1e-15 and sp == 0.0


def test_rows_without_mass_keep_their_colour_and_initial_metrics():
    """At T^(0) (all mass on row 0) every other row keeps x_k exactly; row 0
    moves to the b-weighted target mean; e_c = ||r0 - a|| in closed form, sparsity = 1 - 1/m."""
    d = instance(1, m=50, n=60, seed=2)
    C = _sq(d["X"], d["Y"])
    o = Oracle(d["a"], d["b"], 1.0, C=C, cap=16)
    xh = o.barycentric(d["X"], d["Y"])
    assert np.array_equal(xh[1:], d["X"][1:])
    assert np.abs(xh[0] - (d["b"][:, None] * d["Y"]).sum(0)).max() <= 1e-14
    e_c, sp, lin = o.metrics()
    r = np.zeros(50)
    r[0] = 1.0
    assert abs(e_c - np.linalg.norm(r - d["a"])) <= 1e-14
    assert sp == 1.0 - 1.0 / 50
    assert abs(lin - (d["b"] * C[0]).sum()) <= 1e-14


def test_large_lambda_vertex_plan_projection():
    """lambda -> inf: one P-epoch of BCFW-ELS puts column i on argmin_k C_ki; Eq. 15
    then gives, for each row k with mass, the b-weighted mean of the targets mapped to k."""
    d = instance(1, m=30, n=70, seed=3)
    C = _sq(d["X"], d["Y"])
    o = Oracle(d["a"], d["b"], 1e12, C=C, cap=8)
    o.solve(BCFW, 70, seed=1, step=ELS, sampling=P, epsilon=-1.0)
    T = o.plan()
    assert np.all((T > 0).sum(0) == 1)
    jmap = C.argmin(0)
    assert np.array_equal(T.argmax(0), jmap)
    xh = o.barycentric(d["X"], d["Y"])
    for k in range(30):
        cols = np.nonzero(jmap == k)[0]
        if len(cols) == 0:
            assert np.array_equal(xh[k], d["X"][k])
        else:
            w = d["b"][cols]
            assert np.abs(xh[k] - (w[:, None] * d["Y"][cols]).sum(0) / w.sum()).max() <= 1e-13


def test_value_error_against_lp_bracket():
    """Metric (vi): at large lambda the converged plan's <T, C> approaches the LP optimum
    from below (the relaxed problem drops the source marginal: P:88-94); the oracle's lin
    agrees with <T, C> computed densely."""
    scipy = pytest.importorskip("scipy.optimize")
    d = instance(1, m=12, n=14, seed=4)
    C = _sq(d["X"], d["Y"])
    m, n = C.shape
    A_eq = np.zeros((m + n, m * n))
    for k in range(m):
        A_eq[k, k * n:(k + 1) * n] = 1.0
    for i in range(n):
        A_eq[m + i, i::n] = 1.0
    res = scipy.linprog(C.ravel(), A_eq=A_eq, b_eq=np.concatenate([d["a"], d["b"]]), bounds=(0, None),
                        method="highs")
    lp = res.fun
    o = Oracle(d["a"], d["b"], 1.0, C=C, cap=12)
    o.solve(BCFW, 2000 * n, seed=1, step=ELS, sampling=U, epsilon=1e-12)
    _, _, lin = o.metrics()
    T = o.plan()
    assert abs(lin - (T * C).sum()) <= 1e-13
    f = o.objective()
    assert (d["b"] * C.min(0)).sum() - 1e-12 <= f <= lp + 1e-12


# --------------------------------------------------------------------------- GPU parity
@pytest.mark.gpu
@pytest.mark.parametrize("m,n,prec", [(256, 256, "f64"), (300, 512, "f32"), (4096, 1024, "f32"), (65, 9000, "f32")])
def test_gpu_barycentric_and_metrics_bitexact(m, n, prec):
    sro = pytest.importorskip("paper_2103_05857_b200")
    d = instance(1, m=m, n=n, seed=5)
    C = _sq(d["X"], d["Y"])
    Cs = C.astype(np.float32) if prec == "f32" else C
    g = sro.Solver(d["a"], d["b"], 1.0, C=Cs, prec=prec)
    o = Oracle(d["a"], d["b"], 1.0, C=np.asarray(Cs, dtype=np.float64), cap=31)
    # T^(0), then after a few epochs (several supports per column, rows with and without mass)
    for epochs in (0, 3):
        if epochs:
            o.solve(BCFW, epochs * n, seed=2, step=ELS, sampling=U, epsilon=-1.0)
            g.solve(sro.SRO_BCFW, epochs * n, seed=2, step=sro.STEP_ELS, sampling=sro.SAMPLE_U, epsilon=-1.0)
        assert np.array_equal(g.plan(), o.plan())
        assert np.array_equal(g.barycentric(d["X"], d["Y"]), o.barycentric(d["X"], d["Y"]))
        assert g.metrics() == o.metrics()


# --------------------------------------------------------------------------- metrics (v), (vi) vs T*_LP
def _lp_plan(a, b, C):
    """T*_LP: the unregularised, unrelaxed OT linear program of P:419 (scipy HiGHS), as COO
    sorted by (column, row) with the LP's zeros dropped."""
    scipy = pytest.importorskip("scipy.optimize")
    m, n = C.shape
    A_eq = np.zeros((m + n, m * n))
    for k in range(m):
        A_eq[k, k * n:(k + 1) * n] = 1.0
    for i in range(n):
        A_eq[m + i, i::n] = 1.0
    res = scipy.linprog(C.ravel(), A_eq=A_eq, b_eq=np.concatenate([a, b]), bounds=(0, None), method="highs")
    assert res.status == 0
    T = res.x.reshape(m, n)
    T[T < 1e-15] = 0.0
    cols, rows = np.nonzero(T.T)
    return T, rows.astype(np.int32), cols.astype(np.int32), T[rows, cols], res.fun


def test_lp_metrics_closed_forms():
    """e_m = ||T - T*|| / ||T*|| and e_v = |<T,C> - <T*,C>| / |<T*,C>| in closed form:
    2 x 2, C = [[1, 2], [2, 1]], a = b = (1/2, 1/2): T*_LP = diag(1/2, 1/2) (cost 1); at T^(0) =
    [[1/2, 1/2], [0, 0]] the difference is [[0, 1/2], [0, -1/2]] so e_m = 1, and <T0, C> = 3/2 so
    e_v = 1/2; at T = T*_LP both are exactly 0."""
    a = b = np.array([0.5, 0.5])
    C = np.array([[1.0, 2.0], [2.0, 1.0]])
    o = Oracle(a, b, 1.0, C=C, cap=2)
    rows, cols, vals = np.array([0, 1]), np.array([0, 1]), np.array([0.5, 0.5])
    assert o.lp_metrics(rows, cols, vals) == (1.0, 0.5)
    o.set_plan(np.diag([0.5, 0.5]))
    assert o.lp_metrics(rows, cols, vals) == (0.0, 0.0)


def test_lp_metrics_against_highs_plan():
    """With T*_LP from scipy HiGHS: e_m = e_v = 0 when the oracle's plan is set to T*_LP; after
    BCFW at large lambda (where the relaxed solution approaches the LP's) e_v is
    small and equals |<T,C> - LP| / LP with LP the solver's optimum, and e_m is the relative
    Frobenius distance (dense numpy evaluation, 1e-12); the relaxed solution moves towards the
    LP's as lambda shrinks (the penalty enforces the source marginal): e_v at
    lambda = 1e-2 is far below e_v at lambda = 1; unsorted or out-of-range T* is rejected."""
    d = instance(1, m=10, n=12, seed=6)
    C = _sq(d["X"], d["Y"])
    T, rows, cols, vals, lp = _lp_plan(d["a"], d["b"], C)
    o = Oracle(d["a"], d["b"], 1.0, C=C, cap=12)
    o.set_plan(T)
    assert o.lp_metrics(rows, cols, vals) == (0.0, 0.0)
    evs = []
    for lam in (1.0, 1e-2):
        o = Oracle(d["a"], d["b"], lam, C=C, cap=12)
        o.solve(BCFW, 3000 * 12, seed=1, step=ELS, sampling=P, epsilon=1e-13)
        em, ev = o.lp_metrics(rows, cols, vals)
        Tg = o.plan()
        assert abs(em - np.linalg.norm(Tg - T) / np.linalg.norm(T)) <= 1e-12
        assert abs(ev - abs((Tg * C).sum() - lp) / lp) <= 1e-9
        evs.append(ev)
    assert evs[1] < evs[0] / 10
    from oracle import OracleError
    with pytest.raises(OracleError):
        o.lp_metrics(rows[::-1], cols[::-1], vals[::-1])
    with pytest.raises(OracleError):
        o.lp_metrics(rows + 100, cols, vals)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,prec", [(10, 12, "f64"), (48, 64, "f32"), (64, 40, "f64")])
def test_gpu_lp_metrics_bitexact(m, n, prec):
    """sro_lp_metrics against the oracle on the same plan and the same T*_LP (scipy HiGHS):
    bit-exact e_m and e_v, at T^(0), after a few epochs, and at T = T*_LP (both 0)."""
    sro = pytest.importorskip("paper_2103_05857_b200")
    d = instance(1, m=m, n=n, seed=7)
    C = _sq(d["X"], d["Y"])
    Cs = C.astype(np.float32) if prec == "f32" else C
    Cd = np.asarray(Cs, dtype=np.float64)
    T, rows, cols, vals, _ = _lp_plan(d["a"], d["b"], Cd)
    g = sro.Solver(d["a"], d["b"], 1.0, C=Cs, prec=prec)
    o = Oracle(d["a"], d["b"], 1.0, C=Cd, cap=31)
    for epochs in (0, 4):
        if epochs:
            o.solve(BCFW, epochs * n, seed=2, step=ELS, sampling=U, epsilon=-1.0)
            g.solve(sro.SRO_BCFW, epochs * n, seed=2, step=sro.STEP_ELS, sampling=sro.SAMPLE_U, epsilon=-1.0)
        assert g.lp_metrics(rows, cols, vals) == o.lp_metrics(rows, cols, vals)
    with pytest.raises(sro.SroError):
        g.lp_metrics(rows[::-1], cols[::-1], vals[::-1])
