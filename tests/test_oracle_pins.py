"""Pins of the fp64 oracle against what PAPER.md and the mathematics fix.

Every test here ties an oracle function to something other than itself:
values printed in the paper, closed forms, theorems (two independently coded
formulas that the paper proves equal), brute force over vertices, grid
search, scipy's LP solver, or the exact-rational replay in exact_replay.py.
Citations: P:<line> = /root/reference/PAPER.md, S:<line> = SPEC.md.
"""
from __future__ import annotations

import itertools
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import (BATCHED, BCAFW, BCFW, BCPFW, DEC, ELS, FW, GA, P, U, Oracle, chunk_tree_sum, fenwick_draw,
                    permutation, rng_u64, splitmix64_mix, uniform53)
from sro_inputs import hash_uniform_cost, instance, uniform_colours
from tests.exact_replay import ExactState

GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")


def rand_instance(m, n, seed, lam=1.0):
    rs = np.random.default_rng(seed)
    a = rs.random(m) + 0.1
    a /= a.sum()
    b = rs.random(n) + 0.1
    b /= b.sum()
    C = rs.random((m, n))
    return a, b, C, lam


def rand_plan(b, m, rs, density=0.6):
    n = len(b)
    T = np.zeros((m, n))
    for i in range(n):
        w = rs.random(m) * (rs.random(m) < density)
        if w.sum() == 0:
            w[rs.integers(m)] = 1.0
        T[:, i] = b[i] * w / w.sum()
    return T


def grad_fd(o, T, eps=1e-6):
    """Gradient of the oracle's objective by central finite differences (T > eps)."""
    assert T.min() > eps
    m, n = T.shape
    G = np.zeros((m, n))
    for i in range(n):
        for k in range(m):
            Tp = T.copy(); Tp[k, i] += eps
            Tm = T.copy(); Tm[k, i] -= eps
            o.set_plan(Tp); fp = o.objective()
            o.set_plan(Tm); fm = o.objective()
            G[k, i] = (fp - fm) / (2 * eps)
    o.set_plan(T)
    return G


# --------------------------------------------------------------------------- objective
def test_objective_spec_worked_example():
    """C=[[0,1],[1,0]], a=b=(1/2,1/2), lambda=1: f(diag)=0, f([[.5,.5],[0,0]])=0.75 (Eq. 7)."""
    C = np.array([[0.0, 1.0], [1.0, 0.0]])
    o = Oracle([0.5, 0.5], [0.5, 0.5], 1.0, C=C)
    o.set_plan(np.diag([0.5, 0.5]))
    assert o.objective() == 0.0
    o.set_plan(np.array([[0.5, 0.5], [0.0, 0.0]]))
    assert abs(o.objective() - 0.75) < 1e-15


def test_initial_plan_is_first_row():
    """T^(0) = (b_1 e_1, ..., b_n e_1): r = (1, 0, ..., 0)."""
    a, b, C, lam = rand_instance(5, 4, 1)
    o = Oracle(a, b, lam, C=C)
    T = o.plan()
    assert np.array_equal(T[0], b) and not T[1:].any()
    assert np.array_equal(o.r(), np.r_[b.sum(), np.zeros(4)])


# --------------------------------------------------------------------------- gradient / LMO
def test_gradient_matches_finite_differences():
    """grad_i f = c_i + (T1 - a)/lambda, checked through the LMO value
    min_k grad_ki against a finite-difference gradient of f."""
    a, b, C, lam = rand_instance(4, 3, 11, lam=0.7)
    o = Oracle(a, b, lam, C=C)
    T = rand_plan(b, 4, np.random.default_rng(3), density=1.0)
    o.set_plan(T)
    G = grad_fd(o, T)
    for i in range(3):
        j, mv = o.lmo(i)
        assert abs(mv - G[:, i].min()) < 1e-7
        assert abs(G[j, i] - G[:, i].min()) < 1e-7


@pytest.mark.parametrize("col,expect", [((3.0, 1.0, 2.0), 1), ((2.0, 2.0, 2.0), 0), ((0.0, -0.0, 5.0), 0)])
def test_lmo_hand_cases(col, expect):
    """S:70-71 hand cases (argmin of a 3-vector; lowest-index tie rule R1), with h = 0
    by setting T 1 = a (m = 3, n = 1)."""
    a = np.array([0.25, 0.25, 0.5])
    o = Oracle(a, [1.0], 1.0, C=np.array(col).reshape(3, 1))
    o.set_plan(a.reshape(3, 1))
    j, mv = o.lmo(0)
    assert j == expect and mv == min(col)


def test_lmo_minimises_linear_form_over_simplex():
    """Eq. 9: s_i = b_i e_j minimises <s, grad_i f> over the scaled simplex b_i Delta_m:
    compare with 2000 random feasible points and all m vertices (brute force)."""
    rs = np.random.default_rng(5)
    a, b, C, lam = rand_instance(12, 6, 7, lam=0.3)
    o = Oracle(a, b, lam, C=C)
    T = rand_plan(b, 12, rs, density=1.0)
    o.set_plan(T)
    G = grad_fd(o, T)
    for i in range(6):
        j, mv = o.lmo(i)
        lin_s = b[i] * G[j, i]
        pts = rs.dirichlet(np.ones(12), size=2000) * b[i]
        assert lin_s <= (pts @ G[:, i]).min() + 1e-7
        assert lin_s <= (b[i] * G[:, i]).min() + 1e-7


def test_lmo_ties_with_duplicate_rows():
    """Exact duplicate source colours give exact cost ties; the LMO returns the lowest row (R1)."""
    X = np.array([[0.2, 0.3, 0.4], [0.9, 0.1, 0.0], [0.2, 0.3, 0.4], [0.5, 0.5, 0.5]])
    Y = np.array([[0.2, 0.3, 0.41]])
    a = np.array([0.25, 0.25, 0.25, 0.25])
    o = Oracle(a, [1.0], 1.0, X=X, Y=Y, cost="sqeuclid")
    o.set_plan(a.reshape(4, 1))
    assert o.lmo(0)[0] == 0


# --------------------------------------------------------------------------- gap
def test_gap_theorem2_three_forms_and_weak_duality():
    """Thm 2: the linearization gap <T-S,C> + (1/l)<T1-S1, T1-a> equals
    sum_i g_i (Eq. 11) and equals the Lagrangian gap f - w (App. D);
    g_i >= 0 and w <= f. 100 random instances and plans (S:520 criterion 1)."""
    rs = np.random.default_rng(0)
    for t in range(100):
        m, n = rs.integers(2, 17, size=2)
        lam = float(10 ** rs.uniform(-3, 0))
        a, b, C, _ = rand_instance(m, n, 1000 + t)
        o = Oracle(a, b, lam, C=C)
        o.set_plan(rand_plan(b, m, rs))
        g, gi, _, _ = o.gap()
        f = o.objective()
        w = o.lagrangian_dual()
        g2 = o.gap_thm2()
        tol = 1e-9 * (1 + abs(f))
        assert abs(g - g2) <= tol
        assert abs(g - (f - w)) <= tol
        assert gi.min() >= -1e-12
        assert w <= f + 1e-12


@pytest.mark.parametrize("m,n", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_gap_is_max_over_all_vertex_choices(m, n):
    """Linearization gap g(T) = max_{S' in M} <T - S', grad f(T)> by exhaustive
    enumeration of all m^n vertex combinations, gradient by finite differences."""
    rs = np.random.default_rng(m * 10 + n)
    a, b, C, lam = rand_instance(m, n, 31 + m + n, lam=0.5)
    o = Oracle(a, b, lam, C=C)
    T = rand_plan(b, m, rs, density=1.0)
    o.set_plan(T)
    G = grad_fd(o, T)
    best = -np.inf
    for js in itertools.product(range(m), repeat=n):
        S = np.zeros((m, n))
        for i, j in enumerate(js):
            S[j, i] = b[i]
        best = max(best, float(((T - S) * G).sum()))
    g = o.gap()[0]
    assert abs(g - best) < 1e-6


def test_gap_vanishes_at_optimum_and_bounds_suboptimality():
    """g(T) >= f(T) - f* (FW gap certificate) and g -> 0 at the optimum."""
    a, b, C, lam = rand_instance(6, 5, 2, lam=0.5)
    o = Oracle(a, b, lam, C=C)
    o.solve(BCPFW, 20000, seed=3, step=ELS, sampling=U, epsilon=1e-13)
    fstar = o.objective()
    assert o.gap()[0] <= 1e-12
    o2 = Oracle(a, b, lam, C=C)
    o2.solve(BCFW, 60, seed=1, step=DEC, sampling=U, epsilon=0.0)
    assert o2.objective() - fstar <= o2.gap()[0] + 1e-12


# --------------------------------------------------------------------------- line search
def _segment_f(o, T, i, newcol_fn, gammas):
    vals = []
    for g in gammas:
        T2 = T.copy()
        T2[:, i] = newcol_fn(g)
        o.set_plan(T2)
        vals.append(o.objective())
    o.set_plan(T)
    return np.array(vals)


def test_els_bcfw_is_exact_minimiser_along_segment():
    """Eq. 10: gamma_LS minimises f((1-g) t_i + g s_i) over g in [0,1];
    check against a 1001-point grid and the vertex of the 3-point quadratic fit."""
    rs = np.random.default_rng(21)
    for t in range(25):
        a, b, C, lam = rand_instance(5, 4, 300 + t, lam=float(10 ** rs.uniform(-2, 0.5)))
        o = Oracle(a, b, lam, C=C)
        T = rand_plan(b, 5, rs)
        o.set_plan(T)
        i = int(rs.integers(4))
        j, _ = o.lmo(i)
        s = np.zeros(5); s[j] = b[i]
        tr = o.solve(BCFW, 1, seed=0, visit=[i], trace=True, step=ELS, sampling=U, epsilon=-1.0)["trace"]
        gam = tr["gamma"][0]
        o.set_plan(T)
        col = lambda g: (1 - g) * T[:, i] + g * s  # noqa: E731
        grid = np.linspace(0, 1, 1001)
        fg = _segment_f(o, T, i, col, grid)
        fstar = _segment_f(o, T, i, col, [gam])[0]
        assert fstar <= fg.min() + 1e-12
        f0, fh, f1 = _segment_f(o, T, i, col, [0.0, 0.5, 1.0])
        # quadratic through (0,f0),(1/2,fh),(1,f1): vertex at -B/(2A)
        A = 2 * (f1 - 2 * fh + f0)
        B = f1 - f0 - A
        if A > 1e-14:
            vertex = min(max(-B / (2 * A), 0.0), 1.0)
            assert abs(vertex - gam) < 1e-6


def test_els_fw_and_batched_are_exact_minimisers():
    """Eq. A.1 for FW, and the joint block line search (R18) for batched:
    f at the returned gamma is <= f on a 1001-point grid along the same direction."""
    rs = np.random.default_rng(4)
    for variant, B in ((FW, 0), (BATCHED, 2)):
        a, b, C, lam = rand_instance(6, 4, 77, lam=0.4)
        o = Oracle(a, b, lam, C=C)
        T = rand_plan(b, 6, rs)
        o.set_plan(T)
        cols = list(range(4)) if variant == FW else [2, 3]
        S = np.zeros_like(T)
        for i in cols:
            S[o.lmo(i)[0], i] = b[i]
        kw = dict(block_size=B) if B else {}
        tr = o.solve(variant, 1, seed=0, visit=[1] if B else None, trace=True, step=ELS, sampling=U,
                     epsilon=-1.0, **kw)["trace"]
        gam = tr["gamma"][0]
        fvals = []
        for g in np.r_[np.linspace(0, 1, 1001), gam]:
            T2 = T.copy()
            T2[:, cols] = (1 - g) * T[:, cols] + g * S[:, cols]
            o.set_plan(T2)
            fvals.append(o.objective())
        assert fvals[-1] <= min(fvals[:-1]) + 1e-12


def test_curvature_quotient_is_exact_quadratic():
    """Def. 1 / App. C: f is quadratic, so the block curvature
    quotient 2/g^2 (f(Y) - f(T) - g<s_i - t_i, grad_i f>) equals ||s_i - t_i||^2 / lambda,
    which is <= 4 b_i^2 / lambda."""
    rs = np.random.default_rng(8)
    for t in range(30):
        a, b, C, lam = rand_instance(5, 4, 500 + t, lam=float(10 ** rs.uniform(-2, 1)))
        o = Oracle(a, b, lam, C=C)
        T = rand_plan(b, 5, rs, density=1.0)
        o.set_plan(T)
        i = int(rs.integers(4))
        snew = rs.dirichlet(np.ones(5)) * b[i]
        G = grad_fd(o, T)
        g = float(rs.uniform(0.05, 1))
        Y = T.copy(); Y[:, i] = T[:, i] + g * (snew - T[:, i])
        o.set_plan(Y); fy = o.objective()
        o.set_plan(T); ft = o.objective()
        q = 2 / g**2 * (fy - ft - g * float((snew - T[:, i]) @ G[:, i]))
        assert abs(q - ((snew - T[:, i]) ** 2).sum() / lam) < 1e-5 * (1 + abs(q))
        assert q <= 4 * b[i] ** 2 / lam + 1e-9


def test_initial_gap_bound():
    """App. C: g(T^0) <= max C + 2/lambda at first-row init."""
    for lam in (1e-3, 0.1, 1.0, 10.0):
        d = instance(1, m=64, n=48)
        o = Oracle(d["a"], d["b"], lam, C=d["C64"])
        assert o.gap()[0] <= o.max_cost() + 2 / lam


# --------------------------------------------------------------------------- worked example
def test_three_colour_T1_printed_values():
    """Worked example, Fig. 5(b) P:1046-1052 and Fig. 7(b): BCFW-P-DEC on
    m=n=3, a=(0.1,0.3,0.6), b=(0.6,0.3,0.1). With the decay counter k global (R2) and
    first-row init (R3), the printed T^(1) is reproduced by visit order (3,1,2) (1-based)
    for any colours in [0,1]^3 (the penalty dominates): exact values
    col1 = 0.6(1/7, 0, 6/7), col2 = 0.3(1/4, 3/4, 0), col3 = (0, 0, 0.1)."""
    printed = np.loadtxt(os.path.join(GOLDEN_DIR, "three_colour_T1.txt"))
    exact = np.array([[0.6 / 7, 0.075, 0.0], [0.0, 0.225, 0.0], [3.6 / 7, 0.0, 0.1]])
    for lam in (1e-6, 1e-3):
        for trial in range(3):
            X = uniform_colours(3, 100 + trial)
            Y = uniform_colours(3, 200 + trial)
            o = Oracle([0.1, 0.3, 0.6], [0.6, 0.3, 0.1], lam, X=X, Y=Y, cost="sqeuclid")
            tr = o.solve(BCFW, 3, seed=0, visit=[2, 0, 1], trace=True, step=DEC, sampling=P, epsilon=-1.0)["trace"]
            T1 = o.plan()
            assert np.abs(T1 - printed).max() <= 5e-3 + 1e-12          # printed to 2-3 digits, truncated
            assert np.abs(T1 - exact).max() <= 1e-12
            assert list(tr["gamma"]) == [1.0, 6 / 7, 0.75]


# --------------------------------------------------------------------------- closed forms
def test_lambda_to_infinity_closed_form():
    """with lambda -> inf the problem becomes the one-sided relaxation with
    value sum_i b_i min_k C_ki. One P-epoch of BCFW-ELS reaches it (gamma clamps to 1)."""
    d = instance(1, m=64, n=48)
    o = Oracle(d["a"], d["b"], 1e12, C=d["C64"])
    o.solve(BCFW, 48, seed=5, step=ELS, sampling=P, epsilon=-1.0)
    closed = float((d["b"] * d["C64"].min(axis=0)).sum())
    f = o.objective()
    r = o.r()
    resid = float(((r - d["a"]) ** 2).sum() / (2 * 1e12))
    assert abs(f - closed - resid) <= 1e-14 * closed
    assert o.gap()[0] <= 1e-12


def test_zero_cost_and_identical_marginals_have_zero_optimum():
    """C = 0: T = a b^T is feasible with zero penalty, so f* = 0; X = Y, a = b with
    squared-Euclidean cost: T = diag(a) gives f* = 0 (closed forms)."""
    a, b, C, lam = rand_instance(6, 5, 9)
    o = Oracle(a, b, 1.0, C=np.zeros((6, 5)))
    o.solve(BCPFW, 40000, seed=1, step=ELS, sampling=U, epsilon=1e-14)
    assert o.objective() <= 1e-12
    X = uniform_colours(7, 4)
    aa = np.full(7, 1 / 7)
    o2 = Oracle(aa, aa, 0.1, X=X, Y=X, cost="sqeuclid")
    o2.solve(BCPFW, 40000, seed=1, step=ELS, sampling=U, epsilon=1e-14)
    assert o2.objective() <= 1e-12


def test_lp_bracket_and_certificate():
    """sum_i b_i min_k C_ki <= f* <= <T*_LP, C> (LP by scipy HiGHS),
    and the oracle's certified optimum lies inside with gap <= 1e-10."""
    scipy_opt = pytest.importorskip("scipy.optimize")
    d = instance(0, m=12, n=10)
    a, b, C = d["a"], d["b"], d["C64"]
    m, n = C.shape
    A_eq = []
    for k in range(m):
        row = np.zeros((m, n)); row[k, :] = 1; A_eq.append(row.ravel())
    for i in range(n):
        col = np.zeros((m, n)); col[:, i] = 1; A_eq.append(col.ravel())
    lp = scipy_opt.linprog(C.ravel(), A_eq=np.array(A_eq), b_eq=np.r_[a, b], bounds=(0, None), method="highs")
    assert lp.status == 0
    for lam in (1e-3, 1.0):
        o = Oracle(a, b, lam, C=C)
        o.solve(BCPFW, 200000, seed=2, step=ELS, sampling=U, epsilon=1e-11)
        f = o.objective()
        assert o.gap()[0] <= 1e-10
        assert float((b * C.min(axis=0)).sum()) - 1e-12 <= f <= lp.fun + 1e-10


# --------------------------------------------------------------------------- exact-rational replay
def _rational_instance(m, n, seed):
    rs = np.random.default_rng(seed)
    X = rs.integers(0, 256, size=(m, 3)) / 255.0
    Y = rs.integers(0, 256, size=(n, 3)) / 255.0
    wa = rs.integers(1, 9, size=m); wb = rs.integers(1, 9, size=n)
    a = wa / wa.sum(); b = wb / wb.sum()
    # exact rationals for the replay: the fp64 values themselves (exactly representable)
    C = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(-1)
    return a, b, C


@pytest.mark.parametrize("rule,steps", [("dec", 300), ("els", 18)])
def test_exact_rational_replay_bcfw(rule, steps):
    """BCFW (Alg. 1) in exact rational arithmetic vs the fp64 oracle, same visit order:
    argmins identical, gammas and final T within 1e-13 (SURVEY 8c.11 'exact-rational replay')."""
    m, n = 5, 4
    a, b, C = _rational_instance(m, n, 42)
    lam = 0.25
    o = Oracle(a, b, lam, C=C)
    ex = ExactState(C, a, b, Fraction(1, 4))
    visit = np.random.default_rng(1).integers(0, n, size=steps)
    tr = o.solve(BCFW, steps, seed=0, visit=visit, trace=True, step=DEC if rule == "dec" else ELS,
                 sampling=U, epsilon=-1.0)["trace"]
    for k in range(steps):
        if ex.lmo_tied(int(visit[k])):
            assert rule == "els"       # decay steps never create exact ties
            break                      # exact tie: fp64 rounding decides from here on
        j, g = ex.bcfw_step(int(visit[k]), rule)
        assert tr["j"][k] == j, k
        assert abs(tr["gamma"][k] - float(g)) <= 1e-13 * max(1.0, float(g))
    else:
        Tex = np.array([[float(x) for x in row] for row in ex.T])
        assert np.abs(o.plan() - Tex).max() <= 1e-13
        assert abs(o.objective() - float(ex.f())) <= 1e-13
    assert k >= 5


@pytest.mark.parametrize("rule,steps", [("dec", 60), ("els", 8)])
def test_exact_rational_replay_fw(rule, steps):
    """FW (Alg. A.1 + Eq. A.1) in exact arithmetic vs the oracle's FW (U = [n])."""
    m, n = 4, 5
    a, b, C = _rational_instance(m, n, 7)
    o = Oracle(a, b, 0.5, C=C)
    ex = ExactState(C, a, b, Fraction(1, 2))
    tr = o.solve(FW, steps, seed=0, trace=True, step=DEC if rule == "dec" else ELS, epsilon=-1.0)["trace"]
    for k in range(steps):
        S, g = ex.fw_step(rule)
        assert tr["j"][k] == S[0]
        assert abs(tr["gamma"][k] - float(g)) <= 1e-13 * max(1.0, float(g))
    Tex = np.array([[float(x) for x in row] for row in ex.T])
    assert np.abs(o.plan() - Tex).max() <= 1e-13


@pytest.mark.parametrize("variant", [BCAFW, BCPFW])
def test_exact_rational_replay_away_pairwise(variant):
    """BCAFW (Alg. A.2) / BCPFW (Alg. A.3) with Eq. 14 in exact arithmetic vs the oracle."""
    m, n = 6, 5
    a, b, C = _rational_instance(m, n, 3)
    o = Oracle(a, b, 1.0, C=C)
    ex = ExactState(C, a, b, Fraction(1))
    steps = 12
    visit = np.random.default_rng(5).integers(0, n, size=steps)
    tr = o.solve(variant, steps, seed=0, visit=visit, trace=True, step=ELS, sampling=U, epsilon=-1.0)["trace"]
    kinds = {"fw": 0, "away": 1, "pair": 2, "noop": 3}
    compared = 0
    for k in range(steps):
        if ex.lmo_tied(int(visit[k])):
            break                      # exact ELS tie: fp64 rounding decides from here on
        j, v, g, kind = ex.away_or_pair_step(int(visit[k]), pairwise=(variant == BCPFW))
        assert tr["j"][k] == j and tr["v"][k] == v and tr["dir"][k] == kinds[kind], k
        assert abs(tr["gamma"][k] - float(g)) <= 1e-12 * max(1.0, float(g))
        compared += 1
    assert compared >= 3


# --------------------------------------------------------------------------- special cases
def test_n1_bcfw_equals_fw_bitwise():
    """n = 1: BCFW reduces to FW — identical traces under the decay rule."""
    d = instance(0, m=16, n=1)
    C = d["C64"]
    o1 = Oracle(d["a"], [1.0], 1.0, C=C)
    o2 = Oracle(d["a"], [1.0], 1.0, C=C)
    t1 = o1.solve(BCFW, 50, seed=3, trace=True, step=DEC, sampling=U, epsilon=-1.0)["trace"]
    t2 = o2.solve(FW, 50, seed=3, trace=True, step=DEC, epsilon=-1.0)["trace"]
    assert np.array_equal(t1["gamma"], t2["gamma"]) and np.array_equal(t1["j"], t2["j"])
    assert np.array_equal(o1.plan(), o2.plan())


def test_batched_B1_is_bcfw_and_Bn_is_fw():
    """Batched super-block step (R18): B = 1 reproduces BCFW and B = n reproduces FW bitwise."""
    d = instance(0, m=24, n=16)
    for rule in (DEC, ELS):
        o1 = Oracle(d["a"], d["b"], 1.0, C=d["C64"]); o2 = Oracle(d["a"], d["b"], 1.0, C=d["C64"])
        r1 = o1.solve(BCFW, 160, seed=9, trace=True, step=rule, sampling=P, epsilon=-1.0)
        r2 = o2.solve(BATCHED, 160, seed=9, trace=True, step=rule, sampling=P, block_size=1, epsilon=-1.0)
        assert np.array_equal(r1["trace"]["gamma"], r2["trace"]["gamma"])
        assert np.array_equal(o1.plan(), o2.plan())
        o3 = Oracle(d["a"], d["b"], 1.0, C=d["C64"]); o4 = Oracle(d["a"], d["b"], 1.0, C=d["C64"])
        r3 = o3.solve(FW, 30, seed=9, trace=True, step=rule, epsilon=-1.0)
        r4 = o4.solve(BATCHED, 30, seed=9, trace=True, step=rule, sampling=U, block_size=16, epsilon=-1.0)
        assert np.array_equal(r3["trace"]["gamma"], r4["trace"]["gamma"])
        assert np.array_equal(o3.plan(), o4.plan())


def test_batched_rank_map_is_G_invariant_for_FW_blocks():
    """Summation shapes (R19) align with rank shards: batched with B = n/G per rank and
    G ranks is the same column set U = [n] as FW, so all G give identical trajectories."""
    d = instance(0, m=20, n=32)
    ref = Oracle(d["a"], d["b"], 1.0, C=d["C64"])
    rr = ref.solve(FW, 25, seed=1, trace=True, step=ELS, epsilon=-1.0)
    for G in (2, 4, 8):
        o = Oracle(d["a"], d["b"], 1.0, C=d["C64"])
        r = o.solve(BATCHED, 25, seed=1, trace=True, step=ELS, sampling=U, block_size=32 // G, nranks=G,
                    epsilon=-1.0)
        assert np.array_equal(r["trace"]["gamma"], rr["trace"]["gamma"])
        assert np.array_equal(o.plan(), ref.plan())


# --------------------------------------------------------------------------- trajectory invariants
@pytest.mark.parametrize("variant,step,sampling", [
    (BCFW, ELS, U), (BCFW, DEC, P), (BCAFW, ELS, U), (BCPFW, ELS, P), (BCFW, ELS, GA), (FW, ELS, U), (FW, DEC, U),
    (BATCHED, ELS, P)])
def test_trajectory_invariants(variant, step, sampling):
    """Feasibility T^T 1 = b, T >= 0 (Eq. 8), |r - T1| <= 1e-10 (R6), monotone f under
    ELS, sparsity bound nnz(t_i) <= 1 + #visits of column i."""
    d = instance(1, m=40, n=32)
    o = Oracle(d["a"], d["b"], 1.0, C=d["C64"])
    kw = dict(block_size=8) if variant == BATCHED else {}
    fprev = o.objective()
    visits = np.zeros(32, dtype=int)
    for rnd in range(12):
        r = o.solve(variant, 16, seed=4, trace=True, step=step, sampling=sampling, epsilon=-1.0, **kw)
        for i in r["trace"]["i"]:
            visits[i] += 1
        T = o.plan()
        assert T.min() >= 0.0
        assert np.abs(T.sum(0) - d["b"]).max() <= 1e-10
        assert np.abs(o.r() - T.sum(1)).max() <= 1e-10
        f = o.objective()
        if step == ELS:
            assert f <= fprev + 1e-12 * abs(fprev)
        fprev = f
        if variant in (BCFW, BCPFW) and step == DEC:
            assert ((T > 0).sum(0) <= 1 + visits).all()


def test_resumable_solve_equals_single_call():
    """sro_solve semantics: two calls with a and b iterations equal one call with a+b."""
    d = instance(1, m=30, n=20)
    o1 = Oracle(d["a"], d["b"], 1.0, C=d["C64"]); o2 = Oracle(d["a"], d["b"], 1.0, C=d["C64"])
    o1.solve(BCAFW, 70, seed=5, step=ELS, sampling=U, epsilon=-1.0)
    o1.solve(BCAFW, 130, seed=5, step=ELS, sampling=U, epsilon=-1.0)
    o2.solve(BCAFW, 200, seed=5, step=ELS, sampling=U, epsilon=-1.0)
    assert np.array_equal(o1.plan(), o2.plan())


# --------------------------------------------------------------------------- samplers / RNG / sums
def test_splitmix64_reference_vector():
    """SplitMix64 (public-domain; R21): seeded with 0, the first three outputs are the
    published reference values 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F."""
    G = 0x9E3779B97F4A7C15
    outs = [splitmix64_mix((t * G) & 0xFFFFFFFFFFFFFFFF) for t in (1, 2, 3)]
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    x = rng_u64(7, 1, 12)
    assert uniform53(x) == (x >> 11) * 2.0 ** -53


def test_hash_cost_matches_generator_definition():
    """Config [3] cost C_ki = (splitmix64(seed, i m + k) >> 40) 2^-24: the oracle's
    on-the-fly value equals the independent numpy generator's."""
    m, n, seed = 64, 16, 0x5EED0003
    o = Oracle(np.full(m, 1 / m), np.full(n, 1 / n), 1.0, cost="hash", hash_seed=seed)
    rows, cols = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    ref = hash_uniform_cost(seed, m, rows.ravel(), cols.ravel()).reshape(m, n)
    got = np.array([[o.cost(k, i) for i in range(n)] for k in range(m)])
    assert np.array_equal(got, ref)
    assert (ref >= 0).all() and (ref < 1).all() and abs(ref.mean() - 0.5) < 0.05


def test_permutation_sampling_visits_each_column_once_per_epoch():
    """BCFW-P: each epoch is a fresh permutation of [n]."""
    d = instance(0, m=8, n=13)
    o = Oracle(d["a"], d["b"], 1.0, C=d["C64"])
    tr = o.solve(BCFW, 13 * 4, seed=11, trace=True, step=DEC, sampling=P, epsilon=-1.0)["trace"]
    for e in range(4):
        assert sorted(tr["i"][13 * e:13 * (e + 1)]) == list(range(13))
    perms = {tuple(permutation(11, e, 13)) for e in range(4)}
    assert len(perms) == 4


def test_fenwick_sampler_frequencies():
    """Alg. A.4 line 2: P(i) proportional to max(g_i, 0): 3-sigma multinomial
    bounds over 1e5 draws; a single positive weight is always drawn; all-zero -> uniform."""
    w = np.array([3.0, 1.0, 0.0, 0.0, 2.5, -1.0, 0.5])
    p = np.maximum(w, 0) / np.maximum(w, 0).sum()
    N = 100000
    us = [uniform53(rng_u64(99, 1, t)) for t in range(N)]
    cnt = np.bincount([fenwick_draw(w, u) for u in us], minlength=len(w))
    sig = np.sqrt(N * p * (1 - p))
    assert (np.abs(cnt - N * p) <= 3 * sig + 1e-9).all()
    assert cnt[2] == cnt[3] == cnt[5] == 0
    one = np.zeros(9); one[6] = 1e-3
    assert {fenwick_draw(one, u) for u in us[:500]} == {6}
    zeros = np.zeros(5)
    cz = np.bincount([fenwick_draw(zeros, u) for u in us[:5000]], minlength=5)
    assert (cz > 800).all()


def test_chunk_tree_sum_shape():
    """R19 summation shape: W contiguous chunks [floor(cL/W), floor((c+1)L/W)) summed
    left to right, combined by adjacent pairs. Hand example where order matters, and
    agreement with the exactly rounded sum (math.fsum) within the pairwise error bound."""
    # L = 4, W = 2: ((1e16 + 1) + 0) ... chunk0 = 1e16 + 1 -> 1e16 (ties-to-even), chunk1 = -1e16 + 1
    x = [1e16, 1.0, -1e16, 1.0]
    assert chunk_tree_sum(x, 2) == (1e16 + 1.0) + (-1e16 + 1.0)
    assert chunk_tree_sum(x, 1) == ((1e16 + 1.0) + -1e16) + 1.0
    # W = 8 over L = 3: chunks 2,5,7 hold one element each -> ((0+0)+(0+x0)) ... adjacent pairs
    y = [0.1, 0.2, 0.3]
    c = [0.0] * 8
    for p in range(3):
        for cc in range(8):
            if (cc * 3) // 8 <= p < ((cc + 1) * 3) // 8:
                c[cc] = y[p]
    expect = ((c[0] + c[1]) + (c[2] + c[3])) + ((c[4] + c[5]) + (c[6] + c[7]))
    assert chunk_tree_sum(y, 8) == expect
    rs = np.random.default_rng(0)
    for L in (1, 7, 255, 256, 1000, 65537):
        z = rs.standard_normal(L)
        s = chunk_tree_sum(z, 256)
        assert abs(s - math.fsum(z)) <= 1e-15 * (L / 256 + 8) * np.abs(z).sum()


# --------------------------------------------------------------------------- Theorem 1, qualitative claims
def test_theorem1_decay_envelope_over_seeds():
    """Theorem 1 (proof P:2213-2223): with the decay step 2n/(k+2n) and uniform
    sampling, E[f(T^k)] - f* <= 2n/(k+2n) (C_f^x + h0), with the product curvature
    C_f^x = sum_i C_f^(i) <= sum_i 4 b_i^2 / lambda (Def. 1 / App. C) and
    h0 = f(T^0) - f*. The expectation is the mean over 20 seeds; f* comes from a long ELS run
    whose certified gap bounds its own suboptimality (Thm 2)."""
    d = instance(1, m=24, n=16, seed=6)
    lam = 0.5
    ref = Oracle(d["a"], d["b"], lam, C=d["C64"], cap=24)
    ref.solve(BCPFW, 5000 * 16, seed=1, step=ELS, sampling=U, epsilon=1e-10)   # pairwise: fast to 1e-10
    g = ref.gap()[0]
    assert 0.0 <= g <= 1e-6
    fstar = ref.objective() - g                      # f* >= f(T) - g(T) (Thm 2): conservative
    n = 16
    o0 = Oracle(d["a"], d["b"], lam, C=d["C64"], cap=24)
    h0 = o0.objective() - fstar
    Cx = float((4.0 * d["b"] ** 2 / lam).sum())
    checkpoints = [n, 4 * n, 16 * n, 64 * n]
    subopt = np.zeros((20, len(checkpoints)))
    for s in range(20):
        o = Oracle(d["a"], d["b"], lam, C=d["C64"], cap=24)
        done = 0
        for c, k in enumerate(checkpoints):
            o.solve(BCFW, k - done, seed=100 + s, step=DEC, sampling=U, epsilon=-1.0)
            done = k
            subopt[s, c] = o.objective() - fstar
    for c, k in enumerate(checkpoints):
        assert subopt[:, c].mean() <= 2.0 * n / (k + 2.0 * n) * (Cx + h0)
    assert (subopt >= -1e-12).all()
    assert subopt[:, -1].mean() < subopt[:, 0].mean()


def test_pairwise_needs_fewer_epochs_than_bcfw_u():
    """Qualitative claim: BCPFW reaches the gap threshold in fewer epochs than
    BCFW-U with the line search (median over seeds; scratch at m = n = 256: 123 vs 250)."""
    d = instance(1, m=96, n=96, seed=7)
    ep = {BCFW: [], BCPFW: []}
    for seed in range(5):
        for var in (BCFW, BCPFW):
            o = Oracle(d["a"], d["b"], 1.0, C=d["C64"], cap=31)
            r = o.solve(var, 3000 * 96, seed=seed, step=ELS, sampling=U, epsilon=1e-6)
            assert r["converged"]
            ep[var].append(r["iters_done"] / 96)
    assert np.median(ep[BCPFW]) < np.median(ep[BCFW])
