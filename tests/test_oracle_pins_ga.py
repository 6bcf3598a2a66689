"""Pins of the oracle's gap-adaptive sampler (Alg. A.4) and of its colour cost
kinds, against definitions written independently of the oracle's C code.

* The GA trajectory — draws, stored gaps, inner refresh (after the update, or before it),
  global refresh every M n steps, GAS — is replayed in exact rational arithmetic straight from
  the paper (tests/exact_replay.py::ga_replay: the O(n) cumulative-sum draw of P:407, not a
  tree) on the same u53 stream; the oracle must draw the same columns, take the same argmins
  and step sizes, and end with the same stored gaps.
* The Fenwick tree's point updates (the oracle's fen_add, used by every inner refresh) are
  checked against the cumulative sum of the updated weights and, draw by draw, against the
  plain "smallest i with prefix_i > u W" rule.
* C_ki for the squared-Euclidean and Euclidean colour costs, in binary64 and in binary32
  (R10: ((dx dx + dy dy) + dz dz) evaluated in the storage precision), equals numpy's
  evaluation of the same definition.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

from oracle import BCAFW, BCFW, BCPFW, DEC, ELS, GA, Oracle, fenwick_updates
from tests.exact_replay import ExactState, _mix, ga_replay, u53_exact


def _rational_instance(m, n, seed):
    rs = np.random.default_rng(seed)
    X = rs.integers(0, 256, size=(m, 3)) / 255.0
    Y = rs.integers(0, 256, size=(n, 3)) / 255.0
    wa = rs.integers(1, 9, size=m)
    wb = rs.integers(1, 9, size=n)
    a = wa / wa.sum()
    b = wb / wb.sum()
    C = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(-1)
    return a, b, C


def test_python_splitmix_matches_published_vector():
    """The replay's own SplitMix64 (exact_replay._mix) reproduces the published reference
    outputs for seed 0, so its u53 stream is pinned independently of the oracle's RNG."""
    G = 0x9E3779B97F4A7C15
    assert [_mix((t * G) & ((1 << 64) - 1)) for t in (1, 2, 3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                                     0x06C45D188009454F]
    from oracle import rng_u64, uniform53
    for t in range(50):
        assert float(u53_exact(123, 1, t)) == uniform53(rng_u64(123, 1, t))


GA_CASES = [
    # (id, variant, oracle variant, rule, M, inner, post, steps, min compared)
    ("gad-m1-post-dec", "plain", BCFW, "dec", 1, 1, 1, 400, 400),
    ("gad-m1-pre-dec", "plain", BCFW, "dec", 1, 1, 0, 400, 400),
    ("gad-m2-post-dec", "plain", BCFW, "dec", 2, 1, 1, 400, 400),
    ("gas-dec", "plain", BCFW, "dec", 1, 0, 0, 400, 400),
    ("gad-m1-post-els", "plain", BCFW, "els", 1, 1, 1, 18, 6),
    ("gad-m1-pre-els", "plain", BCFW, "els", 1, 1, 0, 18, 6),
    ("gad-m2-post-els", "plain", BCFW, "els", 2, 1, 1, 18, 6),
    ("gas-els", "plain", BCFW, "els", 1, 0, 0, 18, 6),
    ("ga-away", "away", BCAFW, "els", 1, 1, 1, 18, 5),
    ("ga-pairwise", "pair", BCPFW, "els", 1, 1, 1, 18, 5),
]


@pytest.mark.parametrize("case", GA_CASES, ids=[c[0] for c in GA_CASES])
def test_exact_rational_replay_ga(case):
    """Alg. A.4 in exact arithmetic vs the fp64 oracle: the same drawn column i, argmin j, away
    atom v and gamma at every step (up to the first exact tie, which fp64 rounding decides), and
    after the compared steps the same stored gaps G_i (to 1e-13) with the tree's prefix sums
    equal to the cumulative sums of max(G_i, 0) (to 1e-13). A sign error in the Fenwick delta,
    a refresh at the wrong step or the wrong refresh state changes the draws within a few steps."""
    _, variant, ov, rule, M, inner, post, steps, need = case
    m, n = 5, 4
    lam = Fraction(1, 4)
    a, b, C = _rational_instance(m, n, 17)
    seed = 31
    ex = ExactState(C, a, b, lam)
    cinit = Fraction(float(C.max())) + 2 / lam                     # R14: max C + 2 / lambda
    rec = ga_replay(ex, variant, steps, seed, M, inner, post, cinit, rule=rule)
    assert len(rec) >= need, len(rec)
    o = Oracle(a, b, float(lam), C=C)
    kw = dict(step=DEC if rule == "dec" else ELS, sampling=GA, ga_M=M, ga_inner=inner, ga_post_update=post)
    tr = o.solve(ov, len(rec), seed=seed, trace=True, epsilon=-1.0, **kw)["trace"]
    kinds = {"fw": 0, "away": 1, "pair": 2, "noop": 3}
    for r in rec:
        k = r["k"]
        assert tr["i"][k] == r["i"], (k, tr["i"][k], r["i"])
        assert tr["j"][k] == r["j"], k
        if variant != "plain":
            assert tr["v"][k] == r["v"] and tr["dir"][k] == kinds[r["kind"]], k
        assert abs(tr["gamma"][k] - float(r["gamma"])) <= 1e-13 * max(1.0, float(r["gamma"])), k
    G, prefix = o.ga_state()
    Gex = np.array([float(x) for x in rec[-1]["G"]])
    assert np.abs(G - Gex).max() <= 1e-13 * max(1.0, np.abs(Gex).max())
    w = [x if x > 0 else Fraction(0) for x in rec[-1]["G"]]
    cum = np.array([float(sum(w[:i + 1])) for i in range(n)])
    assert np.abs(prefix - cum).max() <= 1e-13 * max(1.0, cum[-1])
    Tex = np.array([[float(x) for x in row] for row in ex.T])
    assert np.abs(o.plan() - Tex).max() <= 1e-13


def test_ga_global_refresh_happens_every_Mn_steps():
    """every M n steps all stored gaps become the true g_i(T). With GAS (no inner
    refresh) the stored gaps between refreshes stay those of the last refresh: after a multiple
    of n steps they equal the oracle's own per-column gaps exactly; one step later they still
    do for every column (nothing refreshed them), while the plan has moved."""
    m, n = 7, 6
    a, b, C = _rational_instance(m, n, 3)
    o = Oracle(a, b, 1.0, C=C)
    o.solve(BCFW, 2 * n, seed=4, step=ELS, sampling=GA, ga_M=1, ga_inner=0, ga_post_update=0, epsilon=-1.0)
    G, _ = o.ga_state()
    _, g, _, _ = o.gap()
    assert np.array_equal(G, g)
    o.solve(BCFW, 1, seed=4, step=ELS, sampling=GA, ga_M=1, ga_inner=0, ga_post_update=0, epsilon=-1.0)
    G1, _ = o.ga_state()
    assert np.array_equal(G1, G)


def test_fenwick_point_updates_match_cumulative_sums_and_draw_rule():
    """The tree after 400 point updates (some to negative or zero stored gaps, R17): every
    prefix equals the cumulative sum of max(G_i, 0) of the updated weights to 1e-12 W; every
    one of 20000 draws is the smallest i with cumsum_i > u W (away from rounding boundaries),
    and the draw frequencies follow the updated weights within 3 sigma."""
    rs = np.random.default_rng(5)
    n = 37
    w0 = rs.random(n) * 3 - 0.5
    idx = rs.integers(0, n, size=400)
    newv = rs.random(400) * 2 - 0.4
    newv[rs.random(400) < 0.1] = 0.0
    final = w0.copy()
    for i, v in zip(idx, newv):
        final[i] = v
    wpos = np.maximum(final, 0.0)
    cum = np.cumsum(wpos)
    W = cum[-1]
    us = np.array([float(u53_exact(77, 1, t)) for t in range(20000)])
    prefix, draws = fenwick_updates(w0, idx, newv, us)
    assert np.abs(prefix - cum).max() <= 1e-12 * W
    checked = 0
    for u, dr in zip(us, draws):
        uw = u * W
        if np.min(np.abs(cum - uw)) <= 1e-9 * W:
            continue
        assert dr == int(np.argmax(cum > uw)), (u, dr)
        checked += 1
    assert checked > 19900
    p = wpos / W
    cnt = np.bincount(draws, minlength=n)
    sig = np.sqrt(len(us) * p * (1 - p))
    assert (np.abs(cnt - len(us) * p) <= 3 * sig + 1e-9).all()
    assert (cnt[wpos == 0] == 0).all()


# --------------------------------------------------------------------------- cost kinds
@pytest.mark.parametrize("cost", ["sqeuclid", "euclid"])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_colour_cost_kinds_match_numpy(cost, prec):
    """C_ki of the colour costs (R10; P:427 Euclidean, BASELINE configs squared): the oracle's
    value equals numpy's evaluation of d = x_k - y_i, ((d0 d0 + d1 d1) + d2 d2) (and its square
    root for the Euclidean kind) in the storage precision, promoted exactly to binary64."""
    rs = np.random.default_rng(11)
    m, n = 40, 30
    X = rs.random((m, 3))
    Y = rs.random((n, 3))
    X[3] = Y[5]                         # a zero-cost pair (sqrt(0), exact ties)
    o = Oracle(np.full(m, 1 / m), np.full(n, 1 / n), 1.0, X=X, Y=Y, cost=cost, prec=prec)
    ft = np.float32 if prec == "f32" else np.float64
    Xs, Ys = X.astype(ft), Y.astype(ft)
    d = Xs[:, None, :] - Ys[None, :, :]
    sq = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
    ref = (np.sqrt(sq) if cost == "euclid" else sq).astype(np.float64)
    got = np.array([[o.cost(k, i) for i in range(n)] for k in range(m)])
    assert np.array_equal(got, ref)
    assert got[3, 5] == 0.0
    if prec == "f32":      # binary32 evaluation really differs from binary64 somewhere
        d64 = X[:, None, :] - Y[None, :, :]
        sq64 = (d64[..., 0] ** 2 + d64[..., 1] ** 2) + d64[..., 2] ** 2
        assert not np.array_equal(got, np.sqrt(sq64) if cost == "euclid" else sq64)
