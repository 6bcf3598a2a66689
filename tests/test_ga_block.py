"""Gap-adaptive sampling for batched BCFW (R31): the block of a
column drawn from the Fenwick tree over the stored column gaps (Alg. A.4's sampler),
the block's stored gaps refreshed after the step, the global refresh every M n' block steps.

CPU: the oracle's extension is pinned to Alg. A.4 itself — with B = 1 a batched GA run is the
BCFW-GA run step for step — and its block frequencies follow the summed block gaps. GPU: the
device path (draw kernel, cursor-mode steps, refresh kernel) bit-exact against the oracle."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import BATCHED, BCFW, ELS, GA, Oracle, fenwick_draw, rng_u64, uniform53
from sro_inputs import instance


@pytest.mark.parametrize("inner,post,M", [(1, 1, 1), (1, 0, 2), (0, 0, 1)])
def test_block_size_one_is_bcfw_ga(inner, post, M):
    d = instance(1, m=40, n=24, seed=3)
    kw = dict(step=ELS, sampling=GA, ga_M=M, ga_inner=inner, ga_post_update=post)
    o1 = Oracle(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", cap=31)
    o2 = Oracle(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", cap=31)
    r1 = o1.solve(BCFW, 6 * 24, seed=5, trace=True, epsilon=-1.0, **kw)
    r2 = o2.solve(BATCHED, 6 * 24, seed=5, trace=True, epsilon=-1.0, block_size=1, **kw)
    for f in ("i", "j", "gamma", "num", "den", "minval"):
        assert np.array_equal(r1["trace"][f], r2["trace"][f]), f
    assert np.array_equal(o1.plan(), o2.plan()) and r1["gap"] == r2["gap"]


def test_block_draw_frequencies_follow_summed_gaps():
    """The block of a Fenwick-drawn column: P(block) = sum of its columns' weights / total."""
    rng = np.random.default_rng(1)
    n, B = 48, 8
    w = rng.random(n) ** 3
    w[8:16] = 0.0                                  # a block with no weight is never drawn
    counts = np.zeros(n // B)
    N = 60000
    for t in range(N):
        counts[fenwick_draw(w, uniform53(rng_u64(99, 1, t))) // B] += 1
    p = w.reshape(-1, B).sum(1) / w.sum()
    assert counts[1] == 0
    assert np.abs(counts / N - p).max() <= 4 * np.sqrt(p.max() / N)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,B,inner,post,M", [(256, 256, 16, 1, 1, 1), (300, 512, 64, 1, 0, 1),
                                                 (4096, 1024, 256, 1, 1, 2), (700, 640, 32, 0, 0, 1),
                                                 (65, 96, 96, 1, 1, 1)])
def test_gpu_batched_ga_bitexact(m, n, B, inner, post, M):
    sro = pytest.importorskip("paper_2103_05857_b200")
    d = instance(1, m=m, n=n, seed=4)
    kw = dict(step=ELS, sampling=GA, ga_M=M, ga_inner=inner, ga_post_update=post, block_size=B)
    C = d["C32"]
    g = sro.Solver(d["a"], d["b"], 1.0, C=C, prec="f32")
    o = Oracle(d["a"], d["b"], 1.0, C=C, prec="f32", cap=31)
    iters = 5 * (n // B) + 3
    ro = o.solve(BATCHED, iters, seed=7, trace=True, epsilon=-1.0, **kw)
    rg = g.solve(sro.SRO_BATCHED, iters, seed=7, trace=True, epsilon=-1.0, **kw)
    assert rg["iters_done"] == ro["iters_done"] and rg["gap"] == ro["gap"]
    assert rg["entries_scanned"] == ro["entries_scanned"]
    for f in ("k", "i", "j", "gamma", "num", "den", "minval"):
        assert np.array_equal(rg["trace"][f], ro["trace"][f]), f
    assert np.array_equal(g.plan(), o.plan())
    assert np.array_equal(g.rowsums(), o.r())


@pytest.mark.gpu
def test_gpu_batched_ga_converges_before_permutation_sampling():
    """m = n = 512, B = 16: block GA (GAD-M1, post-update refresh) reaches g <= 1e-6 within 400
    epochs (certified by a fresh gap sweep) and no later than permutation sampling does."""
    sro = pytest.importorskip("paper_2103_05857_b200")
    d = instance(1, m=512, n=512, seed=6)
    res = {}
    for samp in (sro.SAMPLE_GA, sro.SAMPLE_P):
        g = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
        r = g.solve(sro.SRO_BATCHED, 400 * 32, seed=1, step=sro.STEP_ELS, sampling=samp, ga_M=1, ga_inner=1,
                    ga_post_update=1, block_size=16, epsilon=1e-6)
        res[samp] = r
        if samp == sro.SAMPLE_GA:
            assert r["converged"] == 1 and r["gap"] <= 1e-6
            total, _, _ = g.gap()
            assert total <= 1e-6
    assert res[sro.SAMPLE_GA]["iters_done"] <= res[sro.SAMPLE_P]["iters_done"]
