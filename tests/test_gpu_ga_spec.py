"""GPU parity of the GA pipe's speculative next column (k_bcfw_pipe.cuh):
the candidate drawn from the tree before the refresh, its pre-scan over the rows
outside its support and T_s, and the fix-up of T_s's rows after the draw must give
exactly the trajectory of the plain scan (SRO_NO_SPEC) and of the oracle (Alg. A.4,
P:1848-1869). Tiny n makes redraws of the same column (no pre-scan) and misses frequent;
ragged m puts T_s rows in the tail lane; m = 4096 fp32 is the bench's instantiation."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import BCAFW, BCFW, BCPFW, ELS, GA, Oracle
from sro_inputs import instance

pytestmark = pytest.mark.gpu

sro = pytest.importorskip("paper_2103_05857_b200")

GA_M1 = dict(step=ELS, sampling=GA, ga_M=1, ga_inner=1, ga_post_update=1)
VARS = [(BCFW, sro.SRO_BCFW, GA_M1), (BCAFW, sro.SRO_BCAFW, GA_M1), (BCPFW, sro.SRO_BCPFW, GA_M1),
        (BCFW, sro.SRO_BCFW, dict(step=ELS, sampling=GA, ga_M=3, ga_inner=1, ga_post_update=0))]


def _instance(m, n, seed, prec):
    d = instance(1, m=m, n=n, seed=seed)
    C = ((d["X"][:, None, :] - d["Y"][None, :, :]) ** 2).sum(-1)
    C = C.astype(np.float32).astype(np.float64) if prec == "f32" else C
    return d, C


def _run(d, C, prec, ov, gv, kw, iters, seed):
    Cc = C.astype(np.float32) if prec == "f32" else C
    o = Oracle(d["a"], d["b"], 1.0, C=Cc, prec=prec, cap=31)
    ro = o.solve(ov, iters, seed=seed, trace=True, epsilon=1e-12, **kw)
    g = sro.Solver(d["a"], d["b"], 1.0, C=Cc, prec=prec, slab_cap=31)
    rg = g.solve(gv, iters, seed=seed, trace=True, epsilon=1e-12, **kw)
    out = (rg["trace"], g.plan(), g.rowsums(), rg["gap"])
    exp = (ro["trace"], o.plan(), o.r(), ro["gap"])
    g.close()
    return out, exp


def _check(out, exp):
    tg, to = out[0], exp[0]
    assert len(tg) == len(to)
    for f in ("k", "i", "j", "v", "dir", "gamma", "num", "den", "minval"):
        bad = np.nonzero(tg[f] != to[f])[0]
        assert len(bad) == 0, f"{f} differs first at step {bad[0]}: gpu {tg[bad[0]]} oracle {to[bad[0]]}"
    assert np.array_equal(out[1], exp[1]) and np.array_equal(out[2], exp[2])
    assert out[3] == exp[3] or (np.isnan(out[3]) and np.isnan(exp[3]))


@pytest.mark.parametrize("spec", [True, False], ids=["spec", "nospec"])
@pytest.mark.parametrize("vi", range(len(VARS)), ids=["bcfw-m1", "bcafw-m1", "bcpfw-m1", "bcfw-m3-pre"])
@pytest.mark.parametrize("m,n,prec", [(40, 2, "f64"), (41, 3, "f64"), (257, 5, "f32"), (1031, 17, "f32"),
                                      (4099, 64, "f32")])
def test_ga_spec_bitexact(monkeypatch, spec, vi, m, n, prec):
    if not spec:
        monkeypatch.setenv("SRO_NO_SPEC", "1")
    ov, gv, kw = VARS[vi]
    d, C = _instance(m, n, 5 + m + n, prec)
    out, exp = _run(d, C, prec, ov, gv, kw, 40 * n + 37, seed=3)
    _check(out, exp)


@pytest.mark.parametrize("ov,gv", [(BCFW, sro.SRO_BCFW), (BCPFW, sro.SRO_BCPFW)], ids=["bcfw", "bcpfw"])
def test_ga_spec_bench_shape(monkeypatch, ov, gv):
    """m = 4096 fp32 (k_bcfw_ga_pipe<float, 3, ·>, the bench's instantiation), n = 1024, two
    epochs: speculation on equals the oracle and equals speculation off."""
    d, C = _instance(4096, 1024, 21, "f32")
    out, exp = _run(d, C, "f32", ov, gv, GA_M1, 2 * 1024, seed=9)
    _check(out, exp)
    monkeypatch.setenv("SRO_NO_SPEC", "1")
    out2, _ = _run(d, C, "f32", ov, gv, GA_M1, 2 * 1024, seed=9)
    _check(out2, exp)
