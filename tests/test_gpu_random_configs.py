"""Randomised GPU parity sweep (fixed seeds, so reproducible): 400 configurations (SRO_FUZZ_N) drawn over the
option space the C-ABI accepts — variant (BCFW / BCAFW / BCPFW / FW / batched), step rule, sampling
(U / P / GA with M, inner refresh and its timing), gap period, cost kind (dense fp32 / fp64, fused
sqeuclid / euclid in binary32 / binary64, hash), slab capacity, lambda over four decades, marginals
with zero-mass columns and zero rows, and ragged m, n (several tiles, vector tails, block sizes
dividing n) — each run for a few epochs through sro_solve and compared with the oracle step by step
(Alg. 1, A.1-A.4, R18): trace, plan, row sums, gap and objective bit-exact, or the same error
status (capacity) at the same step."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import BATCHED, BCAFW, BCFW, BCPFW, DEC, ELS, FW, GA, P, U, Oracle, OracleError
from sro_inputs import mixture_colours

pytestmark = pytest.mark.gpu

sro = pytest.importorskip("paper_2103_05857_b200")

GV = {BCFW: sro.SRO_BCFW, BCAFW: sro.SRO_BCAFW, BCPFW: sro.SRO_BCPFW, FW: sro.SRO_FW, BATCHED: sro.SRO_BATCHED}


def _config(seed):
    rs = np.random.default_rng(1000 + seed)
    # m over the persistent kernels' dispatch edges too (vectors per LMO thread: 384 pipe / 480 GA-pipe
    # threads x 4 fp32 or 2 fp64 entries per vector; register-file and shared-memory fallbacks above)
    m = int(rs.choice([1, 7, 64, 129, 300, 511, 768, 769, 1030, 1536, 1537, 1920, 1921, 2500, 3072, 3073, 3840,
                       3841, 4096, 6001, 6144, 6145, 7680, 7681, 9000, 16385]))
    n = int(rs.choice([1, 5, 33, 64, 96, 200, 257, 512, 1100]))
    variant = int(rs.choice([BCFW, BCAFW, BCPFW, FW, BATCHED]))
    step = ELS if variant in (BCAFW, BCPFW) else int(rs.choice([ELS, DEC]))
    sampling = int(rs.choice([U, P, GA])) if variant != FW else U
    opts = dict(step=step, sampling=sampling, gap_period=int(rs.choice([1, 1, 2])))
    if sampling == GA:
        opts.update(ga_M=int(rs.choice([1, 2])), ga_inner=int(rs.choice([0, 1])), ga_post_update=int(rs.choice([0, 1])))
    if variant == BATCHED:
        divs = [b for b in range(1, n + 1) if n % b == 0]
        opts["block_size"] = int(rs.choice(divs))
    cost = str(rs.choice(["dense32", "dense64", "sq32", "sq64", "eu32", "eu64", "hash"]))
    lam = float(rs.choice([1e-2, 1e-1, 1.0, 10.0]))
    cap = int(rs.choice([4, 8, 31]))
    X, _, _ = mixture_colours(m, 4, 0.05, 2 * seed + 1)
    Y, _, _ = mixture_colours(n, 4, 0.05, 2 * seed + 2)
    a = rs.random(m) + 0.05
    b = rs.random(n) + 0.05
    if m > 3 and rs.random() < 0.3:
        a[rs.integers(0, m, size=max(1, m // 5))] = 0.0
    if n > 3 and rs.random() < 0.3:
        b[rs.integers(0, n, size=max(1, n // 6))] = 0.0
    a /= a.sum()
    b /= b.sum()
    epochs = 3 if variant != FW else 12
    iters = epochs * (n // opts.get("block_size", 1) if variant == BATCHED else (1 if variant == FW else n))
    if m * n > 2_000_000 and variant != FW:
        epochs = 1
        iters = n // opts.get("block_size", 1) if variant == BATCHED else n
    return dict(m=m, n=n, variant=variant, opts=opts, cost=cost, lam=lam, cap=cap, X=X, Y=Y, a=a, b=b,
                iters=max(1, iters), seed=int(rs.integers(0, 1 << 30)))


def _make(cfg):
    m, n, c = cfg["m"], cfg["n"], cfg["cost"]
    kw = dict(cap=cfg["cap"])
    if c.startswith("dense"):
        C = ((cfg["X"][:, None, :] - cfg["Y"][None, :, :]) ** 2).sum(-1)
        prec = "f32" if c == "dense32" else "f64"
        Cs = C.astype(np.float32) if prec == "f32" else C
        g = sro.Solver(cfg["a"], cfg["b"], cfg["lam"], C=Cs, prec=prec, slab_cap=cfg["cap"])
        o = Oracle(cfg["a"], cfg["b"], cfg["lam"], C=np.asarray(Cs, dtype=np.float64), prec=prec, **kw)
    elif c == "hash":
        g = sro.Solver(cfg["a"], cfg["b"], cfg["lam"], cost="hash", hash_seed=77, slab_cap=cfg["cap"])
        o = Oracle(cfg["a"], cfg["b"], cfg["lam"], cost="hash", hash_seed=77, **kw)
    else:
        kind = "sqeuclid" if c.startswith("sq") else "euclid"
        prec = "f32" if c.endswith("32") else "f64"
        g = sro.Solver(cfg["a"], cfg["b"], cfg["lam"], X=cfg["X"], Y=cfg["Y"], cost=kind, prec=prec,
                       slab_cap=cfg["cap"])
        o = Oracle(cfg["a"], cfg["b"], cfg["lam"], X=cfg["X"], Y=cfg["Y"], cost=kind, prec=prec, **kw)
    return g, o


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("SRO_FUZZ_N", "400"))))
def test_random_configuration_bitexact(seed):
    cfg = _config(seed)
    g, o = _make(cfg)
    v, opts, iters = cfg["variant"], cfg["opts"], cfg["iters"]
    err_o = err_g = None
    ro = rg = None
    try:
        ro = o.solve(v, iters, seed=cfg["seed"], trace=True, epsilon=1e-12, **opts)
    except OracleError as e:
        err_o = e.status
    try:
        rg = g.solve(GV[v], iters, seed=cfg["seed"], trace=True, epsilon=1e-12, **opts)
    except sro.SroError as e:
        err_g = e.status
    assert err_o == err_g, (cfg["variant"], opts, err_o, err_g)
    if err_o is None:
        for f in ("k", "i", "j", "v", "dir", "gamma", "num", "den", "minval"):
            if v in (FW, BATCHED) and f in ("v", "dir"):
                continue
            bad = np.nonzero(rg["trace"][f] != ro["trace"][f])[0]
            assert len(bad) == 0, (f, bad[0], {k: cfg[k] for k in ("m", "n", "variant", "opts", "cost", "lam", "cap")})
        assert rg["iters_done"] == ro["iters_done"] and rg["gap_checks"] == ro["gap_checks"]
        assert rg["gap"] == ro["gap"] or (np.isnan(rg["gap"]) and np.isnan(ro["gap"]))
    assert np.array_equal(g.plan(), o.plan())
    assert np.array_equal(g.rowsums(), o.r())
    assert g.objective() == o.objective()
    tg, gg, jg = g.gap()
    to, go, jo, _ = o.gap()
    assert tg == to and np.array_equal(gg, go) and np.array_equal(jg, jo)


def _sharded_config(seed):
    rs = np.random.default_rng(5000 + seed)
    G = int(rs.choice([2, 4, 8]))
    m = int(rs.choice([1, 7, 129, 511, 1030, 4096, 9000]))
    n = G * int(rs.choice([1, 3, 8, 16, 33, 64]))
    variant = int(rs.choice([FW, BATCHED]))
    step = int(rs.choice([ELS, DEC]))
    opts = dict(step=step, gap_period=int(rs.choice([1, 2])))
    Bo = 0
    if variant == BATCHED:
        divs = [b for b in range(G, n + 1, G) if n % b == 0]
        Bo = int(rs.choice(divs))
        opts["block_size"] = Bo
        opts["sampling"] = int(rs.choice([U, P, GA]))
        if opts["sampling"] == GA:
            opts.update(ga_M=int(rs.choice([1, 2])), ga_inner=int(rs.choice([0, 1])),
                        ga_post_update=int(rs.choice([0, 1])))
    cost = str(rs.choice(["dense32", "dense64", "sq32", "eu64", "hash"]))
    lam = float(rs.choice([1e-1, 1.0, 10.0]))
    cap = int(rs.choice([4, 31]))
    X, _, _ = mixture_colours(m, 4, 0.05, 2 * seed + 101)
    Y, _, _ = mixture_colours(n, 4, 0.05, 2 * seed + 102)
    a = rs.random(m) + 0.05
    b = rs.random(n) + 0.05
    if n > 3 and rs.random() < 0.3:
        b[rs.integers(0, n, size=max(1, n // 6))] = 0.0
    a /= a.sum()
    b /= b.sum()
    iters = 10 if variant == FW else 3 * (n // Bo)
    split = int(rs.integers(0, iters + 1))
    return dict(G=G, m=m, n=n, variant=variant, opts=opts, Bo=Bo, cost=cost, lam=lam, cap=cap, X=X, Y=Y, a=a, b=b,
                iters=iters, split=split, seed=int(rs.integers(0, 1 << 30)))


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("SRO_FUZZ_SHARDED_N", "150"))))
def test_random_sharded_configuration_bitexact(seed):
    """Column-sharded FW / batched (one process holding G = 2, 4, 8 shards) over
    random options, costs, capacities and zero-mass columns, the solve split into two calls at a
    random point (the calls must compose, sro.h): plan, row sums, gap, objective and the gap
    checks equal the UNSHARDED oracle's, or the same error status."""
    cfg = _sharded_config(seed)
    c = cfg["cost"]
    kw = dict(shards=cfg["G"], shard_block=cfg["Bo"], slab_cap=cfg["cap"])
    if c.startswith("dense"):
        C = ((cfg["X"][:, None, :] - cfg["Y"][None, :, :]) ** 2).sum(-1)
        prec = "f32" if c == "dense32" else "f64"
        Cs = C.astype(np.float32) if prec == "f32" else C
        g = sro.Solver(cfg["a"], cfg["b"], cfg["lam"], C=Cs, prec=prec, **kw)
        o = Oracle(cfg["a"], cfg["b"], cfg["lam"], C=np.asarray(Cs, dtype=np.float64), prec=prec, cap=cfg["cap"])
    elif c == "hash":
        g = sro.Solver(cfg["a"], cfg["b"], cfg["lam"], cost="hash", hash_seed=91, **kw)
        o = Oracle(cfg["a"], cfg["b"], cfg["lam"], cost="hash", hash_seed=91, cap=cfg["cap"])
    else:
        kind = "sqeuclid" if c.startswith("sq") else "euclid"
        prec = "f32" if c.endswith("32") else "f64"
        g = sro.Solver(cfg["a"], cfg["b"], cfg["lam"], X=cfg["X"], Y=cfg["Y"], cost=kind, prec=prec, **kw)
        o = Oracle(cfg["a"], cfg["b"], cfg["lam"], X=cfg["X"], Y=cfg["Y"], cost=kind, prec=prec, cap=cfg["cap"])
    v, opts = cfg["variant"], cfg["opts"]
    err_o = err_g = None
    outs_o, outs_g = [], []
    for part in (cfg["split"], cfg["iters"] - cfg["split"]):
        try:
            if err_o is None:
                outs_o.append(o.solve(v, part, seed=cfg["seed"], epsilon=1e-12, **opts))
        except OracleError as e:
            err_o = e.status
        try:
            if err_g is None:
                outs_g.append(g.solve(GV[v], part, seed=cfg["seed"], epsilon=1e-12, **opts))
        except sro.SroError as e:
            err_g = e.status
    assert err_o == err_g, ({k: cfg[k] for k in ("G", "m", "n", "variant", "opts", "cost", "cap")}, err_o, err_g)
    for ro, rg in zip(outs_o, outs_g):
        assert rg["iters_done"] == ro["iters_done"] and rg["gap_checks"] == ro["gap_checks"]
        assert rg["gap"] == ro["gap"] or (np.isnan(rg["gap"]) and np.isnan(ro["gap"]))
    assert np.array_equal(g.plan(), o.plan())
    assert np.array_equal(g.rowsums(), o.r())
    assert g.objective() == o.objective()
    tg, gg, jg = g.gap()
    to, go, jo, _ = o.gap()
    assert tg == to and np.array_equal(gg, go) and np.array_equal(jg, jo)


@pytest.mark.parametrize("seed", range(40))
def test_random_plan_functions_bitexact(seed):
    """After a random solve, the functions of the plan — Eq. 15 (sro_barycentric), metrics (iii),
    (iv), (vi) (sro_metrics) and (v), (vi) against a random reference plan (sro_lp_metrics) — equal
    the oracle's bit for bit."""
    cfg = _config(seed)
    if cfg["cost"] == "hash":
        cfg["cost"] = "dense64"
    g, o = _make(cfg)
    v, opts, iters = cfg["variant"], cfg["opts"], cfg["iters"]
    for solver, var in ((o, v), (g, GV[v])):
        try:
            solver.solve(var, iters, seed=cfg["seed"], epsilon=1e-12, **opts)
        except (OracleError, sro.SroError):
            pass   # the same capacity failure on both sides (test_random_configuration_bitexact)
    assert np.array_equal(g.plan(), o.plan())
    X, Y = cfg["X"], cfg["Y"]
    assert np.array_equal(g.barycentric(X, Y), o.barycentric(X, Y))
    assert g.metrics() == o.metrics()
    rs = np.random.default_rng(seed)
    m, n = cfg["m"], cfg["n"]
    nnz = int(rs.integers(1, 3 * n + 2))
    flat = np.unique(rs.integers(0, m * n, size=nnz))
    cols, rows = flat // m, flat % m                      # column-major order: sorted by (col, row)
    vals = rs.random(len(flat)) / n
    assert g.lp_metrics(rows, cols, vals) == o.lp_metrics(rows, cols, vals)
