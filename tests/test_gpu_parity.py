"""GPU parity: the CUDA path (through the C-ABI, include/sro.h) against the
fp64 oracle, element by element on the same seeded inputs.

The arithmetic of both sides is fixed operation by operation,
so the bar here is BIT-EXACT for argmin rows, step sizes, plan entries, row
sums and the duality gap — stronger than BASELINE's "indices bit-exact,
values within 1e-9 relative", which is asserted as well where it applies.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import BATCHED, BCAFW, BCFW, BCPFW, DEC, ELS, FW, GA, P, U, Oracle
from sro_inputs import instance, uniform_colours

pytestmark = pytest.mark.gpu

sro = pytest.importorskip("paper_2103_05857_b200")


def pair(d, prec="f64", cost=None, cap=31, lam=None):
    """(gpu, oracle) for one instance dict from sro_inputs.instance."""
    lam = d["lam"] if lam is None else lam
    cost = cost or d["cost"]
    if cost == "dense":
        C = d["C32"] if (prec == "f32" and d["C32"] is not None) else d["C64"]
        g = sro.Solver(d["a"], d["b"], lam, C=C, prec=prec, slab_cap=cap)
        o = Oracle(d["a"], d["b"], lam, C=np.asarray(C, dtype=np.float32 if prec == "f32" else np.float64), prec=prec,
                   cap=cap)
    elif cost == "hash":
        g = sro.Solver(d["a"], d["b"], lam, cost="hash", hash_seed=d["hash_seed"], slab_cap=cap)
        o = Oracle(d["a"], d["b"], lam, cost="hash", hash_seed=d["hash_seed"], cap=cap)
    else:
        g = sro.Solver(d["a"], d["b"], lam, X=d["X"], Y=d["Y"], cost=cost, prec=prec, slab_cap=cap)
        o = Oracle(d["a"], d["b"], lam, X=d["X"], Y=d["Y"], cost=cost, prec=prec, cap=cap)
    return g, o


def assert_same_state(g, o, exact=True):
    Tg, To = g.plan(), o.plan()
    rg, ro = g.rowsums(), o.r()
    if exact:
        assert np.array_equal(Tg, To), np.abs(Tg - To).max()
        assert np.array_equal(rg, ro), np.abs(rg - ro).max()
    else:
        assert np.abs(Tg - To).max() <= 1e-9 * max(1e-300, np.abs(To).max())
    fg, fo = g.objective(), o.objective()
    assert abs(fg - fo) <= 1e-9 * abs(fo)
    if exact:
        assert fg == fo


def assert_same_trace(tg, to):
    assert len(tg) == len(to)
    for f in ("k", "i", "j", "v", "dir"):
        bad = np.nonzero(tg[f] != to[f])[0]
        assert len(bad) == 0, f"{f} differs first at step {bad[0]}: gpu {tg[bad[0]]} oracle {to[bad[0]]}"
    for f in ("gamma", "num", "den", "minval"):
        bad = np.nonzero(tg[f] != to[f])[0]
        assert len(bad) == 0, f"{f} differs first at step {bad[0]}: gpu {tg[bad[0]]} oracle {to[bad[0]]}"


# --------------------------------------------------------------------------- LMO sweep + gap
@pytest.mark.parametrize("cfg,m,n,prec,cost", [
    (0, 256, 256, "f64", "dense"), (1, 512, 300, "f32", "dense"), (1, 1023, 77, "f64", "dense"),
    (1, 9001, 40, "f32", "dense"), (1, 16390, 33, "f64", "dense"), (2, 700, 129, "f32", "sqeuclid"),
    (2, 700, 129, "f64", "sqeuclid"), (1, 257, 31, "f64", "euclid"), (1, 8300, 17, "f32", "sqeuclid"),
    (3, 1000, 64, "f32", "hash"), (1, 1, 5, "f64", "dense"), (1, 3, 1, "f32", "dense")])
def test_gap_sweep_bitexact(cfg, m, n, prec, cost):
    """Eq. 9 LMO over every column + Eq. 11 column gaps + psum256 total: argmin rows,
    per-column gaps and the total identical to the oracle (several tiles, ragged tails,
    multi-slab m > 8192, every cost kind and precision)."""
    d = instance(cfg, m=m, n=n, seed=3)
    if cost == "dense" and d["C64"] is None:
        d["C64"] = ((d["X"][:, None, :] - d["Y"][None, :, :]) ** 2).sum(-1)
        d["C32"] = d["C64"].astype(np.float32)
    g, o = pair(d, prec=prec, cost=cost)
    # move the plan away from T0 so h and the supports are non-trivial
    o.solve(BCFW, 3 * n, seed=1, step=ELS, sampling=U, epsilon=-1.0)
    g.solve(sro.SRO_BCFW, 3 * n, seed=1, step=sro.STEP_ELS, sampling=sro.SAMPLE_U, epsilon=-1.0)
    tg, gg, jg = g.gap()
    to, go, jo, _ = o.gap()
    assert np.array_equal(jg, jo)
    assert np.array_equal(gg, go)
    assert tg == to


# --------------------------------------------------------------------------- trajectories, config [0]
VARIANTS = [
    ("bcfw-U-ELS", BCFW, sro.SRO_BCFW, dict(step=ELS, sampling=U)),
    ("bcfw-U-DEC", BCFW, sro.SRO_BCFW, dict(step=DEC, sampling=U)),
    ("bcfw-P-ELS", BCFW, sro.SRO_BCFW, dict(step=ELS, sampling=P)),
    ("bcafw-U", BCAFW, sro.SRO_BCAFW, dict(step=ELS, sampling=U)),
    ("bcpfw-P", BCPFW, sro.SRO_BCPFW, dict(step=ELS, sampling=P)),
    ("ga-gad-m1", BCFW, sro.SRO_BCFW, dict(step=ELS, sampling=GA, ga_M=1, ga_inner=1, ga_post_update=1)),
    ("ga-gad-m5-pre", BCFW, sro.SRO_BCFW, dict(step=ELS, sampling=GA, ga_M=5, ga_inner=1, ga_post_update=0)),
    ("ga-gas", BCFW, sro.SRO_BCFW, dict(step=ELS, sampling=GA, ga_M=1, ga_inner=0, ga_post_update=0)),
    ("ga-pairwise", BCPFW, sro.SRO_BCPFW, dict(step=ELS, sampling=GA, ga_M=1, ga_inner=1, ga_post_update=1)),
    ("ga-away-dec", BCAFW, sro.SRO_BCAFW, dict(step=ELS, sampling=GA, ga_M=2, ga_inner=1, ga_post_update=1)),
]


def _gpu_opts(kw):
    m = {"step": "step", "sampling": "sampling", "ga_M": "ga_M", "ga_inner": "ga_inner",
         "ga_post_update": "ga_post_update", "block_size": "block_size"}
    return {m[k]: v for k, v in kw.items()}


@pytest.mark.parametrize("name,ov,gv,kw", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_config0_trajectory_bitexact(name, ov, gv, kw):
    """BASELINE config [0]: m = n = 256 fp64, 20 n seeded visits, every BCFW-family
    variant: per-step (i, j, v, direction, gamma, num, den, minval) bit-exact, then
    plan, row sums, objective and the gap-check sequence identical."""
    d = instance(0, seed=0)
    g, o = pair(d)
    iters = 20 * 256
    ro = o.solve(ov, iters, seed=7, trace=True, epsilon=1e-12, **kw)
    rg = g.solve(gv, iters, seed=7, trace=True, epsilon=1e-12, **_gpu_opts(kw))
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)
    assert rg["gap"] == ro["gap"] and rg["gap_checks"] == ro["gap_checks"]
    assert rg["entries_scanned"] == ro["entries_scanned"]


@pytest.mark.parametrize("step", [ELS, DEC])
def test_fw_trajectory_bitexact(step):
    """Full FW (Alg. A.1, Eq. A.1): per-iteration gap G_[n] and gamma bit-exact."""
    d = instance(1, m=300, n=260, seed=2)
    g, o = pair(d, prec="f32")
    ro = o.solve(FW, 40, trace=True, step=step, epsilon=1e-9)
    rg = g.solve(sro.SRO_FW, 40, trace=True, step=step, epsilon=1e-9)
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)
    assert rg["gap"] == ro["gap"]


@pytest.mark.parametrize("n,B,sampling,step", [(256, 16, P, ELS), (256, 64, U, ELS), (260, 1, P, DEC),
                                                 (260, 260, U, ELS), (260, 13, P, ELS), (256, 16, U, DEC)])
def test_batched_trajectory_bitexact(n, B, sampling, step):
    """Batched BCFW (R18 super-block step, joint line search): bit-exact, incl. B = 1 and B = n."""
    d = instance(1, m=300, n=n, seed=4)
    g, o = pair(d, prec="f32")
    iters = 6 * (n // B)
    ro = o.solve(BATCHED, iters, seed=3, trace=True, step=step, sampling=sampling, block_size=B, epsilon=1e-9)
    rg = g.solve(sro.SRO_BATCHED, iters, seed=3, trace=True, step=step, sampling=sampling, block_size=B,
                 epsilon=1e-9)
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)


@pytest.mark.parametrize("prec,cost", [("f32", "sqeuclid"), ("f64", "sqeuclid"), ("f32", "dense"), ("f64", "euclid")])
def test_colour_paths_bitexact(prec, cost):
    """Fused colour costs (binary32 and binary64 evaluation) and materialised costs:
    BCPFW trajectories identical to the oracle evaluating the same cost definition."""
    d = instance(2, m=640, n=320, seed=5)
    if cost == "dense":
        d["C64"] = ((d["X"][:, None, :] - d["Y"][None, :, :]) ** 2).sum(-1)
        d["C32"] = d["C64"].astype(np.float32)
    g, o = pair(d, prec=prec, cost=cost)
    ro = o.solve(BCPFW, 5 * 320, seed=9, trace=True, step=ELS, sampling=U, epsilon=1e-9)
    rg = g.solve(sro.SRO_BCPFW, 5 * 320, seed=9, trace=True, step=sro.STEP_ELS, sampling=sro.SAMPLE_U,
                 epsilon=1e-9)
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)


def test_three_colour_worked_example_on_gpu():
    """Fig. 5(b): the printed T^(1) of BCFW-P-DEC on m = n = 3, reproduced by
    the CUDA path with the explicit visit order (3,1,2)."""
    printed = np.loadtxt(__file__.replace("test_gpu_parity.py", "golden/three_colour_T1.txt"))
    X, Y = uniform_colours(3, 100), uniform_colours(3, 200)
    g = sro.Solver([0.1, 0.3, 0.6], [0.6, 0.3, 0.1], 1e-6, X=X, Y=Y, cost="sqeuclid")
    r = g.solve(sro.SRO_BCFW, 3, visit=[2, 0, 1], trace=True, step=sro.STEP_DEC, sampling=sro.SAMPLE_P,
                epsilon=-1.0)
    assert np.abs(g.plan() - printed).max() <= 5e-3 + 1e-12
    assert list(r["trace"]["gamma"]) == [1.0, 6 / 7, 0.75]


def test_resumable_and_reset():
    """Two solve calls equal one call of the summed length; reset returns to T^(0)."""
    d = instance(1, m=200, n=150, seed=6)
    g, _ = pair(d, prec="f32")
    g.solve(sro.SRO_BCAFW, 170, seed=4, step=sro.STEP_ELS, epsilon=-1.0)
    g.solve(sro.SRO_BCAFW, 230, seed=4, step=sro.STEP_ELS, epsilon=-1.0)
    T1 = g.plan()
    g.reset()
    assert np.array_equal(g.plan()[0], d["b"])
    g.solve(sro.SRO_BCAFW, 400, seed=4, step=sro.STEP_ELS, epsilon=-1.0)
    assert np.array_equal(g.plan(), T1)


def test_errors_fail_loudly():
    """Capacity overflow, option lock and invalid options raise (no silent fallback);
    state is left at the last completed step."""
    d = instance(0, m=64, n=64, seed=1)
    g, o = pair(d, cap=2)
    with pytest.raises(sro.SroError) as e:
        g.solve(sro.SRO_BCFW, 64 * 30, seed=1, step=sro.STEP_DEC, epsilon=-1.0)
    assert e.value.status == 6
    g2, _ = pair(d)
    g2.solve(sro.SRO_BCFW, 10, seed=1, epsilon=-1.0)
    with pytest.raises(sro.SroError) as e:
        g2.solve(sro.SRO_BCFW, 10, seed=2, epsilon=-1.0)
    assert e.value.status == 10
    with pytest.raises(sro.SroError):
        g2.solve(sro.SRO_BCAFW, 10, seed=1, step=sro.STEP_DEC, epsilon=-1.0)
    with pytest.raises(sro.SroError):
        sro.Solver(d["a"], d["b"] * 2, 1.0, C=d["C64"])
    with pytest.raises(sro.SroError):
        sro.Solver(d["a"], d["b"], -1.0, C=d["C64"])


def test_capacity_error_matches_oracle_step():
    """The CUDA path stops at the same step as the oracle on capacity overflow, with the
    same state (the failing step is not applied)."""
    d = instance(0, m=64, n=64, seed=1)
    g, o = pair(d, cap=3)
    vis = np.random.default_rng(0).integers(0, 64, size=4000)
    err_o = err_g = None
    try:
        o.solve(BCFW, 4000, seed=1, visit=vis, step=DEC, sampling=U, epsilon=-1.0)
    except Exception as e:  # noqa: BLE001
        err_o = e
    try:
        g.solve(sro.SRO_BCFW, 4000, seed=1, visit=vis, step=sro.STEP_DEC, epsilon=-1.0)
    except sro.SroError as e:
        err_g = e
    assert err_o is not None and err_g is not None
    assert np.array_equal(g.plan(), o.plan())


# --------------------------------------------------------------------------- full-size configs
def test_config1_full_size_two_epochs_bitexact():
    """BASELINE config [1] at full size (m = n = 4096, fp32 costs, lambda = 1), the
    launch configuration bench.py times: two epochs of BCFW-P-ELS with gap checks,
    every step bit-exact against the oracle."""
    d = instance(1, seed=0)
    g, o = pair(d, prec="f32")
    ro = o.solve(BCFW, 2 * 4096, seed=1, trace=True, step=ELS, sampling=P, epsilon=1e-6)
    rg = g.solve(sro.SRO_BCFW, 2 * 4096, seed=1, trace=True, step=sro.STEP_ELS, sampling=sro.SAMPLE_P,
                 epsilon=1e-6)
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)
    assert rg["gap"] == ro["gap"]


def test_config1_full_size_converges_certified():
    """Config [1] to g <= 1e-6 on the GPU; the oracle re-evaluates the GPU's final plan
    (its own r = T 1 and gap, Thm 2): feasible, gap certified <= 1e-6 (+1e-12 for the
    row-sum summation order), objective within 1e-9."""
    d = instance(1, seed=0)
    g = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
    r = g.solve(sro.SRO_BCFW, 200 * 4096, seed=1, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, epsilon=1e-6)
    assert r["converged"] == 1 and r["gap"] <= 1e-6
    T = g.plan()
    assert np.abs(T.sum(0) - d["b"]).max() <= 1e-10 and T.min() >= 0
    assert np.abs(g.rowsums() - T.sum(1)).max() <= 1e-10
    o = Oracle(d["a"], d["b"], 1.0, C=d["C32"].astype(np.float64), cap=64)
    o.set_plan(T)
    assert o.gap()[0] <= 1e-6 + 1e-12
    fo = o.objective()
    assert abs(fo - g.objective()) <= 1e-9 * abs(fo)


@pytest.mark.parametrize("name,ov,gv,kw", [VARIANTS[0], VARIANTS[3], VARIANTS[5]], ids=["bcfw", "bcafw", "ga"])
def test_config0_shared_memory_kernel_bitexact(name, ov, gv, kw, monkeypatch):
    """The shared-memory persistent kernel (used when the register-file kernel does not
    apply) forced on config [0]: same bit-exact trajectory as the oracle."""
    monkeypatch.setenv("SRO_NO_RF", "1")
    d = instance(0, seed=0)
    g, o = pair(d)
    ro = o.solve(ov, 4 * 256, seed=7, trace=True, epsilon=1e-12, **kw)
    rg = g.solve(gv, 4 * 256, seed=7, trace=True, epsilon=1e-12, **_gpu_opts(kw))
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)


@pytest.mark.parametrize("coop,runs", [(True, "sort"), (False, "sort"), (False, "search")],
                         ids=["cooperative", "per-phase", "per-phase-run-search"])
@pytest.mark.parametrize("variant,B", [(BATCHED, 16), (FW, 0)])
def test_block_step_multikernel_path_bitexact(variant, B, coop, runs, monkeypatch):
    """The large-U block step (one cooperative launch, or the per-phase kernels) forced on
    small instances: same bit-exact trajectory as the single-CTA tail path and the oracle. The
    per-phase k_runs forms the (row, chunk) runs by a per-chunk key sort, or (SRO_RUNS_KMAX=0, its
    fallback for chunks of more than 4096 pairs) by searching the earlier columns' supports."""
    monkeypatch.setenv("SRO_NO_TAIL", "1")
    if coop:
        monkeypatch.setenv("SRO_COOP", "1")
    if runs == "search":
        monkeypatch.setenv("SRO_RUNS_KMAX", "0")
    d = instance(1, m=300, n=256, seed=8)
    g, o = pair(d, prec="f32")
    kw = dict(block_size=B, sampling=P) if B else {}
    gv = sro.SRO_BATCHED if B else sro.SRO_FW
    ro = o.solve(variant, 40, seed=3, trace=True, step=ELS, epsilon=1e-9, **kw)
    rg = g.solve(gv, 40, seed=3, trace=True, step=sro.STEP_ELS, epsilon=1e-9, **kw)
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)


@pytest.mark.parametrize("name,ov,gv,kw", [VARIANTS[0], VARIANTS[3], VARIANTS[4], VARIANTS[5], VARIANTS[8]],
                         ids=["bcfw", "bcafw", "bcpfw", "ga", "ga-pairwise"])
def test_config0_register_file_kernel_bitexact(name, ov, gv, kw, monkeypatch):
    """The register-file persistent kernel k_bcfw_rf (the pipelined kernels forced off):
    same bit-exact trajectory as the oracle."""
    monkeypatch.setenv("SRO_NO_PIPE", "1")
    d = instance(0, seed=0)
    g, o = pair(d)
    ro = o.solve(ov, 4 * 256, seed=9, trace=True, epsilon=1e-12, **kw)
    rg = g.solve(gv, 4 * 256, seed=9, trace=True, epsilon=1e-12, **_gpu_opts(kw))
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)


@pytest.mark.parametrize("var,kw", [(BCFW, dict(step=ELS, sampling=U)), (BCPFW, dict(step=ELS, sampling=P)),
                                    (BCFW, dict(step=ELS, sampling=GA, ga_M=1, ga_inner=1, ga_post_update=1))],
                         ids=["bcfw-U", "bcpfw-P", "ga"])
def test_config1_shape_pipelined_kernels_bitexact(var, kw):
    """The pipelined kernels at the config-[1] row count (m = 4096, three 128-bit vectors per
    LMO thread, fp32 costs) on fewer columns: every step bit-exact vs the oracle."""
    d = instance(1, m=4096, n=512, seed=4)
    d["C32"] = (((d["X"][:, None, :] - d["Y"][None, :, :]) ** 2).sum(-1)).astype(np.float32)
    g, o = pair(d, prec="f32")
    gv = {BCFW: sro.SRO_BCFW, BCPFW: sro.SRO_BCPFW}[var]
    ro = o.solve(var, 6 * 512, seed=2, trace=True, epsilon=1e-9, **kw)
    rg = g.solve(gv, 6 * 512, seed=2, trace=True, epsilon=1e-9, **_gpu_opts(kw))
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)


@pytest.mark.parametrize("name,ov,gv,kw", [VARIANTS[0], VARIANTS[3], VARIANTS[5]], ids=["bcfw", "bcafw", "ga"])
def test_converges_mid_call_then_continues_like_oracle(name, ov, gv, kw):
    """Epochs are enqueued one ahead of the host's gap check (a speculative epoch after the
    converging one is a no-op): the call stops at the oracle's gap check with the oracle's
    state, and a second call continues exactly as the oracle's second call."""
    d = instance(0, seed=3)
    g, o = pair(d)
    for iters, conv in ((3 * 256 + 100, False), (400 * 256, True), (400 * 256, True)):
        ro = o.solve(ov, iters, seed=5, epsilon=1e-5, **kw)
        rg = g.solve(gv, iters, seed=5, epsilon=1e-5, **_gpu_opts(kw))
        assert bool(rg["converged"]) == bool(ro["converged"]) == conv
        assert rg["iters_done"] == ro["iters_done"] and rg["gap"] == ro["gap"]
        assert rg["gap_checks"] == ro["gap_checks"] and rg["entries_scanned"] == ro["entries_scanned"]
        assert_same_state(g, o)


def test_max_sms_does_not_change_results():
    """sro_params.max_sms only resizes the device-wide kernels' grids: FW, batched and GA
    trajectories are identical with 3 SMs and with all of them."""
    d = instance(1, m=300, n=260, seed=8)
    runs = [(sro.SRO_FW, dict(step=sro.STEP_ELS), 12), (sro.SRO_BATCHED, dict(step=sro.STEP_ELS, block_size=13), 60),
            (sro.SRO_BCFW, dict(step=sro.STEP_ELS, sampling=sro.SAMPLE_GA, ga_M=1, ga_inner=1, ga_post_update=1), 1300)]
    for v, kw, iters in runs:
        out = []
        for ms in (0, 3):
            g = sro.Solver(d["a"], d["b"], d["lam"], C=d["C32"], prec="f32", max_sms=ms)
            r = g.solve(v, iters, seed=2, trace=True, epsilon=1e-12, **kw)
            out.append((r["trace"], g.plan(), r["gap"]))
            g.close()
        assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1]) and out[0][2] == out[1][2]


def test_ga_pipelined_kernel_global_gaps_bitexact():
    """m = 4096, n = 8192: a and the stored gaps no longer fit in shared memory next to the
    GA tree, so the pipelined GA kernel keeps them in global memory (GaPipeLayout, GSM =
    false): every step still bit-exact against the oracle."""
    d = instance(1, m=4096, n=8192, seed=12)
    d["C32"] = (((d["X"][:, None, :] - d["Y"][None, :, :]) ** 2).sum(-1)).astype(np.float32)
    g, o = pair(d, prec="f32")
    kw = dict(step=ELS, sampling=GA, ga_M=1, ga_inner=1, ga_post_update=1)
    ro = o.solve(BCFW, 12288, seed=3, trace=True, epsilon=1e-9, **kw)
    rg = g.solve(sro.SRO_BCFW, 12288, seed=3, trace=True, epsilon=1e-9, **_gpu_opts(kw))
    assert_same_trace(rg["trace"], ro["trace"])
    assert_same_state(g, o)
