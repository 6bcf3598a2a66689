"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py and
tools/configs_probe.py time.

[2] and [4] (fused fp32 colour costs, batched BCFW): two epochs of block steps, every step
(block, argmin of the first column, gamma, numerator, denominator) and the final plan / row
sums bit-exact against the oracle, which is slow but exact at this size.
[3] (65536 x 65536 materialised iid cost, full FW): too large for the oracle to follow (one FW
iteration is 4.3e9 oracle cost evaluations), so the GPU solve to g <= 1e-6 is checked on sampled
outputs the definition gives one by one (Eq. 9 / Eq. 11 on 64 columns against the GPU's own h)
and on properties that hold at any size (feasibility, r = T 1, certified gap).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import BATCHED, ELS, P, Oracle
from sro_inputs import hash_uniform_cost, instance

pytestmark = pytest.mark.gpu

sro = pytest.importorskip("paper_2103_05857_b200")


def _coo_equal(g, o):
    rg, cg, vg = g.plan_coo()
    ro, co, vo = o.plan_coo()
    assert np.array_equal(cg, co) and np.array_equal(rg, ro) and np.array_equal(vg, vo)


@pytest.mark.parametrize("cfg,B", [(2, 256), (4, 1024)], ids=["config2", "config4"])
def test_batched_fullsize_two_epochs_bitexact(cfg, B):
    d = instance(cfg, seed=0)
    n = d["n"]
    g = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
    o = Oracle(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32", cap=31)
    iters = 2 * (n // B)
    ro = o.solve(BATCHED, iters, seed=1, trace=True, step=ELS, sampling=P, block_size=B, epsilon=1e-6)
    rg = g.solve(sro.SRO_BATCHED, iters, seed=1, trace=True, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=B,
                 epsilon=1e-6)
    assert rg["iters_done"] == ro["iters_done"] and rg["gap"] == ro["gap"]
    for f in ("k", "i", "j", "gamma", "num", "den", "minval"):
        assert np.array_equal(rg["trace"][f], ro["trace"][f]), f
    _coo_equal(g, o)
    assert np.array_equal(g.rowsums(), o.r())
    assert g.objective() == o.objective()


def test_config3_fullsize_fw_sampled_and_certified():
    d = instance(3, seed=0)
    m = n = 65536
    g = sro.Solver(d["a"], d["b"], 1.0, cost="hash", hash_seed=d["hash_seed"])
    r = g.solve(sro.SRO_FW, 200, step=sro.STEP_ELS, epsilon=1e-6)
    assert r["converged"] == 1 and r["gap"] <= 1e-6
    total, gcol, jcol = g.gap()
    assert total == r["gap"] or total <= 1e-6
    rows, cols, vals = g.plan_coo()
    # feasibility (Eq. 8) and r = T 1 (the maintained row sums, R6)
    colsum = np.bincount(cols, weights=vals, minlength=n)
    assert np.abs(colsum - d["b"]).max() <= 1e-15
    assert vals.min() > 0.0
    rs = g.rowsums()
    assert np.abs(rs - np.bincount(rows, weights=vals, minlength=m)).max() <= 1e-12
    # Eq. 9 / Eq. 11 on sampled columns against the GPU's own h = (r - a) / lambda
    h = (rs - d["a"]) / 1.0
    order = np.argsort(cols, kind="stable")
    rows, cols, vals = rows[order], cols[order], vals[order]
    starts = np.searchsorted(cols, np.arange(n + 1))
    rng = np.random.default_rng(0)
    for i in rng.choice(n, 64, replace=False):
        c = hash_uniform_cost(d["hash_seed"], m, np.arange(m), np.full(m, i))
        v = c + h
        j = int(np.argmin(v))                       # first minimum = lowest row on ties (R1)
        assert j == jcol[i]
        dot = 0.0
        for q in range(starts[i], starts[i + 1]):    # support rows ascending (R19)
            k = rows[q]
            dot = dot + vals[q] * (c[k] + h[k])
        assert dot - d["b"][i] * v[j] == gcol[i]


def test_bench_step_concurrent_equals_serial():
    """bench.py's launch configuration: the six solves of a step run concurrently on their own
    (priority) streams sharing one device copy of C; every solve's plan, row sums, gap and
    iteration count equal those of the same solves run one after another (each solve is a
    deterministic function of its inputs; the serial path is the one the parity tests pin)."""
    import torch

    import bench
    d = bench.make_instance(0)
    dev = torch.device("cuda", 0)
    Cd = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).to(dev)
    out = {}
    for conc in (True, False):
        r = bench.StepRunner(d, dev, Cd, concurrent=conc)
        ttg = {}
        r.run([], ttg)
        out[conc] = [(s.plan_coo(), s.rowsums(), s.gap()[0]) for s in r.solvers]
        r.close()
    for (pa, ra, ga), (pb, rb, gb) in zip(out[True], out[False]):
        assert all(np.array_equal(x, y) for x, y in zip(pa, pb))
        assert np.array_equal(ra, rb) and ga == gb and ga <= 1e-6
