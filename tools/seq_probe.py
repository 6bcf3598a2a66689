"""Time-to-gap of the sequential BCFW family on config [1] (device ms; A/B with env flags)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

d = instance(1, seed=0)
s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
plan = [("bcfw-P-ELS", 1, dict(step=1, sampling=1)), ("bcfw-U-ELS", 1, dict(step=1, sampling=0)),
        ("bcafw-U-ELS", 2, dict(step=1, sampling=0)), ("bcpfw-U-ELS", 3, dict(step=1, sampling=0)),
        ("bcfw-GA", 1, dict(step=1, sampling=2, ga_M=1, ga_inner=1, ga_post_update=1))]
for rep in range(2):
    for name, v, kw in plan:
        s.reset()
        s.set_timing(True)
        s.stats(reset=True)
        r = s.solve(v, 400 * 4096, seed=11, epsilon=1e-6, **kw)
        st = s.stats(reset=True)
        if rep:
            print(json.dumps(dict(name=name, ms=round(r["device_ms"], 3), iters=r["iters_done"], gap=r["gap"],
                                  us_per_step=round(st["bcfw_ms"] * 1e3 / max(1, st["bcfw_steps"]), 4),
                                  flags=[k for k in ("SRO_NO_PIPE", "SRO_NO_RF") if os.environ.get(k)])), flush=True)
