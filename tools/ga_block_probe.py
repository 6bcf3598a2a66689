"""Batched BCFW with gap-adaptive block sampling (NEXT-4) against permutation sampling, to g <= 1e-6:
block steps, device time, time per step. Config [1] (dense fp32, B = 256) and config [2] (fused
colour costs, B = 256), plus a small instance at B = 16."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

for cfg, B, m in ((1, 256, None), (2, 256, None), (1, 16, 512)):
    d = instance(cfg, m=m, n=m, seed=6 if m else 0)
    n = len(d["b"])
    for samp, name in ((sro.SAMPLE_P, "P"), (sro.SAMPLE_GA, "GA-GAD-M1-post"), (sro.SAMPLE_GA, "GA-GAD-M1-pre")):
        post = 0 if name.endswith("pre") else 1
        for rep in range(2):
            if cfg == 1:
                g = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
            else:
                g = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
            r = g.solve(sro.SRO_BATCHED, 400 * (n // B), seed=1, step=sro.STEP_ELS, sampling=samp, ga_M=1, ga_inner=1,
                        ga_post_update=post, block_size=B, epsilon=1e-6)
            g.close()
        print(json.dumps(dict(cfg=cfg, n=n, B=B, sampling=name, converged=r["converged"], steps=r["iters_done"],
                              gap=r["gap"], device_ms=round(r["device_ms"], 2),
                              us_per_step=round(r["device_ms"] * 1e3 / max(1, r["iters_done"]), 2))), flush=True)
