"""Batched BCFW (P sampling, ELS) to gap 1e-6 on configs [1] (B=256), [2] (B=256), [4] (B=1024):
device time of the whole solve (timing off), host wall time, repeated (probe, not the bench)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

reps = int(os.environ.get("REPS", "3"))
for cfg, B in [(int(c.split(":")[0]), int(c.split(":")[1])) for c in (sys.argv[1:] or ["1:256", "2:256", "4:1024"])]:
    d = instance(cfg, seed=0)
    if cfg == 1:
        s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
    else:
        s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
    n = len(d["b"])
    out = []
    for r in range(reps + 1):
        s.reset()
        t0 = time.perf_counter()
        res = s.solve(sro.SRO_BATCHED, 400 * (n // B), seed=1, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=B,
                      epsilon=1e-6)
        wall = (time.perf_counter() - t0) * 1e3
        if r:
            out.append((res["device_ms"], wall, res["iters_done"]))
    print(json.dumps(dict(cfg=cfg, B=B, iters=out[0][2], device_ms=[round(o[0], 2) for o in out],
                          wall_ms=[round(o[1], 2) for o in out],
                          us_per_step=round(min(o[0] for o in out) * 1e3 / out[0][2], 2))), flush=True)
    s.close()
