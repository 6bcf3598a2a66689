"""BCFW-GA-GAD-M1-ELS alone on config [1] to g <= 1e-6 with the speculative next
draw on and off (SRO_NO_SPEC): device time, steps, and the trajectory's final
objective / gap (identical by construction)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_05857_b200 as sro  # noqa: E402

d = bench.make_instance(0)
dev = torch.device("cuda", 0)
Cd = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).to(dev)
name, variant, opts, cap = [p for p in bench.PLAN if "GA" in p[0]][0]
for mode in sys.argv[1:] or ("spec", "nospec", "spec"):
    if mode == "nospec":
        os.environ["SRO_NO_SPEC"] = "1"
    else:
        os.environ.pop("SRO_NO_SPEC", None)
    s = sro.Solver(d["a"], d["b"], 1.0, C=Cd, prec="f32", ld=bench.M)
    out = []
    for rep in range(4):
        s.reset()
        torch.cuda.synchronize()
        r = s.solve(variant, cap, seed=11, epsilon=bench.EPS, **opts)
        if rep:
            out.append(round(r["device_ms"], 2))
    print(json.dumps(dict(mode=mode, iters=r["iters_done"], converged=r["converged"], gap=r["gap"],
                          device_ms=out, us_per_iter=round(min(out) * 1e3 / r["iters_done"], 3))), flush=True)
