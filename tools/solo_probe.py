"""Each solve of bench.PLAN alone (one handle, one stream) from T^(0) to g <= 1e-6 on config [1]:
device time (library events), host wall time, iterations; 3 repetitions after one warm-up."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_05857_b200 as sro  # noqa: E402

d = bench.make_instance(0)
dev = torch.device("cuda", 0)
Cd = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).to(dev)
for name, variant, opts, cap in bench.PLAN:
    s = sro.Solver(d["a"], d["b"], 1.0, C=Cd, prec="f32", ld=bench.M)
    out = []
    for rep in range(4):
        s.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = s.solve(variant, cap, seed=11, epsilon=bench.EPS, **opts)
        wall = (time.perf_counter() - t0) * 1e3
        if rep:
            out.append((round(r["device_ms"], 2), round(wall, 2)))
    print(json.dumps(dict(name=name, iters=r["iters_done"], converged=r["converged"], device_ms=[o[0] for o in out],
                          wall_ms=[o[1] for o in out], us_per_iter=round(min(o[0] for o in out) * 1e3 / r["iters_done"], 3))),
          flush=True)
    s.close()
