"""Sequential step latency against the problem shape: BCFW-P-ELS and BCFW-GA (GAD-M1) on
dense fp32 mixture-colour costs, 4 epochs from T^(0) (no convergence stop), device time per
step. Shows which kernel serves each shape (pipelined / GA-pipelined kernels while h, r, a and
the GA state fit in shared memory, the register-file / generic kernels beyond)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

for m, n in ((1024, 1024), (2048, 2048), (4096, 4096), (8192, 2048), (4096, 8192), (16384, 1024), (512, 16384)):
    d = instance(1, m=m, n=n, seed=0)
    out = {}
    for name, samp in (("P", sro.SAMPLE_P), ("GA", sro.SAMPLE_GA)):
        s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
        s.solve(sro.SRO_BCFW, n, seed=1, step=sro.STEP_ELS, sampling=samp, epsilon=-1.0)   # warm
        s.reset()
        r = s.solve(sro.SRO_BCFW, 4 * n, seed=1, step=sro.STEP_ELS, sampling=samp, epsilon=-1.0)
        out[name] = round(r["device_ms"] * 1e3 / r["iters_done"], 3)
        s.close()
    print(json.dumps(dict(m=m, n=n, us_per_step_P=out["P"], us_per_step_GA=out["GA"])), flush=True)
