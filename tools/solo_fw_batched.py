"""FW-ELS on config [1] and [3] and batched on [1]/[2]/[4] to g <= 1e-6, alone, warm (probe):
device ms per solve and per iteration (SRO_PDL=1 for the A/B with programmatic dependent launches)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

runs = sys.argv[1:] or ["fw1", "fw3", "b1", "b2", "b4"]
for r in runs:
    cfg = int(r[-1])
    d = instance(cfg, seed=0)
    if cfg == 1:
        s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
    elif cfg == 3:
        s = sro.Solver(d["a"], d["b"], 1.0, cost="hash", hash_seed=d["hash_seed"])
    else:
        s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
    B = 1024 if cfg == 4 else 256
    out = []
    for rep in range(3):
        s.reset()
        if r.startswith("fw"):
            res = s.solve(sro.SRO_FW, 20000, epsilon=1e-6, step=sro.STEP_ELS)
        else:
            res = s.solve(sro.SRO_BATCHED, 400 * (d["n"] // B), epsilon=1e-6, step=sro.STEP_ELS,
                          sampling=sro.SAMPLE_P, block_size=B, seed=1)
        out.append(res["device_ms"])
    print(json.dumps(dict(run=r, pdl=os.environ.get("SRO_PDL") is not None, iters=res["iters_done"],
                          ms=[round(x, 2) for x in out], us_per_iter=round(1e3 * min(out) / res["iters_done"], 2))),
          flush=True)
    s.close()
