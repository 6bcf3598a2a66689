"""Per block step: the LMO sweep's and the whole step's device time (library CUDA events, graph
replay off while timing) at configs [1], [2], [4] (probe)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

for cfg, B in ((1, 256), (2, 256), (4, 1024)):
    d = instance(cfg, seed=0)
    if cfg == 1:
        s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
    else:
        s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
    kw = dict(step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=B, epsilon=-1.0)
    s.solve(sro.SRO_BATCHED, 2 * (d["n"] // B), seed=1, **kw)
    s.set_timing(True)
    s.stats(reset=True)
    steps = d["n"] // B - 1
    r = s.solve(sro.SRO_BATCHED, steps, seed=1, **kw)
    st = s.stats(reset=True)
    print(json.dumps(dict(cfg=cfg, B=B, steps=st["block_steps"], us_step_total=round(1e3 * st["block_ms"] / st["block_steps"], 2),
                          us_sweep=round(1e3 * st["sweep_ms"] / st["sweep_launches"], 2),
                          us_device_per_step_call=round(1e3 * r["device_ms"] / steps, 2))), flush=True)
    s.close()
