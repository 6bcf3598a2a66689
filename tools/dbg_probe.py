"""Timing experiment: us/step of the pipelined BCFW kernel with parts switched off (SRO_DBG)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402
d = instance(1, seed=0)
s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
for rep in range(2):
    s.reset(); s.set_timing(True); s.stats(reset=True)
    r = s.solve(1, 8 * 4096, seed=11, epsilon=-1.0, step=1, sampling=1)
    st = s.stats(reset=True)
    if rep:
        print(json.dumps(dict(dbg=os.environ.get("SRO_DBG", "0"), no_pipe=bool(os.environ.get("SRO_NO_PIPE")),
                              us_per_step=round(st["bcfw_ms"] * 1e3 / st["bcfw_steps"], 4))), flush=True)
