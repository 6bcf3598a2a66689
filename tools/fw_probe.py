"""Run FW-ELS and batched-B256 on config [1] once (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

d = instance(1, seed=0)
s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
which = sys.argv[1] if len(sys.argv) > 1 else "fw"
if which == "fw":
    r = s.solve(sro.SRO_FW, 20000, epsilon=1e-6, step=sro.STEP_ELS)
else:
    r = s.solve(sro.SRO_BATCHED, 6400, epsilon=1e-6, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=256)
print(which, r["iters_done"], r["gap"], r["device_ms"])
