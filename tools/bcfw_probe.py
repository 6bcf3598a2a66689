"""One BCFW-family solve segment on config [1] (for ncu captures of k_bcfw_rf)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

d = instance(1, seed=0)
s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
samp = {"P": 1, "U": 0, "GA": 2}[sys.argv[1] if len(sys.argv) > 1 else "P"]
var = int(sys.argv[2]) if len(sys.argv) > 2 else 1
r = s.solve(var, 4096 * 3, seed=1, epsilon=-1.0, step=1, sampling=samp)
print(r["iters_done"], r["device_ms"])
