"""Gap sweeps at config [2] (fused fp32 colour cost; for an ncu capture of k_lmo_sweep<SrcColour>)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402
d = instance(2, seed=0)
s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
for _ in range(2):
    print(s.gap()[0])
