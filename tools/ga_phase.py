"""clock64 breakdown of warp 0 in k_bcfw_ga_pipe (debug build libsro_phase.so)."""
import ctypes as ct
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SRO_LIB", os.path.join(ROOT, "paper_2103_05857_b200", "libsro_phase.so"))
import numpy as np  # noqa: E402

import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

L = sro.load_library()
L.sro_debug_phase.argtypes = [ct.c_void_p, ct.c_void_p]
d = instance(1, seed=0)
names = ["top(u53)", "slab+mask", "cw+gk+supp", "BAR_PART", "merge", "serial", "refresh+fenwick", "draw"]
s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
s.solve(1, 4096 * 4, seed=1, epsilon=-1.0, step=1, sampling=2, ga_M=1, ga_inner=1, ga_post_update=1)
ph = np.zeros(32, dtype=np.int64)
L.sro_debug_phase(s.h, ph.ctypes.data_as(ct.c_void_p))
steps = 4096 * 4
print("ga warp0 cycles/step", round(ph[:8].sum() / steps, 1), {n: round(float(v) / steps, 1) for n, v in zip(names, ph[:8])})
print("LMO warp 1: scan", round(ph[16] / steps, 1), "reduce+arrive", round(ph[17] / steps, 1),
      "| last LMO warp: scan", round(ph[18] / steps, 1), "reduce+arrive", round(ph[19] / steps, 1))
print("LMO warp 1 speculation: draw + fetch + pre-scan", round(ph[20] / steps, 1), "then waiting for the next column",
      round(ph[21] / steps, 1), "| pre-scanned", round(ph[23] / steps, 3), "hits", round(ph[22] / steps, 3),
      "| SRO_NO_SPEC" if os.environ.get("SRO_NO_SPEC") else "")
