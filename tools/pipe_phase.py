"""Per-phase clock64 breakdown of k_bcfw_pipe (debug build libsro_phase.so): warp 0 (serial) and warp 1 (LMO)."""
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
w0 = ["prefetch+gk", "serial_step", "publish", "B1", "merge", "slab+mask", "B2"]
w1 = ["refresh", "lmo", "redux", "B1", "-", "-", "B2"]
for name, var, kw in [("bcfw-P-ELS", 1, dict(step=1, sampling=1)), ("bcpfw-U", 3, dict(step=1, sampling=0)),
                      ("bcafw-U", 2, dict(step=1, sampling=0))]:
    s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
    s.solve(var, 4096 * 4, seed=1, epsilon=-1.0, **kw)
    ph = np.zeros(16, dtype=np.int64)
    L.sro_debug_phase(s.h, ph.ctypes.data_as(ct.c_void_p))
    steps = 4096 * 4
    print(name, "warp0", round(ph[:7].sum() / steps, 1), {n: round(float(v) / steps, 1) for n, v in zip(w0, ph[:7])})
    print(name, "warp1", round(ph[8:15].sum() / steps, 1), {n: round(float(v) / steps, 1) for n, v in zip(w1, ph[8:15]) if n != "-"})
