"""Per-phase clock64 breakdown of the persistent BCFW kernel (debug build)."""
import ctypes as ct
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SRO_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "paper_2103_05857_b200", "libsro_phase.so"))
import numpy as np  # noqa: E402

import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

L = sro.load_library()
L.sro_debug_phase.argtypes = [ct.c_void_p, ct.c_void_p]
d = instance(1, seed=0)
names = ["top", "lmo_local", "warp_argmin", "barrierB", "final_argmin", "serial_tail", "prefetch",
         "barrierC", "sp:gk+dot", "sp:merge", "sp:den", "sp:gamma+tnew", "sp:keep", "sp:apply", "x14", "x15"]
for name, var, kw in [("bcfw-P-ELS", 1, dict(step=1, sampling=1)), ("bcpfw-U", 3, dict(step=1, sampling=0)),
                      ("bcafw-U", 2, dict(step=1, sampling=0)), ("ga", 1, dict(step=1, sampling=2))]:
    s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
    s.solve(var, 4096 * 4, seed=1, epsilon=-1.0, **kw)
    ph = np.zeros(32, dtype=np.int64)
    L.sro_debug_phase(s.h, ph.ctypes.data_as(ct.c_void_p))
    steps = 4096 * 4
    tot = ph.sum()
    print(name, "cycles/step", round(tot / steps, 1), {n: round(float(v) / steps, 1) for n, v in zip(names, ph) if v})
