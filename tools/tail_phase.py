"""clock64 breakdown of k_block_tail_sm (debug build libsro_phase.so): batched B=256 on config [1]."""
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
names = ["G_U", "count+scan", "pairs", "sort", "sums0", "den+gamma", "cap", "update", "sums1", "structure", "merge:epi", "merge:partials", "entry", "den:chunks", "den:gamma", "sums:runs"]
for cfg, B in ((1, 256), (2, 256), (4, 1024)):
    d = instance(cfg, seed=0)
    if cfg == 1:
        s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
    else:
        s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
    steps = 3 * (len(d["b"]) // B)
    s.solve(sro.SRO_BATCHED, steps, seed=1, epsilon=-1.0, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=B)
    ph = np.zeros(32, dtype=np.int64)
    L.sro_debug_phase(s.h, ph.ctypes.data_as(ct.c_void_p))
    print(cfg, B, "cycles/step", round(ph[:13].sum() / steps), {n: round(float(v) / steps) for n, v in zip(names, ph)})
    print("   per step: touched rows", round(ph[20] / steps, 1), "runs", round(ph[21] / steps, 1), "mid rows",
          round(ph[22] / steps, 1), "hot rows", round(ph[23] / steps, 1), "| sums0 sub-phases (avg cycles per thread):",
          "rows<=2", round(ph[24] / steps), "mid", round(ph[25] / steps), "hot", round(ph[26] / steps))
    s.close()
