"""Kernel list of batched block steps (for ncu --metrics gpu__time_duration.sum): configs [2]
(B=256) and [4] (B=1024), fused colour costs, a warm-up solve then STEPS block steps (probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

steps = int(os.environ.get("STEPS", "12"))
for cfg, B in [(int(c.split(":")[0]), int(c.split(":")[1])) for c in (sys.argv[1:] or ["2:256", "4:1024"])]:
    d = instance(cfg, seed=0)
    s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
    s.solve(sro.SRO_BATCHED, 3 * (d["n"] // B), seed=1, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=B,
            epsilon=-1.0)
    r = s.solve(sro.SRO_BATCHED, steps, seed=1, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=B, epsilon=-1.0)
    print(cfg, B, "device_ms", r["device_ms"], "us/step", 1e3 * r["device_ms"] / steps, flush=True)
    s.close()
