"""Fused colour gap sweeps (k_lmo_sweep<SrcColour<float>>) at configs [2] and [4]: device time per
sweep from the library's CUDA-event accounting, entries/s (probe; SRO_LIB selects a build)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

for cfg in (2, 4):
    d = instance(cfg, seed=0)
    s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
    s.solve(sro.SRO_BATCHED, 2 * (d["n"] // 256), seed=1, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=256,
            epsilon=-1.0)
    g0 = s.gap()[0]
    s.set_timing(True)
    s.stats(reset=True)
    for _ in range(10):
        assert s.gap()[0] == g0
    st = s.stats(reset=True)
    ms = st["sweep_ms"] / st["sweep_launches"]
    print(json.dumps(dict(lib=os.path.basename(os.environ.get("SRO_LIB", "libsro.so")), cfg=cfg, sweep_ms=round(ms, 4),
                          entries_per_s=d["m"] * d["n"] / (ms * 1e-3), gap=g0)), flush=True)
    s.close()
