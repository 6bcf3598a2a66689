"""Config [3] gap sweep (17.18 GB, k_lmo_sweep_bulk + merge) device time per sweep, library CUDA
events, 5 sweeps after a warm-up (probe; SRO_LIB selects a build, SRO_SLAB the row slab)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402

d = instance(3, seed=0)
s = sro.Solver(d["a"], d["b"], 1.0, cost="hash", hash_seed=d["hash_seed"])
g0 = s.gap()[0]
s.set_timing(True)
s.stats(reset=True)
for _ in range(5):
    assert s.gap()[0] == g0
st = s.stats(reset=True)
ms = st["sweep_ms"] / st["sweep_launches"]
print(json.dumps(dict(lib=os.path.basename(os.environ.get("SRO_LIB", "libsro.so")), slab=os.environ.get("SRO_SLAB"),
                      sweep_ms=round(ms, 4), tbps=round(65536.0 * 65536 * 4 / (ms * 1e-3) / 1e12, 3))), flush=True)
