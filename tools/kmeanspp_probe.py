"""k-means++ seeding (sro_kmeanspp) wall time on a 1024 x 1024 synthetic image, k = 256 / 4096 (probe)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import kmeanspp_uniforms, synthetic_image  # noqa: E402

img = synthetic_image(1024, 1024, seed=3).reshape(-1, 3)
for k in (256, 4096):
    u = kmeanspp_uniforms(k, 1)
    sro.kmeanspp_init(img, k, u)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        sro.kmeanspp_init(img, k, u)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(json.dumps(dict(npix=len(img), k=k, ms=[round(t, 2) for t in ts], us_per_centre=round(min(ts) * 1e3 / k, 2))),
          flush=True)
