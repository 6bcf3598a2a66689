"""k-means front end at image scale: Lloyd iterations of sro_kmeans on a synthetic 1024 x 1024
image for k = 256 and 4096 (config [1]'s m). Reports time per iteration (wall, the call
synchronises per iteration) and the assignment's fp64 rate: 8 fp64 operations (3 sub, 3 mul,
2 add) per (pixel, centroid) pair, against the FP64 add/mul issue rate measured on this GPU
(64 lanes / clk / SM, tools/microbench/f2f.cu) at the max SM clock."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import kmeans_init, synthetic_image  # noqa: E402

img = synthetic_image(1024, 1024, K=12, seed=5)
N = len(img)
peak = 148 * 64 * 1.965e9
for k, iters in ((256, 30), (4096, 8)):
    init = kmeans_init(N, k, 1)
    sro.kmeans_quantize(img, k, init, 2)
    t0 = time.perf_counter()
    cen, lab, cnt, it, conv = sro.kmeans_quantize(img, k, init, iters)
    dt = time.perf_counter() - t0
    per = dt / it
    ops = 8.0 * N * k
    print(json.dumps(dict(npix=N, k=k, iters=it, converged=conv, ms_per_iter=round(per * 1e3, 3),
                          fp64_gops=round(ops / per / 1e9, 1), peak_gops=round(peak / 1e9, 1),
                          frac=round(ops / per / peak, 3))), flush=True)
