"""k-means front end at image scale: Lloyd iterations of sro_kmeans on a synthetic 1024 x 1024
image for k = 256 and 4096 (config [1]'s m). Reports time per iteration (wall, the call
synchronises per iteration) and the assignment's (pixel, centroid) pair rate against its ALU
bound: the fp32 prefilter issues 9 FP32-pipe instructions per pair (3 sub, 1 mul, 2 fma, the
candidate compare, the running minimum, its margin) at 128 lanes / clk / SM and 1965 MHz; the
exact binary64 evaluation runs only for candidates."""
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
peak = 148 * 128 * 1.965e9 / 9.0   # pairs / s
for k, iters in ((256, 30), (4096, 8)):
    init = kmeans_init(N, k, 1)
    sro.kmeans_quantize(img, k, init, 2)
    pers = []
    for rep in range(3):
        t0 = time.perf_counter()
        cen, lab, cnt, it, conv = sro.kmeans_quantize(img, k, init, iters)
        pers.append((time.perf_counter() - t0) / it)
    per = min(pers)
    pairs = float(N) * k
    print(json.dumps(dict(npix=N, k=k, iters=it, converged=conv, ms_per_iter=round(per * 1e3, 3),
                          ms_per_iter_reps=[round(x * 1e3, 3) for x in pers],
                          tera_pairs_per_s=round(pairs / per / 1e12, 3), bound_tera_pairs_per_s=round(peak / 1e12, 3),
                          frac=round(pairs / per / peak, 3))), flush=True)
