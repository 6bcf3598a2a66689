import sys, os, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2103_05857_b200 as sro
from sro_inputs import instance
for cfg, B in ((1, 256), (2, 256), (4, 1024)):
    d = instance(cfg, seed=0)
    if cfg == 1:
        s = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
    else:
        s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
    n = len(d["b"])
    for ep in range(6):
        r = s.solve(sro.SRO_BATCHED, n // B, epsilon=-1.0, step=sro.STEP_ELS, sampling=sro.SAMPLE_P, block_size=B, seed=1)
        rows, cols, vals = s.plan_coo()
        cnt = np.bincount(cols, minlength=n)
        blk = cnt.reshape(-1, B).sum(1) + B
        print(cfg, ep, "nnz/col mean %.2f max %d; block P (<= sum+B) mean %.0f max %d" % (cnt.mean(), cnt.max(), blk.mean(), blk.max()), flush=True)
