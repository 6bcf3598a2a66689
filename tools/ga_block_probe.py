import sys; sys.path.insert(0, '/root/repo')
import paper_2103_05857_b200 as sro
from sro_inputs import instance
d = instance(1, m=512, n=512, seed=6)
for samp in (sro.SAMPLE_P, sro.SAMPLE_GA):
    for B in (64, 16):
        g = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
        r = g.solve(sro.SRO_BATCHED, 400 * (512 // B), seed=1, step=sro.STEP_ELS, sampling=samp, ga_M=1, ga_inner=1,
                    ga_post_update=1, block_size=B, epsilon=1e-6)
        print(samp, B, r["converged"], r["iters_done"], r["gap"])
