import sys; sys.path.insert(0, '/root/repo')
import paper_2103_05857_b200 as sro
from sro_inputs import instance
d = instance(1, seed=0)
g = sro.Solver(d["a"], d["b"], 1.0, C=d["C32"], prec="f32")
r = g.solve(sro.SRO_BATCHED, 300, seed=1, step=sro.STEP_ELS, sampling=sro.SAMPLE_GA, ga_M=1, ga_inner=1, ga_post_update=0, block_size=256, epsilon=-1.0)
print(r["iters_done"], r["device_ms"])
