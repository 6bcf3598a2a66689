"""Where does the end-to-end step lose time vs the device-timed one? fresh solver vs reused."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2103_05857_b200 as sro  # noqa: E402

d = bench.make_instance(0)
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
C32 = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).pin_memory()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    Cd = C32.to(dev, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s = sro.Solver(d["a"], d["b"], 1.0, C=Cd, prec="f32", stream=stream.cuda_stream, ld=bench.M)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    per = {}
    for name, variant, opts, cap in bench.PLAN:
        s.reset()
        ta = time.perf_counter()
        r = s.solve(variant, cap, seed=11, epsilon=bench.EPS, **opts)
        per[name] = (round((time.perf_counter() - ta) * 1e3, 2), round(r["device_ms"], 2))
    torch.cuda.synchronize(); t3 = time.perf_counter()
    s.close()
    print(json.dumps(dict(rep=rep, h2d_ms=round((t1 - t0) * 1e3, 2), create_ms=round((t2 - t1) * 1e3, 2),
                          solve_ms=round((t3 - t2) * 1e3, 2), per_variant_wall_vs_device=per)), flush=True)
