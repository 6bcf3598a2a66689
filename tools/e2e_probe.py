"""Breakdown of the bench's end-to-end step (fresh handles, H2D inside the timed region)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402

d = bench.make_instance(0)
dev = torch.device("cuda", 0)
C32 = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).pin_memory()
for rep in range(int(os.environ.get("REPS", "6"))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    Cd = C32.to(dev, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = bench.StepRunner(d, dev, Cd)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    ttg = {}
    ms = r.run([], ttg)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    fs = r.objective()
    t4 = time.perf_counter()
    r.close()
    torch.cuda.synchronize(); t5 = time.perf_counter()
    print(json.dumps(dict(rep=rep, h2d=round((t1 - t0) * 1e3, 1), create=round((t2 - t1) * 1e3, 1),
                          run_wall=round((t3 - t2) * 1e3, 1), run_dev=round(ms, 1), objective=round((t4 - t3) * 1e3, 1),
                          close=round((t5 - t4) * 1e3, 1), ttg={k: round(v[0], 1) for k, v in ttg.items()})), flush=True)
