"""Does a concurrent FW / batched solve slow the latency-bound GA solve (L2 / HBM contention)?
GA alone, then GA with FW-ELS and batched-B256 running concurrently on other streams, with the
latter two at several SM budgets (sro_params.max_sms). Device ms of each solve to g <= 1e-6."""
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_05857_b200 as sro  # noqa: E402

dev = torch.device("cuda", 0)
d = bench.make_instance(0)
Cd = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).to(dev)
plan = {name: (variant, opts, cap) for name, variant, opts, cap in bench.PLAN}
names = ["bcfw-GA-GAD-M1-ELS", "fw-ELS", "batched-B256-P-ELS"]
for budget in [None, 0, 74, 37, 16]:
    streams = {nm: torch.cuda.Stream(dev, priority=-1 if nm.startswith("bcfw") else 0) for nm in names}
    run = names[:1] if budget is None else names
    solvers = {nm: sro.Solver(d["a"], d["b"], 1.0, C=Cd, prec="f32", ld=bench.M, stream=streams[nm].cuda_stream,
                              max_sms=0 if nm.startswith("bcfw") else (budget or 0)) for nm in run}
    res = {nm: [] for nm in run}
    for rep in range(3):
        out = {}

        def work(nm):
            variant, opts, cap = plan[nm]
            s = solvers[nm]
            s.reset()
            out[nm] = s.solve(variant, cap, seed=11, epsilon=bench.EPS, **opts)

        torch.cuda.synchronize()
        th = [threading.Thread(target=work, args=(nm,)) for nm in run]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        if rep:
            for nm in run:
                res[nm].append(round(out[nm]["device_ms"], 2))
    print(json.dumps(dict(budget=budget, **res)), flush=True)
    for s in solvers.values():
        s.close()
