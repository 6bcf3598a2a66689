"""Is the single-CTA GA kernel slowed by a low-occupancy issue throttle? BCFW-GA alone on config [1]
to g <= 1e-6 (device time), while nothing else runs, and while a keep-alive kernel occupies the
other SMs (one 32-thread CTA per SM, issuing or in __nanosleep) on another stream."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_05857_b200 as sro  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "microbench", "libspin.so"))
dev = torch.device("cuda", 0)
sink = torch.zeros(1, dtype=torch.int32, device=dev)
d = bench.make_instance(0)
Cd = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).to(dev)
plan = {name: (variant, opts, cap) for name, variant, opts, cap in bench.PLAN}
st = torch.cuda.Stream(dev)
side = torch.cuda.Stream(dev)
for name in ["bcfw-GA-GAD-M1-ELS", "bcfw-P-ELS"]:
    variant, opts, cap = plan[name]
    s = sro.Solver(d["a"], d["b"], 1.0, C=Cd, prec="f32", ld=bench.M, stream=st.cuda_stream)
    for mode in ["alone", "spin-issue", "spin-sleep", "alone"]:
        out = []
        for rep in range(3):
            s.reset()
            torch.cuda.synchronize()
            if mode != "alone":
                rc = lib.spin(ctypes.c_int(147), ctypes.c_longlong(int(1.2e9)), ctypes.c_int(0 if mode == "spin-issue" else 1),
                              ctypes.c_void_p(side.cuda_stream), ctypes.c_void_p(sink.data_ptr()))
                assert rc == 0
            r = s.solve(variant, cap, seed=11, epsilon=bench.EPS, **opts)
            torch.cuda.synchronize()
            if rep:
                out.append(r["device_ms"])
        print(json.dumps(dict(name=name, mode=mode, iters=r["iters_done"], device_ms=[round(x, 2) for x in out],
                              us_per_iter=round(min(out) * 1e3 / r["iters_done"], 3))), flush=True)
    s.close()
