"""Does the GA solve's column fetch pay for L2 misses? BCFW-GA alone on config [1] (one handle,
one stream) to g <= 1e-6, with and without an L2 access-policy window (persisting) over the
cost matrix on the solver stream. Prints device ms and us per step for both."""
import ctypes
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_05857_b200 as sro  # noqa: E402


def cudart():
    torch.cuda.init()
    for cand in glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                       "libcudart.so*")) + ["libcudart.so.12", "libcudart.so"]:
        try:
            return ctypes.CDLL(cand)
        except OSError:
            pass
    raise RuntimeError("libcudart not found")


class Window(ctypes.Structure):
    _fields_ = [("base_ptr", ctypes.c_void_p), ("num_bytes", ctypes.c_size_t), ("hitRatio", ctypes.c_float),
                ("hitProp", ctypes.c_int), ("missProp", ctypes.c_int)]


class AttrValue(ctypes.Union):
    _fields_ = [("accessPolicyWindow", Window), ("pad", ctypes.c_char * 64)]


rt = cudart()
dev = torch.device("cuda", 0)
props = torch.cuda.get_device_properties(0)
maxp = ctypes.c_int(0)
rt.cudaDeviceGetAttribute(ctypes.byref(maxp), 108, 0)   # cudaDevAttrMaxPersistingL2CacheSize
maxw = ctypes.c_int(0)
rt.cudaDeviceGetAttribute(ctypes.byref(maxw), 109, 0)   # cudaDevAttrMaxAccessPolicyWindowSize
l2 = ctypes.c_int(0)
rt.cudaDeviceGetAttribute(ctypes.byref(l2), 38, 0)     # cudaDevAttrL2CacheSize
print(json.dumps(dict(l2_bytes=l2.value, max_persisting_l2=maxp.value, max_window=maxw.value)), flush=True)

d = bench.make_instance(0)
Cd = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).to(dev)
plan = {name: (variant, opts, cap) for name, variant, opts, cap in bench.PLAN}
for mode in ["none", "persist", "none", "persist"]:
    st = torch.cuda.Stream(dev)
    if mode == "persist":
        rc0 = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(maxp.value))   # cudaLimitPersistingL2CacheSize
        v = AttrValue()
        nb = min(Cd.numel() * 4, maxw.value)
        v.accessPolicyWindow = Window(Cd.data_ptr(), nb, min(1.0, maxp.value / nb), 2, 1)
        rc1 = rt.cudaStreamSetAttribute(ctypes.c_void_p(st.cuda_stream), 1, ctypes.byref(v))
        print(json.dumps(dict(set_limit=rc0, set_window=rc1, window=nb, hit_ratio=min(1.0, maxp.value / nb))), flush=True)
    for name in ["bcfw-GA-GAD-M1-ELS", "bcfw-P-ELS"]:
        variant, opts, cap = plan[name]
        s = sro.Solver(d["a"], d["b"], 1.0, C=Cd, prec="f32", ld=bench.M, stream=st.cuda_stream)
        out = []
        for rep in range(3):
            s.reset()
            torch.cuda.synchronize()
            r = s.solve(variant, cap, seed=11, epsilon=bench.EPS, **opts)
            if rep:
                out.append(r["device_ms"])
        print(json.dumps(dict(mode=mode, name=name, iters=r["iters_done"], device_ms=[round(x, 2) for x in out],
                              us_per_iter=round(min(out) * 1e3 / r["iters_done"], 3))), flush=True)
        s.close()
    if mode == "persist":
        rt.cudaCtxResetPersistingL2Cache()
