"""Full-size runs of BASELINE configs [2], [3], [4] on one GPU (probe, not the bench).

[3]: m = n = 65536 iid uniform fp32 cost materialised on the device (16 GiB):
     LMO gap sweeps (HBM roofline of k_lmo_sweep) and FW-ELS to g <= 1e-6.
[2]: m = n = 16384 quantised mixture colours, fused fp32 sqeuclid, batched B = 256, P, ELS.
[4]: m = 4096, n = 262144 mixture colours, fused fp32 sqeuclid, batched B = 1024, P, ELS.
Prints one JSON object per measurement.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05857_b200 as sro  # noqa: E402
from sro_inputs import instance  # noqa: E402


def emit(**kw):
    print(json.dumps(kw), flush=True)


def cfg3(sweeps=5, fw_iters=200, fw=True):
    d = instance(3, seed=0)
    t0 = time.perf_counter()
    s = sro.Solver(d["a"], d["b"], 1.0, cost="hash", hash_seed=d["hash_seed"])
    emit(cfg=3, what="create", s=time.perf_counter() - t0)
    s.gap()
    s.set_timing(True)
    s.stats(reset=True)
    for _ in range(sweeps):
        s.gap()
    st = s.stats(reset=True)
    per = st["sweep_ms"] / st["sweep_launches"]
    byts = 65536.0 * 65536.0 * 4
    emit(cfg=3, what="gap_sweep", ms=per, GBps=byts / per / 1e6, entries_per_s=65536.0 ** 2 / per * 1e3,
         slab=os.environ.get("SRO_SLAB", "default"))
    if not fw:
        s.close()
        return
    r = s.solve(sro.SRO_FW, fw_iters, step=sro.STEP_ELS, epsilon=1e-6)
    st = s.stats(reset=True)
    emit(cfg=3, what="fw_els", iters=r["iters_done"], gap=r["gap"], converged=r["converged"], ms=r["device_ms"],
         sweep_ms=st["sweep_ms"], block_ms=st["block_ms"], sweeps=st["sweep_launches"],
         GBps_sweep=byts * st["sweep_launches"] / st["sweep_ms"] / 1e6 if st["sweep_ms"] else None)
    s.close()


def batched(cfg, B, epochs=40):
    d = instance(cfg, seed=0)
    s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32")
    s.set_timing(True)
    s.stats(reset=True)
    r = s.solve(sro.SRO_BATCHED, epochs * (d["n"] // B), seed=1, step=sro.STEP_ELS, sampling=sro.SAMPLE_P,
                block_size=B, epsilon=1e-6)
    st = s.stats(reset=True)
    emit(cfg=cfg, what=f"batched_B{B}", iters=r["iters_done"], epochs=r["iters_done"] / (d["n"] // B), gap=r["gap"],
         converged=r["converged"], ms=r["device_ms"], entries=r["entries_scanned"],
         entries_per_s=r["entries_scanned"] / r["device_ms"] * 1e3, sweep_ms=st["sweep_ms"], block_ms=st["block_ms"],
         launches=st["kernel_launches"])
    tot, _, _ = s.gap()
    s.set_timing(True)
    s.stats(reset=True)
    for _ in range(3):
        s.gap()
    st = s.stats(reset=True)
    per = st["sweep_ms"] / st["sweep_launches"]
    emit(cfg=cfg, what="gap_sweep", ms=per, entries_per_s=d["m"] * d["n"] / per * 1e3,
         slab=os.environ.get("SRO_SLAB", "default"))
    s.close()


if __name__ == "__main__":
    which = sys.argv[1:] or ["3", "2", "4"]
    for w in which:
        if w == "3":
            cfg3()
        elif w == "3s":
            cfg3(fw=False)
        elif w == "2":
            batched(2, 256)
        elif w == "4":
            batched(4, 1024)
