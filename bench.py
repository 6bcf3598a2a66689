#!/usr/bin/env python
"""bench.py — BASELINE.json's metric on BASELINE config [1], through the C-ABI.

Metric: oracle cost-entries/s (GB/s vs HBM peak) and wall time to duality gap <= 1e-6.
Workload (BASELINE configs[1]): m = n = 4096 colour-transfer shape, source and target
colours from 8-component Gaussian mixtures in [0,1]^3 (sigma 0.05, clipped), density
histogram marginals, squared-Euclidean cost materialised in fp32 (promoted to fp64),
lambda = 1. One step = one pass of the whole hot path (every SURVEY §8(a) row) over
that instance: BCFW-P-ELS, BCAFW, BCPFW and BCFW-GA (the paper's BCFW + three fast
variants) plus full FW (Alg. A.1) and batched BCFW (B = 256), each from T^(0) to
g <= 1e-6. The six solves are independent and run concurrently (one handle and CUDA stream
each; a sequential solve is one persistent CTA); --serial-solves runs them one after
another. value = cost entries the kernels read (sro_result.entries_read) / device time of
the step.

Extra keys: `sweep_roofline` (config [3]: the HBM-bound dense gap sweep and FW-ELS to gap),
`configs` (configs [2] and [4]: batched BCFW to gap with fused colour costs, and their fused
gap sweeps) at N = 1; `sharded` at N > 1: FW-ELS on [3] and batched B = 1024 on [4], column-
sharded over the N GPUs with NCCL all-gathers, time to gap as the max over ranks.

N > 1 (torchrun): the sequential BCFW family does not shard (each step depends on
the previous r), so the headline step's ranks are independent replicas on their own seeded
instances (weak scaling, no data-path collective); value = all ranks' entries / max time.

--impl reference times the oracle (plain fp64 C, one host core) on a bounded sample
of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import shutil
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "oracle cost-entries/s (GB/s vs HBM peak) and wall time to duality gap <=1e-6"
UNIT = "cost-entries/s"
EPS = 1e-6
M = N = 4096

# (name, variant, options, iteration cap)
PLAN = [
    ("bcfw-P-ELS", 1, dict(step=1, sampling=1), 400 * N),
    ("bcafw-U-ELS", 2, dict(step=1, sampling=0), 400 * N),
    ("bcpfw-U-ELS", 3, dict(step=1, sampling=0), 400 * N),
    ("bcfw-GA-GAD-M1-ELS", 1, dict(step=1, sampling=2, ga_M=1, ga_inner=1, ga_post_update=1), 400 * N),
    ("fw-ELS", 0, dict(step=1), 20000),
    ("batched-B256-P-ELS", 4, dict(step=1, sampling=1, block_size=256), 400 * (N // 256)),
]


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        if os.environ.get("SRO_BENCH_NO_CLOCKS"):   # A/B only: the contract needs the samples
            return
        try:
            # lowest CPU priority (nice 19): the sampler must not delay the solver threads
            nice = ["nice", "-n", "19"] if shutil.which("nice") else []
            self.proc = subprocess.Popen(nice + ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                                 "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def make_instance(seed):
    from sro_inputs import instance
    return instance(1, seed=seed)


# --------------------------------------------------------------------------- CUDA path
class StepRunner:
    """One step = the six solves of PLAN from T^(0) to g <= EPS on one instance. Each solve has
    its own Solver handle and CUDA stream and all six run concurrently from host threads (the
    C-ABI calls release the GIL): a sequential BCFW-family solve is one persistent CTA (one SM,
    bound by the latency of its dependent steps), so independent solves share the GPU
    instead of queueing. The cost matrix is ONE device copy borrowed by every handle (column-major,
    ld = m), so the L2 holds it once."""

    def __init__(self, d, dev, Cd, concurrent=True, ready=None):
        import torch
        import paper_2103_05857_b200 as sro
        self.torch = torch
        self.concurrent = concurrent
        # the sequential solves (one persistent CTA each, latency-bound, with short full-GPU gap
        # sweeps between segments) get high-priority streams, so those sweeps are not queued
        # behind the FW / batched solves' GPU-wide kernels
        self.streams = [torch.cuda.Stream(dev, priority=-1 if variant in (1, 2, 3) else 0)
                        for _, variant, _, _ in PLAN]
        # the borrowed C must be complete before sro_create validates it on each handle's stream
        ready = ready if ready is not None else torch.cuda.current_stream(dev).record_event()
        for st in self.streams:
            st.wait_event(ready)
        self.solvers = [sro.Solver(d["a"], d["b"], 1.0, C=Cd, prec="f32", device=dev.index, stream=st.cuda_stream,
                                   ld=M) for st in self.streams]
        self.ga_steps = 0   # GA steps run (the roofline's traffic weighting)

    def run(self, entries_acc, ttg):
        """Enqueue the step after the current stream's pending work; returns after it completes.
        Device time: (e0 on the caller's stream) ... (e1 after every solver stream)."""
        torch = self.torch
        main = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for st in self.streams:
            st.wait_event(e0)
        results = [None] * len(PLAN)
        errors = []

        dbg = os.environ.get("SRO_BENCH_DEBUG")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in PLAN] if dbg else None

        def work(q):
            try:
                name, variant, opts, cap = PLAN[q]
                s = self.solvers[q]
                if self.concurrent and variant in (0, 4) and hasattr(os, "setpriority"):
                    # FW / batched are throughput work whose host threads launch often; on a
                    # host with few cores they would delay the wake-ups of the latency-bound
                    # sequential solves' threads (whose GPU then idles between segments)
                    try:
                        os.setpriority(os.PRIO_PROCESS, threading.get_native_id(), 10)
                    except OSError:
                        pass
                if dbg:
                    evs[q][0].record(self.streams[q])
                s.reset()
                results[q] = s.solve(variant, cap, seed=11, epsilon=EPS, **opts)
                if dbg:
                    evs[q][1].record(self.streams[q])
            except Exception as e:  # noqa: BLE001
                errors.append(e)

        if self.concurrent:
            threads = [threading.Thread(target=work, args=(q,)) for q in range(len(PLAN))]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
        else:
            for q in range(len(PLAN)):
                work(q)
        if errors:
            raise errors[0]
        for st in self.streams:
            ev = torch.cuda.Event()
            ev.record(st)
            main.wait_event(ev)
        e1.record(main)
        e1.synchronize()
        if dbg:
            print(json.dumps({PLAN[q][0]: (round(e0.elapsed_time(evs[q][0]), 2), round(e0.elapsed_time(evs[q][1]), 2),
                                           round(results[q]["device_ms"], 2)) for q in range(len(PLAN))}),
                  file=sys.stderr, flush=True)
        for (name, _, opts, cap), r in zip(PLAN, results):
            if not r["converged"]:
                raise RuntimeError(f"{name} did not reach g <= {EPS} within {cap} iterations (gap {r['gap']})")
            entries_acc.append(r["entries_read"])
            ttg[name] = ttg.get(name, []) + [r["device_ms"]]
            if opts.get("sampling") == 2:
                self.ga_steps += r["iters_done"]
        return e0.elapsed_time(e1)

    def objective(self):
        return [s.objective() for s in self.solvers]

    def stats(self, reset=False):
        tot = {"ga_steps": self.ga_steps}
        for s in self.solvers:
            for k, v in s.stats(reset).items():
                tot[k] = tot.get(k, 0) + v
        if reset:
            self.ga_steps = 0
        return tot

    def set_timing(self, on):
        # per-kernel event timing on the sequential solves only (the roofline's dominant family):
        # on FW / batched it would put events around every block step and turn off the CUDA
        # graph replay of their steps
        for (_, variant, _, _), s in zip(PLAN, self.solvers):
            s.set_timing(on and variant in (1, 2, 3))

    def close(self):
        for s in self.solvers:
            s.close()


# Test-only emulation of N ranks on ONE GPU (SRO_BENCH_EMULATE_RANKS=1 under torchrun): gloo instead
# of NCCL for the process group, every rank on cuda:0, and the sharded legs exchange through the
# library's host all-gather (sro_params.exchange) — so the N > 1 control flow of this file runs
# end to end on a 1-GPU box. Its numbers are not bench values.
EMULATE = os.environ.get("SRO_BENCH_EMULATE_RANKS") == "1"


def _max_sum(vals, dev):
    """Element-wise max and sum over ranks of a small float64 vector (NCCL on the device, or gloo
    on the host in emulation)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device="cpu" if EMULATE else dev)
    tmax, tsum = t.clone(), t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    return tmax.tolist(), tsum.tolist()


def bench_sro(args, rank, world, local_rank):
    import torch

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    d = make_instance(seed=rank)
    C32 = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).pin_memory()   # column-major (n, m)
    Cd = C32.to(dev)
    runner = StepRunner(d, dev, Cd, concurrent=not args.serial_solves)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up; the clock sampler (an nvidia-smi process whose start-up stalls the GPU's host side
    # for tens of ms) and the per-kernel event timing start before the last warm-up step, so their
    # first-use costs stay out of the timed steps; the sampler runs through the timed region
    clocks = ClockSampler(local_rank)
    for w in range(args.warmup):
        if w == args.warmup - 1:
            clocks.start()
            runner.set_timing(True)
        runner.run([], {})
    torch.cuda.synchronize()
    runner.stats(reset=True)
    entries, ttg = [], {}
    step_ms = []
    barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.fill_(1.0)                      # L2 flushed between timed steps (outside the events)
        step_ms.append(runner.run(entries, ttg))
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    stats = runner.stats(reset=True)
    runner.set_timing(False)
    runner.close()
    total_ms = float(sum(step_ms))
    my_entries = float(sum(entries))

    # e2e: the same step through the public API from pinned host buffers: H2D of C, a, b and
    # handle creation inside the timed region, D2H of every solve's objective at the end
    a_h = torch.from_numpy(d["a"]).pin_memory()
    b_h = torch.from_numpy(d["b"]).pin_memory()
    e2e_ms, e2e_entries = [], []
    for _ in range(max(1, min(args.steps, 3))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Cd2 = C32.to(dev, non_blocking=True)
        d2 = dict(d, a=a_h.numpy(), b=b_h.numpy())
        r2 = StepRunner(d2, dev, Cd2, concurrent=not args.serial_solves)
        ent = []
        r2.run(ent, {})
        fs = r2.objective()                    # D2H of the step's results
        r2.close()
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_entries.append(sum(ent))
        assert np.all(np.isfinite(fs))
        del Cd2
    h2d = C32.numel() * 4 + a_h.numel() * 8 + b_h.numel() * 8
    d2h = (8 * 4 + 8) * len(PLAN)      # per-solve result scalars + objective

    if world > 1:
        import torch.distributed as dist
        tmax, tsum = _max_sum([total_ms, my_entries, sum(e2e_ms), sum(e2e_entries)], dev)
        max_ms, all_entries = tmax[0], tsum[1]
        e2e_max_ms, e2e_all_entries = tmax[2], tsum[3]
    else:
        max_ms, all_entries = total_ms, my_entries
        e2e_max_ms, e2e_all_entries = sum(e2e_ms), sum(e2e_entries)
    sweep_rf, legs, sharded = None, None, None
    if not args.no_sweep_check:
        del flush, Cd
        torch.cuda.synchronize()
        if world > 1:
            sharded = sharded_legs(rank, world, local_rank)
        elif rank == 0:
            sweep_rf = sweep_roofline_config3(local_rank, measured_peaks())
            legs = configs_legs_single(local_rank)
    return dict(max_ms=max_ms, all_entries=all_entries, stats=stats, clocks=clk, ttg=ttg, step_ms=step_ms,
                sweep_roofline=sweep_rf, configs_legs=legs, sharded=sharded,
                e2e_value=e2e_all_entries / (e2e_max_ms * 1e-3), h2d=h2d, d2h=d2h, instance=d,
                e2e_ms=[round(x, 2) for x in e2e_ms])


def roofline_from_stats(stats, peaks):
    """Dominant kernel family by device time; achieved = algorithmic bytes / its time."""
    fam = {"bcfw": stats["bcfw_ms"], "sweep": stats["sweep_ms"], "block": stats["block_ms"]}
    dom = max(fam, key=fam.get)
    peak = float(peaks.get("hbm_gbs", 6650.0))
    if dom == "bcfw":
        # one fp32 column (m entries x 4 B) per BCFW step, + its support, per launch
        bytes_ = stats["bcfw_steps"] * M * 4.0
        launches = max(1, stats["bcfw_launches"])
        name = "k_bcfw_pipe / k_bcfw_ga_pipe (persistent sequential BCFW-family loop, 1 CTA)"
    elif dom == "sweep":
        bytes_ = stats["sweep_columns"] * M * 4.0
        launches = max(1, stats["sweep_launches"])
        name = "k_lmo_sweep (column LMO + gap epilogue)"
    else:
        bytes_ = 0.0
        launches = max(1, stats["block_steps"])
        name = "FW / batched plain step"
    t_ms = fam[dom]
    achieved = bytes_ / (t_ms * 1e-3) / 1e9 if t_ms > 0 else 0.0
    shares = {k: round(v / max(1e-9, sum(fam.values())), 4) for k, v in fam.items()}
    shares["timed"] = "the sequential solves (their persistent kernels and gap sweeps)"
    out = {"bound": "hbm", "kernel": name, "achieved": round(achieved, 3), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 5), "traffic": None, "avg_launch_ms": round(t_ms / launches, 4),
           "algorithmic_bytes_per_launch": bytes_ / launches, "time_share": shares,
           "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, of measured)"}
    if dom == "bcfw" and stats["bcfw_steps"]:
        # the sequential family is bound by the latency of one dependent step, not by HBM.
        # traffic: DRAM bytes per step of each kernel from this build's ncu captures
        # (profiles/r02_ncu_traffic.json), weighted by the steps each kernel ran in the timed region
        us = t_ms * 1e3 / stats["bcfw_steps"]
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")))
            per = {k: (tr[k]["dram_bytes_read"] + tr[k]["dram_bytes_write"]) / tr[k]["steps"]
                   for k in ("k_bcfw_ga_pipe", "k_bcfw_pipe")}
            ga_steps = min(stats["bcfw_steps"], stats.get("ga_steps", 0))
            tot = ga_steps * per["k_bcfw_ga_pipe"] + (stats["bcfw_steps"] - ga_steps) * per["k_bcfw_pipe"]
            out["traffic"] = round(tot / launches, 1)
            out["traffic_source"] = ("ncu --set full dram__bytes_read+write per step (profiles/r02_ncu_traffic.json): "
                                     f"k_bcfw_ga_pipe {per['k_bcfw_ga_pipe']:.0f} B, k_bcfw_pipe {per['k_bcfw_pipe']:.0f} B, "
                                     f"weighted by the timed region's steps ({ga_steps} GA of {stats['bcfw_steps']})")
        except (OSError, KeyError, ValueError):
            out["traffic"] = None
        out["step_latency"] = {"us_per_step": round(us, 4), "cycles_per_step_at_1965MHz": round(us * 1965.0, 1),
                               "single_cta_floor_cycles": 420,
                               "floor_source": "profiles/r01_lmo_microbench.log: register LMO + REDUX argmin + 2 barriers"}
    return out


def sweep_roofline_config3(local_rank, peaks, sweeps=3):
    """The HBM-bound row of the path at BASELINE config [3]: m = n = 65536 iid uniform fp32
    cost materialised on the device (2^32 entries = 17.18 GB, far above the 126 MB L2),
    LMO + column-gap sweeps (k_lmo_sweep_bulk + k_lmo_merge) timed by the library's CUDA
    events on the solver stream, then FW-ELS from T^(0) to g <= 1e-6."""
    import paper_2103_05857_b200 as sro
    from sro_inputs import instance
    d = instance(3, seed=0)
    s = sro.Solver(d["a"], d["b"], 1.0, cost="hash", hash_seed=d["hash_seed"], device=local_rank)
    s.gap()                                   # warm-up
    s.set_timing(True)
    s.stats(reset=True)
    for _ in range(sweeps):
        s.gap()
    st = s.stats(reset=True)
    per_ms = st["sweep_ms"] / max(1, st["sweep_launches"])
    byts = 65536.0 * 65536.0 * 4.0
    peak = float(peaks.get("hbm_gbs", 6650.0))
    ach = byts / (per_ms * 1e-3) / 1e9
    r = s.solve(sro.SRO_FW, 500, step=sro.STEP_ELS, epsilon=EPS)
    st2 = s.stats(reset=True)
    s.close()
    return {"workload": "BASELINE configs[3]: m=n=65536, C iid U[0,1) fp32 materialised column-major (17.18 GB)",
            "kernel": "k_lmo_sweep_bulk + k_lmo_merge (one gap sweep: LMO + column gaps over all 65536 columns)",
            "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
            "peak_note": ("the measured peak is a copy (read + write bytes); this kernel only reads, so it can "
                          "exceed it: against the 8 TB/s nominal HBM3e rate frac = "
                          f"{ach / 8000.0:.3f}, against the read-only stream microbenchmark (7.3 TB/s, "
                          f"profiles/r01_microbench.jsonl) {ach / 7300.0:.3f}"),
            "algorithmic_bytes_per_launch": byts, "avg_launch_ms": round(per_ms, 4), "sweeps_timed": sweeps,
            "traffic": 17181008000.0 + 16534016.0,
            "traffic_source": ("ncu --set full dram__bytes_read.sum + dram__bytes_write.sum of one k_lmo_sweep_bulk "
                               "launch on this workload, closing round-2 build "
                               "(profiles/r02_ncu_sweep3.md): 1.0010 x the algorithmic bytes"),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, of measured)",
            "fw_els_time_to_gap_ms": round(r["device_ms"], 3), "fw_els_iterations": r["iters_done"],
            "fw_els_converged": bool(r["converged"]), "fw_gap": r["gap"],
            "fw_entries_per_s": r["entries_read"] / (r["device_ms"] * 1e-3),
            "fw_sweep_share": round(st2["sweep_ms"] / max(1e-9, st2["block_ms"]), 4)}


def _timed_solve(s, variant, cap, **opts):
    """One solve from T^(0) after an untimed warm-up solve of the same call (workspaces, CUDA
    graph capture): the device time of the call (CUDA events on the solver stream)."""
    s.reset()
    s.solve(variant, cap, seed=11, epsilon=EPS, **opts)
    s.reset()
    return s.solve(variant, cap, seed=11, epsilon=EPS, **opts)


def configs_legs_single(local_rank):
    """BASELINE configs [2] and [4] on one GPU (fused fp32 squared-Euclidean costs from d = 3
    colours, batched BCFW with B = 256 / 1024, P order, exact line search) from T^(0) to
    g <= 1e-6: time to gap, block steps, cost entries read per second, and the fused colour
    gap sweep alone (the whole m x n LMO + column gaps, timed by the library's CUDA events)."""
    import paper_2103_05857_b200 as sro
    from sro_inputs import instance
    out = {}
    for cfg, B in ((2, 256), (4, 1024)):
        d = instance(cfg, seed=0)
        s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=d["Y"], cost="sqeuclid", prec="f32", device=local_rank)
        r = _timed_solve(s, sro.SRO_BATCHED, 400 * (d["n"] // B), step=sro.STEP_ELS, sampling=sro.SAMPLE_P,
                         block_size=B)
        s.gap()
        s.set_timing(True)
        s.stats(reset=True)
        for _ in range(3):
            s.gap()
        st = s.stats(reset=True)
        s.close()
        sweep_ms = st["sweep_ms"] / max(1, st["sweep_launches"])
        ent = float(d["m"]) * d["n"]
        # the fused colour sweep is bound by instruction issue, not memory: 201 SASS instructions
        # per 4 rows x 4 columns in its inner loop (k_lmo_sweep<SrcColour<float>, 4, 512>: 24 FADD2 +
        # 24 FMUL2 for the packed differences and squares, 32 FADD, 16 F2F, 16 DADD, 16 DSETP, 44
        # selects, 8 LDS, ...), one issue per cycle per SM sub-partition
        import torch
        sms = torch.cuda.get_device_properties(local_rank).multi_processor_count
        mhz = float(measured_peaks().get("sm_max_mhz", 1965.0))
        per_entry = 201 / 16.0
        issue_peak = sms * 4 * mhz * 1e6 * 32 / per_entry
        out[f"config{cfg}"] = {
            "workload": f"BASELINE configs[{cfg}]: m={d['m']}, n={d['n']}, fused fp32 sqeuclid, batched B={B}, P, ELS",
            "time_to_gap_ms": round(r["device_ms"], 3), "block_steps": r["iters_done"],
            "converged": bool(r["converged"]), "gap": r["gap"], "us_per_block_step": round(
                1e3 * r["device_ms"] / max(1, r["iters_done"]), 2),
            "entries_per_s": r["entries_read"] / (r["device_ms"] * 1e-3),
            "gap_sweep_ms": round(sweep_ms, 4), "gap_sweep_entries_per_s": ent / (sweep_ms * 1e-3),
            "gap_sweep_roofline": {"bound": "alu", "achieved": ent / (sweep_ms * 1e-3), "peak": issue_peak,
                                   "unit": "entries/s", "frac": round(ent / (sweep_ms * 1e-3) / issue_peak, 4),
                                   "peak_derivation": f"{sms} SMs x 4 sub-partitions x {mhz:.0f} MHz x 32 lanes / "
                                                      "12.56 instructions per entry (SASS of the inner loop, "
                                                      "packed fp32; the unpacked loop took 16)"}}
    return out


def sharded_legs(rank, world, local_rank):
    """N > 1: the column-sharded variants of north_star through NCCL (one shard per GPU,
    sro_params.nranks = shards = N). [3]: FW-ELS from T^(0) to g <= 1e-6 on the
    m = n = 65536 iid cost, each rank generating its own 65536 x 65536/N column shard on the
    device; [4]: batched B = 1024 (shard_block = 1024, each rank B/N columns of every block),
    P, ELS, to g <= 1e-6. Time = max over ranks of the solve's device time; entries = all
    ranks' cost entries read."""
    import torch
    import torch.distributed as dist

    import paper_2103_05857_b200 as sro
    from paper_2103_05857_b200.dist import host_allgather, share_unique_id, shard_cost_inputs
    from sro_inputs import instance
    dev = torch.device("cuda", local_rank)
    out = {}
    for cfg in (3, 4):
        d = instance(cfg, seed=0)
        # NCCL unique id (or, emulating ranks on one GPU, the host all-gather over gloo)
        xk = dict(exchange=host_allgather()) if EMULATE else dict(nccl_id=share_unique_id())
        if cfg == 3:
            s = sro.Solver(d["a"], d["b"], 1.0, cost="hash", hash_seed=d["hash_seed"], device=local_rank,
                           shards=world, nranks=world, rank=rank, **xk)
            r = _timed_solve(s, sro.SRO_FW, 500, step=sro.STEP_ELS)
            per = "FW iteration"
        else:
            _, Yl = shard_cost_inputs(world, rank, 1024, Y=d["Y"])
            s = sro.Solver(d["a"], d["b"], 1.0, X=d["X"], Y=Yl, cost="sqeuclid", prec="f32", device=local_rank,
                           shards=world, shard_block=1024, nranks=world, rank=rank, **xk)
            r = _timed_solve(s, sro.SRO_BATCHED, 400 * (d["n"] // 1024), step=sro.STEP_ELS, sampling=sro.SAMPLE_P,
                             block_size=1024)
            per = "block step"
        s.close()
        tmax, tsum = _max_sum([r["device_ms"], float(r["entries_read"])], dev)
        ms = tmax[0]
        out[f"config{cfg}"] = {
            "workload": (f"BASELINE configs[{cfg}] column-sharded over {world} GPUs (" +
                         ("FW-ELS, hash cost generated per shard" if cfg == 3 else
                          "batched B=1024, P, ELS, fused fp32 sqeuclid") + ")"),
            "shards": world, "exchange": "ncclAllGather of the per-shard 256-chunk subtrees (R19), 2 per " + per,
            "time_to_gap_ms": round(ms, 3), "iterations": r["iters_done"], "converged": bool(r["converged"]),
            "gap": r["gap"], f"ms_per_{per.replace(' ', '_')}": round(ms / max(1, r["iters_done"]), 4),
            "entries_per_s": tsum[1] / (ms * 1e-3)}
        if EMULATE:
            out[f"config{cfg}"]["emulated"] = "ranks share one GPU, host all-gather over gloo: not a bench value"
    return out


# --------------------------------------------------------------------------- oracle (CPU)
def oracle_sample(d, epochs=3, time_budget_s=25.0):
    """The oracle as it stands, single host core, on a bounded sample of the step:
    every PLAN variant from T^(0) for `epochs` epochs (FW: 3*epochs iterations,
    batched: `epochs` epochs), stopping early when the time budget is spent."""
    import oracle as orc
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    o = orc.Oracle(d["a"], d["b"], 1.0, C=d["C32"].astype(np.float64), cap=31)
    entries, wall = 0, 0.0
    done = []
    for name, variant, opts, _ in PLAN:
        iters = epochs * N if variant in (1, 2, 3) else (3 * epochs if variant == 0 else epochs * (N // 256))
        o.reset()
        kw = dict(opts)
        t0 = time.perf_counter()
        r = o.solve(variant, iters, seed=11, epsilon=EPS, **kw)
        wall += time.perf_counter() - t0
        entries += r["entries_scanned"]
        done.append(f"{name}:{r['iters_done']}")
        if wall > time_budget_s:
            break
    return entries, wall, done


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return 1


def host_cpu():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def bench_reference(args, rank, world):
    if rank != 0:
        return None
    d = make_instance(seed=0)
    per = []
    tot_e, tot_t = 0, 0.0
    for s in range(args.warmup + args.steps):
        e, t, done = oracle_sample(d, epochs=1, time_budget_s=60.0)
        if s >= args.warmup:
            per.append(t)
            tot_e += e
            tot_t += t
    v = tot_e / tot_t
    sample = ("each step: every PLAN variant from T^(0) for 1 epoch (FW 3 iterations, batched 1 epoch of B=256 "
              f"blocks) on the config-[1] instance; variants/iterations: {done}")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "host_cpu": host_cpu()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def config_block(world):
    return {"workload": "BASELINE configs[1]: m=n=4096 colour-transfer (8-comp. Gaussian mixtures, sigma 0.05, "
                        "density marginals), squared-Euclidean C materialised fp32 -> fp64, lambda=1",
            "m": M, "n": N, "lambda": 1.0, "epsilon": EPS, "cost_storage": "f32",
            "variants": [p[0] for p in PLAN], "replicas": world, "parallelism": f"replicas{world}",
            "solves": "the six solves of a step run concurrently, one stream and handle each (--serial-solves: one after another)",
            "l2": "flushed between timed steps (256 MiB write outside the timed events)",
            "global_batch": world, "seq_len": None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sro", choices=["sro", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--serial-solves", action="store_true",
                    help="run the six solves of a step one after another instead of concurrently")
    ap.add_argument("--no-sweep-check", action="store_true",
                    help="skip the extra legs (sweep_roofline, configs [2]/[4], the sharded legs at N > 1)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = 0 if EMULATE else int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = bench_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return 0
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if EMULATE else "nccl")
    res = bench_sro(args, rank, world, local_rank)
    if rank == 0:
        peaks = measured_peaks()
        value = res["all_entries"] / (res["max_ms"] * 1e-3)
        ttg = {k: round(statistics.median(v), 3) for k, v in res["ttg"].items()}
        cfg = config_block(world)
        cfg["host_cpus"] = {"os_cpu_count": os.cpu_count(), "affinity": cpu_cores()}
        if args.serial_solves:
            cfg["solves"] = "the six solves of a step run one after another on one stream each"
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["max_ms"] / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": cfg,
                "time_to_gap_ms": ttg,
                "gb_per_s_equiv": round(value * 4 / 1e9, 3),
                "roofline": roofline_from_stats(res["stats"], peaks),
                "sweep_roofline": res.get("sweep_roofline"),
                "configs": res.get("configs_legs"),
                "sharded": res.get("sharded"),
                "clocks": res["clocks"],
                "e2e": {"value": res["e2e_value"], "unit": UNIT, "h2d_bytes_per_step": res["h2d"],
                        "d2h_bytes_per_step": res["d2h"], "ms_per_step": res["e2e_ms"]},
                "gpu_launches": int(res["stats"]["kernel_launches"])}
        if world == 1 and not args.no_cpu_baseline:
            e, t, done = oracle_sample(res["instance"], epochs=3)
            line["cpu_baseline"] = {"value": e / t, "unit": UNIT, "cores": 1, "kind": "oracle",
                                    "sample": f"every PLAN variant from T^(0) for <=3 epochs on the same instance "
                                              f"(FW 9 iterations, batched 3 epochs), 25 s budget: {done}",
                                    "host_cpu": host_cpu(), "host_cores_available": cpu_cores()}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
