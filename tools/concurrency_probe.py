"""Where the concurrent bench step spends its time: per solve, host timestamps (thread start, after
reset, after solve) and device timestamps (events on the solver stream before reset / after the
solve) relative to the step's start event."""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

d = bench.make_instance(0)
dev = torch.device("cuda", 0)
Cd = torch.from_numpy(np.ascontiguousarray(d["C32"].T)).to(dev)
runner = bench.StepRunner(d, dev, Cd)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev) if os.environ.get("FLUSH") else None
if os.environ.get("TIMING"):
    runner.set_timing(True)
for rep in range(4):
    if flush is not None:
        flush.fill_(1.0)
    main = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(main)
    h0 = time.perf_counter()
    for st in runner.streams:
        st.wait_event(e0)
    rec = [dict() for _ in bench.PLAN]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in bench.PLAN]

    def work(q):
        name, variant, opts, cap = bench.PLAN[q]
        s = runner.solvers[q]
        rec[q]["t_start"] = (time.perf_counter() - h0) * 1e3
        evs[q][0].record(runner.streams[q])
        s.reset()
        rec[q]["t_reset"] = (time.perf_counter() - h0) * 1e3
        r = s.solve(variant, cap, seed=11, epsilon=bench.EPS, **opts)
        evs[q][1].record(runner.streams[q])
        rec[q]["t_done"] = (time.perf_counter() - h0) * 1e3
        rec[q]["dev_ms"] = r["device_ms"]

    th = [threading.Thread(target=work, args=(q,)) for q in range(len(bench.PLAN))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    e1 = torch.cuda.Event(enable_timing=True)
    for st in runner.streams:
        ev = torch.cuda.Event()
        ev.record(st)
        main.wait_event(ev)
    e1.record(main)
    e1.synchronize()
    step = e0.elapsed_time(e1)
    for q, (name, *_rest) in enumerate(bench.PLAN):
        rec[q]["d_begin"] = e0.elapsed_time(evs[q][0])
        rec[q]["d_end"] = e0.elapsed_time(evs[q][1])
    if rep:
        print(json.dumps(dict(step_ms=round(step, 1), host_ms=round((time.perf_counter() - h0) * 1e3, 1),
                              solves={bench.PLAN[q][0]: {k: round(v, 1) for k, v in rec[q].items()} for q in range(len(bench.PLAN))})),
              flush=True)
runner.close()
