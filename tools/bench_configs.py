#!/usr/bin/env python
"""Steps/s of every BASELINE config (configs[0..3]) on one GPU, plus the F1 sweep
of configs[1]. Device time with CUDA events; prints one JSON line per config."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402


def timed(fn, stream):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


stream = torch.cuda.Stream(device=0)  # non-default: libqaa launches on it, events too
torch.cuda.set_stream(stream)
rows = []
for n, T, K, Kmeas in ((8, 10.0, 100, 100), (16, 50.0, 1000, 1000), (24, 100.0, 5000, 1000), (30, 200.0, 10000, 60)):
    cl, sol = cnf.load_instance(n)
    with q.Context(0, stream=stream.cuda_stream) as c:
        c.load_instance(n, cl)
        c.init_uniform()
        dt = T / K
        sched = (np.arange(Kmeas) + 0.5) / K
        c.evolve(dt * 5, 5, sched[:5])  # warm-up
        c.reset_stats()
        import time
        t0 = time.perf_counter()
        ms = timed(lambda: c.evolve(dt * Kmeas, Kmeas, sched), stream)
        wall_ms = (time.perf_counter() - t0) * 1e3
        st = c.stats()
        row = {"config": f"n={n} T={T} K={K}", "steps_timed": Kmeas, "ms": ms, "wall_ms": wall_ms,
               "steps_per_s": Kmeas / (ms / 1e3), "groups": st["groups"], "pass_launches": st["pass_launches"], "p_succ_after_timed_prefix": c.success_prob()}
        if n == 8:
            Ts = np.array([1, 2, 5, 10, 20, 50, 100, 200], dtype=float)
            Ks = (Ts / 0.05).astype(np.int64)
            c.sweep(Ts, Ks)
            sms = timed(lambda: c.sweep(Ts, Ks), stream)
            row["sweep_T"] = Ts.tolist()
            row["sweep_p_succ"] = c.sweep(Ts, Ks).tolist()
            row["sweep_ms"] = sms
            row["sweep_total_steps_per_s"] = float(Ks.sum()) / (sms / 1e3)
        rows.append(row)
        print(json.dumps(row), flush=True)
