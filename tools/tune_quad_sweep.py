"""Tuning probe for the quad-warp team sweep (QAA_OPT_SWEEP_TUNE): tiles per CTA
x team-barrier poll backoff, 16 replicas of configs[1]'s sweep (T = 1..200 at
dt = 0.05), device time. python tools/tune_quad_sweep.py [n,...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
Ts = np.array([1, 2, 5, 10, 20, 50, 100, 200, 3, 7, 15, 30, 70, 150, 40, 60], dtype=float)
Ks = (Ts / 0.05).astype(np.int64)
NS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [13, 14, 15, 16]
for n in NS:
    cl = cnf.load_instance(n)[0] if os.path.exists(cnf.instance_path(n)) else cnf.random_instance(
        n, int(round(4.3 * n)), 1000 + n)
    for rep in range(2):
        for poll in (0, 256):
            for lt in (0, 1, 2, 3):
                with q.Context(0, stream=stream.cuda_stream) as c:
                    c.set_option(q.OPT_WARPTILE, 3)
                    c.set_option(q.OPT_SWEEP_TUNE, poll * 16 + lt)
                    c.load_instance(n, cl)
                    c.sweep(Ts[:2], Ks[:2])
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    c.sweep(Ts, Ks)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                print(json.dumps({"n": n, "rep": rep, "poll_ns": poll, "tpc": (1 << (lt - 1)) if lt else "auto",
                                  "ms": round(ms, 3), "replica_steps_per_s": round(float(Ks.sum()) / (ms / 1e3))}),
                      flush=True)
        with q.Context(0, stream=stream.cuda_stream) as c:
            c.set_option(q.OPT_WARPTILE, 0)
            c.load_instance(n, cl)
            c.sweep(Ts[:2], Ks[:2])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c.sweep(Ts, Ks)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        print(json.dumps({"n": n, "rep": rep, "engine": "cluster", "ms": round(ms, 3),
                          "replica_steps_per_s": round(float(Ks.sum()) / (ms / 1e3))}), flush=True)
