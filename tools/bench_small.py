"""Per-step device time of small states (configs[0]/[1] sizes and the range
13..21): one evolve of K steps timed with CUDA events, for the cluster-resident
launch (QAA_OPT_CLUSTER, 13 <= n <= 16), the persistent grid-barrier kernel
(QAA_OPT_PERSIST) and the per-pass kernels; then the F1 sweep (16 replicas of
configs[1]'s T values at dt = 0.05) per kernel. python tools/bench_small.py [K]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)


def inst(n):
    return cnf.load_instance(n)[0] if os.path.exists(cnf.instance_path(n)) else cnf.random_instance(
        n, int(round(4.3 * n)), 1000 + n)


NS = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 12, 13, 14, 15, 16, 18, 20, 21, 22]
for n in NS:
    modes = [("warp", 2, 0, 0), ("quad", 3, 0, 0)] if 13 <= n <= 21 else []
    modes += [("cluster", 0, 1, 0)] if 13 <= n <= 16 else []
    modes += [("persist", 0, 0, 1), ("passes", 0, 0, 0)] if 13 <= n <= 21 else [("default", 1, 1, 0)]
    for name, wflag, cflag, persist in modes:
        with q.Context(0, stream=stream.cuda_stream) as c:
            c.set_option(q.OPT_WARPTILE, wflag)
            c.set_option(q.OPT_CLUSTER, cflag)
            c.set_option(q.OPT_PERSIST, persist)
            c.load_instance(n, inst(n))
            c.init_uniform()
            c.evolve(0.02 * 50, 50)  # warm
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c.evolve(0.02 * K, K)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            st = c.stats()
        print(json.dumps({"n": n, "mode": name, "K": K, "us_per_step": ms * 1e3 / K, "steps_per_s": K / (ms / 1e3),
                          "warp_launches": st["warp_launches"], "cluster_launches": st["cluster_launches"],
                          "persist_launches": st["persist_launches"],
                          "pass_launches": st["pass_launches"]}), flush=True)
# F1 sweep: 16 replicas, T = 1..200 at dt = 0.05 (configs[1]'s sweep style)
Ts = np.array([1, 2, 5, 10, 20, 50, 100, 200, 3, 7, 15, 30, 70, 150, 40, 60], dtype=float)
Ks = (Ts / 0.05).astype(np.int64)
for n in ([] if len(sys.argv) > 3 else (13, 14, 15, 16)):
    for name, wflag, cflag in (("quad-teams", 3, 0), ("warp-teams", 2, 0), ("cluster", 0, 1), ("smem-cluster", 0, 0)):
        with q.Context(0, stream=stream.cuda_stream) as c:
            c.set_option(q.OPT_WARPTILE, wflag)
            c.set_option(q.OPT_CLUSTER, cflag)
            c.load_instance(n, inst(n))
            c.sweep(Ts[:2], Ks[:2])  # warm
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c.sweep(Ts, Ks)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        print(json.dumps({"sweep_n": n, "mode": name, "replicas": len(Ts), "replica_steps": int(Ks.sum()),
                          "ms": ms, "replica_steps_per_s": float(Ks.sum()) / (ms / 1e3),
                          "longest_replica_us_per_step": ms * 1e3 / float(Ks.max())}), flush=True)
