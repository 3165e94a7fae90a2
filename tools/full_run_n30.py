"""configs[3] end to end on one B200: the n = 30 unique-solution instance, T = 200,
K = 10^4 midpoint schedule (dt = 0.02), run in windows of 1000 steps.
Records the norm drift every window (R15), the final P_succ and <H_P>, and a
second identical run's final state checksum (determinism). If the host has
room for the oracle at n = 30, the first 10 steps are also compared with the
oracle on sampled amplitudes.

    python tools/full_run_n30.py [--oracle-steps 10] > profiles/r01_full_run_n30.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--oracle-steps", type=int, default=10)
ap.add_argument("--window", type=int, default=1000)
args = ap.parse_args()

n, T, K = 30, 200.0, 10_000
cl, sol = cnf.load_instance(n)
sched = (np.arange(K) + 0.5) / K
dt = T / K
out = {"config": "n=30 unique-solution 3-SAT, T=200, K=1e4 (dt=0.02), midpoint schedule", "m": len(cl),
       "solution": int(sol)}
idx = np.random.default_rng(7).integers(0, 1 << n, 256)


# libqaa enqueues on this (non-default) stream; the timing events go on the same stream
stream = torch.cuda.Stream(device=0)
torch.cuda.set_stream(stream)


def run(record):
    with q.Context(0, stream=stream.cuda_stream) as c:
        c.load_instance(n, cl)
        c.init_uniform()
        norms, t_dev = [], 0.0
        for w in range(K // args.window):
            s = sched[w * args.window:(w + 1) * args.window]
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            ev0.record(stream)
            c.evolve(dt * args.window, args.window, s)
            ev1.record(stream)
            torch.cuda.synchronize()
            t_dev += ev0.elapsed_time(ev1) / 1e3
            if record:
                norms.append(c.norm2() - 1.0)
        res = {"device_s": t_dev, "steps_per_s": K / t_dev, "p_succ": c.success_prob(), "energy_s1": c.energy(1.0),
               "norm_minus_1": c.norm2() - 1.0, "sample": c.state(0, 1)[0]}
        samp = np.array([c.state(int(i), 1)[0] for i in idx])
        res["sample_checksum"] = float(np.abs(samp).sum())
        res["_samp"] = samp
        if record:
            res["norm_minus_1_per_window"] = norms
        return res


t0 = time.time()
a = run(True)
b = run(False)
out["run"] = {k: v for k, v in a.items() if not k.startswith("_") and k != "sample"}
out["deterministic"] = bool(np.array_equal(a["_samp"], b["_samp"]))
out["max_abs_norm_drift"] = float(max(abs(x) for x in a["norm_minus_1_per_window"]))

# oracle on the first steps (the oracle's own step count, sampled amplitudes)
try:
    import psutil
    avail = psutil.virtual_memory().available
except Exception:
    avail = 0
need = (1 << n) * (16 * 2 + 2)  # state + scratch + energies
if args.oracle_steps > 0 and avail > 1.5 * need:
    from oracle import oracle
    k0 = args.oracle_steps
    t1 = time.time()
    E = oracle.energy_table(n, cl)
    want = oracle.evolve(n, E, oracle.init_uniform(n), dt * k0, k0, sched[:k0])
    with q.Context(0, stream=stream.cuda_stream) as c:
        c.load_instance(n, cl)
        c.init_uniform()
        c.evolve(dt * k0, k0, sched[:k0])
        got = np.array([c.state(int(i), 1)[0] for i in idx])
    out["oracle_prefix"] = {"steps": k0, "samples": len(idx), "max_abs_diff": float(np.abs(got - want[idx]).max()),
                            "oracle_s": time.time() - t1, "host_cores": os.cpu_count()}
    del want, E
else:
    out["oracle_prefix"] = {"skipped": f"host memory available {avail / 2**30:.0f} GiB < 1.5 x {need / 2**30:.0f} GiB"}
out["wall_s"] = time.time() - t0
print(json.dumps(out))
