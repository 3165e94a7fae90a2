#!/usr/bin/env python
"""F2 workload: the paper's own GPU kernel -- the clause-energy
table E(x) for every assignment -- timed on the B200 through
qaa_time_energy_table, next to the CPU oracle's O-2 loop on the host cores
(the paper's CPU-vs-GPU methodology). Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

out = {"workload": "energy table E(x), x in [0, 2^n) (K1 / the paper's kernel)", "rows": []}
with q.Context(0) as c:
    for n in (20, 24, 30, 32):
        cl, _ = cnf.load_instance(n)
        c.load_instance(n, cl)
        ms = c.time_energy_table(5)
        m = len(cl)
        amps = 1 << n
        # issue-rate roofline: per 16 assignments and clause the test needs at
        # least 6 integer instructions (32-bit AND + compare, 4 predicated
        # packed-byte adds; the clause-record load is amortised over 4 groups)
        issue_peak = 148 * 4 * 32 * 1.965e9  # thread-instructions / s
        roof_ms = amps / 16 * m * 6 / issue_peak * 1e3
        out["rows"].append({"n": n, "m": m, "gpu_ms": ms, "assignments_per_s": amps / (ms / 1e3),
                            "clause_evals_per_s": amps * m / (ms / 1e3), "issue_roofline_ms": roof_ms,
                            "frac_of_issue_roofline": roof_ms / ms})
# CPU oracle (plain literal loops, OpenMP over x), bounded sample
from oracle import oracle  # noqa: E402

oracle.build()
n = 24
cl, _ = cnf.load_instance(n)
t0 = time.perf_counter()
oracle.energy_table(n, cl)
dt = time.perf_counter() - t0
out["cpu_oracle"] = {"n": n, "s": dt, "assignments_per_s": (1 << n) / dt, "cores": oracle.num_threads()}
print(json.dumps(out))
