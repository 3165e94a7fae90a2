"""A/B of the L2-blocked step's publish batching (QAA_OPT_SUPER_PUB) at n = 30,
interleaved in one process: per-launch kernel ms from the library's events, and
the group-k deferral rate (QAA_OPT_SUPER bit 10). usage: ab_pub.py K pub1 [pub2 ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

K = int(sys.argv[1])
pubs = [int(x) for x in sys.argv[2:]]
n = 30
cl = cnf.load_instance(n)[0]
res = {p: [] for p in pubs}
idx = np.random.default_rng(3).integers(0, 1 << n, 64)
amps = {}
with q.Context(0) as c:
    c.load_instance(n, cl)
    for rep in range(4):
        for p in pubs:
            c.set_option(q.OPT_SUPER_PUB, p)
            c.init_uniform()
            c.evolve(200.0 * 2 / 10000, 2)  # warm
            c.reset_stats()
            c.set_option(q.OPT_PROFILE, 1)
            c.evolve(200.0 * K / 10000, K)
            st = c.stats()
            c.set_option(q.OPT_PROFILE, 0)
            res[p].append(st["super_kernel_ms"] / max(st["super_kernels_timed"], 1))
            if rep == 0:
                amps[p] = np.array([c.state(int(i), 1)[0] for i in idx])
for p in pubs:
    same = np.array_equal(amps[p], amps[pubs[0]])
    print(f"pub={p}: super launch ms {' '.join(f'{x:.3f}' for x in res[p])} (median {np.median(res[p]):.3f}) "
          f"bitwise equal to pub={pubs[0]}: {same}", flush=True)
for p in pubs:
    with q.Context(0) as c:
        c.set_option(q.OPT_SUPER, 1 | 1024)
        c.set_option(q.OPT_SUPER_PUB, p)
        c.load_instance(n, cl)
        c.init_uniform()
        c.evolve(200.0 * K / 10000, K)
        d = c.stats()["tm_diag"]
        print(f"pub={p}: deferred group-k tiles {d[5] / max(d[6], 1):.3f}, wait cycles per deferred "
              f"{d[7] / max(d[5], 1):.0f}", flush=True)
