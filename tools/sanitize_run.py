"""A short run of every hot-path kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): resident kernel (n = 10), register pass
(n = 14), TMA passes (n = 18), the L2-blocked step forced at n = 22 (shared-memory
-- default split-phase synchronisation and the round-1 barriers -- and
tensor-memory variants), the warp-tile whole-evolve launch (n = 16), the
cluster-resident launch (n = 14), the energy-table / compaction / reduction
kernels, and the n = 12 and n = 14 sweeps. Prints one line per case with the max deviation from the
oracle. usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py [quick]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402
from oracle import oracle  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
# (n, QAA_OPT_SUPER, QAA_OPT_KERNEL, K, QAA_OPT_WARPTILE)
cases = [(10, 0, 2, 3, 1), (14, 0, 0, 2, 1), (18, 0, 1, 2, 1), (22, 17, 2, 2, 1), (22, 17 | 32768, 2, 2, 1),
         (22, 17 | 64, 2, 2, 1), (16, 1, 2, 3, 1), (14, 1, 2, 3, 0)]
if quick:
    cases = [(10, 0, 2, 2, 1), (14, 0, 0, 1, 1), (22, 17, 2, 1, 1), (16, 1, 2, 2, 1), (14, 1, 2, 2, 0)]
for n, sup, kern, K, wt in cases:
    cl = cnf.random_instance(n, int(round(4.3 * n)), 3000 + n)
    E = oracle.energy_table(n, cl)
    sched = np.random.default_rng(n).uniform(0, 1, K)
    with q.Context(0) as c:
        c.set_option(q.OPT_SUPER, sup)
        c.set_option(q.OPT_KERNEL, kern)
        c.set_option(q.OPT_WARPTILE, wt)
        c.load_instance(n, cl)
        c.init_uniform()
        c.evolve(1.1, K, sched)
        got = c.state()
        obs = (c.norm2(), c.success_prob(), c.energy(0.5))
        st = c.stats()
    want = oracle.evolve(n, E, oracle.init_uniform(n), 1.1, K, sched)
    print(f"n={n} super={sup} kernel={kern} K={K}: max|d psi| = {np.max(np.abs(got - want)):.2e} "
          f"super_launches={st['super_launches']} tm={st['tm_launches']} warp={st['warp_launches']} "
          f"cluster={st['cluster_launches']} norm2={obs[0]:.15f}", flush=True)
if not quick:
    n = 12
    cl = cnf.load_instance(n)[0]
    with q.Context(0) as c:
        c.load_instance(n, cl)
        out = c.sweep([1.0, 2.0], [10, 20])
    print(f"sweep n=12: {out}", flush=True)
    n = 14
    cl = cnf.random_instance(n, int(round(4.3 * n)), 3014)
    with q.Context(0) as c:
        c.load_instance(n, cl)
        out = c.sweep([1.0, 2.0], [10, 20])
        st = c.stats()
    print(f"sweep n=14 (cluster launches {st['cluster_launches']}): {out}", flush=True)
