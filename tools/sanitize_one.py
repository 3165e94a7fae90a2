"""One evolve for a sanitizer run: python tools/sanitize_one.py n super kernel K [warptile]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402
from oracle import oracle  # noqa: E402

n, sup, kern, K = (int(x) for x in sys.argv[1:5])
wt = int(sys.argv[5]) if len(sys.argv) > 5 else 1
cl = cnf.random_instance(n, int(round(4.3 * n)), 3000 + n)
sched = np.random.default_rng(n).uniform(0, 1, K)
with q.Context(0) as c:
    c.set_option(q.OPT_SUPER, sup)
    c.set_option(q.OPT_KERNEL, kern)
    c.set_option(q.OPT_WARPTILE, wt)
    c.load_instance(n, cl)
    c.init_uniform()
    c.evolve(1.1, K, sched)
    got = c.state()
    st = c.stats()
want = oracle.evolve(n, oracle.energy_table(n, cl), oracle.init_uniform(n), 1.1, K, sched)
print(f"n={n} super={sup} kernel={kern} K={K}: max|d psi| = {np.max(np.abs(got - want)):.2e} "
      f"pass_launches={st['pass_launches']} super_launches={st['super_launches']} tm={st['tm_launches']} "
      f"warp={st['warp_launches']} cluster={st['cluster_launches']}")
