"""Debug driver for the tensor-memory L2-blocked step: one config per process
(a device trap poisons the CUDA context). Usage: python tools/diag_tm.py n K sup"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

n, K, sup = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cl = cnf.random_instance(n, int(round(4.3 * n)), 1000 + n)
c = q.Context(0)
c.set_option(q.OPT_SUPER, sup)
c.load_instance(n, cl)
c.init_uniform()
sched = np.random.default_rng(n + K).uniform(0, 1, K)
try:
    c.evolve(1.3, K, sched)
    nrm = c.norm2()
    st = c.stats()
    print(f"n={n} K={K} sup={sup}: ok norm2-1={nrm - 1:.3e} super={st['super_launches']} tm={st['tm_launches']}")
except Exception as e:
    print(f"n={n} K={K} sup={sup}: FAIL {e}")
