"""Diagnostic: run the experimental L2-blocked pass with a given option value."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

n, sup, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cl = cnf.load_instance(n)[0] if n in (24, 30) else cnf.random_instance(n, int(4.3 * n), 1000 + n)
with q.Context(0) as c:
    c.set_option(q.OPT_SUPER, sup)
    c.load_instance(n, cl)
    c.init_uniform()
    t0 = time.time()
    c.evolve(0.5, K)
    print("norm", c.norm2(), "time", time.time() - t0, c.stats()["pass_launches"], flush=True)
