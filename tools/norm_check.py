"""Norm drift of K steps of the n-qubit schedule with one QAA_OPT_SUPER value.
usage: norm_check.py n K sup"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

n, K, sup = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cl = cnf.load_instance(n)[0] if os.path.exists(cnf.instance_path(n)) else cnf.random_instance(n, int(round(4.5 * n)), 1000 + n)
with q.Context(0) as c:
    c.set_option(q.OPT_SUPER, sup)
    c.load_instance(n, cl)
    c.init_uniform()
    for i in range(3):
        c.evolve(200.0 * K / 10000, K)
        st = c.stats()
        print(f"n={n} sup={sup} after {K*(i+1)} steps: norm2-1 = {c.norm2() - 1:.3e} p_succ={c.success_prob():.12e} "
              f"super={st['super_launches']} tm={st['tm_launches']}", flush=True)
