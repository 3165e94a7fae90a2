"""Diagnostic: how many group-k tiles of the L2-blocked step are issued before
their chunk is complete ("deferred", loaded late by their own group), and the
cycles their groups spend waiting (QAA_OPT_SUPER bit 10 -> tm_flags 8).
usage: diag_defer.py [K] [extra super bits]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
extra = [int(x) for x in sys.argv[2:]] or [0]
n = 30
cl = cnf.load_instance(n)[0]
for ex in extra:
    for diag in (0, 1024):
        with q.Context(0) as c:
            c.set_option(q.OPT_SUPER, 1 | diag | ex)
            c.set_option(q.OPT_PROFILE, 1)
            c.load_instance(n, cl)
            c.init_uniform()
            c.evolve(200.0 * 3 / 10000, 3)
            c.norm2()
            c.reset_stats()
            c.evolve(200.0 * K / 10000, K)
            c.norm2()
            st = c.stats()
            d = st["tm_diag"]
            ms = st["pass_kernel_ms"] / max(st["pass_launches"], 1)
            print(f"super={1 | diag | ex} ms/launch={ms:.3f} launches={st['pass_launches']} "
                  f"gk_tiles={d[6]} deferred={d[5]} ({d[5] / max(d[6], 1):.3f}) "
                  f"wait_cycles_per_deferred={d[7] / max(d[5], 1):.0f}", flush=True)
