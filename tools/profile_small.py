"""One evolve of the quad-warp-tile launch (default, n = 16, K = 200), of the
single-warp-tile launch (n = 16) and of the cluster-resident launch (n = 14),
for ncu (tools/gpu_profile_round.sh)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

for n, wt in ((16, 1), (16, 2), (14, 0)):
    with q.Context(0) as c:
        c.set_option(q.OPT_WARPTILE, wt)
        c.load_instance(n, cnf.load_instance(n)[0])
        c.init_uniform()
        c.evolve(4.0, 200)
        st = c.stats()
        print(n, "warp", st["warp_launches"], "cluster", st["cluster_launches"], "norm2", c.norm2())
