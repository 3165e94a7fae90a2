"""A/B timing of the L2-blocked step variants at one size, interleaved in one
process (same box, same clocks): per-launch kernel ms from the library's
event timing. usage: ab_super.py n K sup1 [sup2 ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

n, K = int(sys.argv[1]), int(sys.argv[2])
sups = [int(x) for x in sys.argv[3:]]
cl = cnf.load_instance(n)[0] if os.path.exists(cnf.instance_path(n)) else cnf.random_instance(n, int(round(4.5 * n)), 1000 + n)
res = {s: [] for s in sups}
GRID = int(os.environ.get("GRID", "0"))
with q.Context(0) as c:
    c.set_option(q.OPT_SUPER_GRID, GRID)
    c.set_option(q.OPT_SUPER_SPLIT, int(os.environ.get("SPLIT", "0")))
    c.load_instance(n, cl)
    c.init_uniform()
    for rep in range(3):
        for s in sups:
            c.set_option(q.OPT_SUPER, s)
            c.evolve(200.0 * 2 / 10000, 2)  # warm
            c.reset_stats()
            c.set_option(q.OPT_PROFILE, 1)
            c.evolve(200.0 * K / 10000, K)
            st = c.stats()
            c.set_option(q.OPT_PROFILE, 0)
            res[s].append(st["super_kernel_ms"] / max(st["super_kernels_timed"], 1))
    nrm = c.norm2()
for s in sups:
    print(f"n={n} grid={GRID} split={os.environ.get('SPLIT', '0')} sup={s}: super launch ms {' '.join(f'{x:.3f}' for x in res[s])}  (best {min(res[s]):.3f})")
print(f"norm2-1 = {nrm - 1:.3e}")
# diagnostics (bit 10 of the option): where the warps' time goes
if any(s & 1024 for s in sups):
    with q.Context(0) as c:
        c.load_instance(n, cl)
        c.init_uniform()
        s = [x for x in sups if x & 1024][0]
        c.set_option(q.OPT_SUPER, s)
        c.evolve(200.0 * K / 10000, K)
        d = c.stats()["tm_diag"]
        nw = 148 * 16
        print(f"diag per warp per launch (K={K}): items {d[1] / nw / K:.0f}, deferred {d[2] / nw / K:.1f}, "
              f"landed-wait cyc {d[0] / nw / K:.3g}, deferred-wait cyc {d[3] / nw / K:.3g}, "
              f"g0 prog cyc {d[4] / nw / K:.3g}, gk prog cyc {d[5] / nw / K:.3g}, "
              f"done-spin cyc (group leader) {d[6] / (148 * 2) / K:.3g}, issued early at arrival {d[7] / nw / K:.1f}")
# producer-warp diagnostics (bit 14 + bit 10)
if any((s & 16384) and (s & 1024) for s in sups):
    with q.Context(0) as c:
        c.load_instance(n, cl)
        c.init_uniform()
        s = [x for x in sups if (x & 16384) and (x & 1024)][0]
        c.set_option(q.OPT_SUPER, s)
        c.evolve(200.0 * K / 10000, K)
        d = c.stats()["tm_diag"]
        nw = 148 * 16
        print(f"pw diag per launch (K={K}): consumer items/warp {d[1] / nw / K:.0f}, consumer full-wait cyc/warp "
              f"{d[0] / nw / K:.3g}, producer chunk-wait cyc/CTA {d[2] / 148 / K:.3g}, B-not-ready decisions/CTA "
              f"{d[3] / 148 / K:.1f}, producer empty-wait cyc/CTA {d[4] / 148 / K:.3g}")
