"""Diagnostic: time the L2-blocked pass (QAA_OPT_SUPER) against the default plan at
n = 30 and compare a sample of amplitudes.  usage: diag_super2.py MODE [K]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

mode = int(sys.argv[1])
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
import os
cl = cnf.load_instance(n)[0] if os.path.exists(cnf.instance_path(n)) else cnf.random_instance(n, int(round(4.5 * n)), 1000 + n)
idx = np.random.default_rng(5).integers(0, 1 << n, 64)
with q.Context(0) as c:
    c.set_option(q.OPT_SUPER, mode)
    c.set_option(q.OPT_PROFILE, 1)
    c.load_instance(n, cl)
    c.init_uniform()
    c.evolve(200.0 * 4 / 10000, 4)
    c.norm2()
    c.reset_stats()
    t0 = time.time()
    c.evolve(200.0 * K / 10000, K)
    nn = c.norm2()
    dt = time.time() - t0
    st = c.stats()
    amps = np.array([c.state(int(i), 1)[0] for i in idx])
    if n == 30:
        np.save(f"gpurun_out/super_amps_{mode}.npy", amps)
    print(f"mode={mode} K={K} wall={dt*1e3:.1f}ms per_step={dt/K*1e3:.2f}ms "
          f"pass_ms={st['pass_kernel_ms']:.1f} per_step_kernel={st['pass_kernel_ms']/K:.2f}ms "
          f"launches={st['pass_launches']} norm-1={nn-1:.3e}", flush=True)
