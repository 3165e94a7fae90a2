python - <<'PY'
import sys, time; sys.path.insert(0,'.')
import numpy as np, torch, paper_1103_1399_b200 as q
from inputs import cnf
for n in (13, 14, 16, 18, 20, 21):
    cl = cnf.load_instance(n)[0] if n in (13,14,16,20) else cnf.random_instance(n, int(4.5*n), 1000+n)
    with q.Context(0) as c:
        c.load_instance(n, cl); c.init_uniform(); c.evolve(1.0, 50); c.norm2()
        c.set_option(q.OPT_PROFILE, 1); c.reset_stats()
        torch.cuda.synchronize(); t0=time.perf_counter(); c.evolve(10.0, 1000); c.norm2(); t1=time.perf_counter()
        st=c.stats()
        print(f"n={n}: wall {1e3*(t1-t0)/1000:.1f} us/step, kernel sum {1e3*st['pass_kernel_ms']/st['pass_launches']:.1f} us/launch, launches {st['pass_launches']}, groups {st['groups']}")
PY
