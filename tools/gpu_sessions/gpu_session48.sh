python - <<'PY'
import sys, time; sys.path.insert(0,'.')
import numpy as np, torch, paper_1103_1399_b200 as q
from inputs import cnf
stream = torch.cuda.Stream(device=0); torch.cuda.set_stream(stream)
for n in (19, 22, 23, 24, 25, 26, 27):
    cl = cnf.load_instance(n)[0] if n in (13,14,16,20) else cnf.random_instance(n, int(4.5*n), 1000+n)
    row = []
    for kern in (1, 0):
        with q.Context(0, stream=stream.cuda_stream) as c:
            c.set_option(q.OPT_KERNEL, kern)
            c.load_instance(n, cl); c.init_uniform(); c.evolve(1.0, 50); c.norm2()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record(stream); c.evolve(10.0, 200); b.record(stream); torch.cuda.synchronize()
            row.append(a.elapsed_time(b))
    print(f"n={n}: tma {row[0]:.2f} ms / 200 steps, register {row[1]:.2f} ms")
PY
