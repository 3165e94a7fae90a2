python - <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np, torch, paper_1103_1399_b200 as q
from inputs import cnf
stream = torch.cuda.Stream(device=0); torch.cuda.set_stream(stream)
for n in (8, 10, 11, 12):
    cl = cnf.load_instance(n)[0] if n in (8,10,12) else cnf.random_instance(n, int(4.5*n), 1000+n)
    with q.Context(0, stream=stream.cuda_stream) as c:
        c.load_instance(n, cl); c.init_uniform(); c.evolve(1.0, 50); c.norm2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(stream); c.evolve(10.0, 1000); b.record(stream); torch.cuda.synchronize()
        print(f"n={n}: {a.elapsed_time(b):.2f} ms / 1000 steps")
PY
