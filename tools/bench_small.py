"""Per-step device time of small states (configs[0]/[1] sizes and the persistent
range 13..21): one evolve of K steps timed with CUDA events, persistent on and
off. python tools/bench_small.py [K]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1103_1399_b200 as q  # noqa: E402
from inputs import cnf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
rows = []
for n in (8, 12, 13, 14, 16, 18, 20, 21, 22):
    cl = cnf.load_instance(n)[0] if os.path.exists(cnf.instance_path(n)) else cnf.random_instance(n, int(round(4.3 * n)), 1000 + n)
    for persist in (1, 0):
        with q.Context(0, stream=stream.cuda_stream) as c:
            c.set_option(q.OPT_PERSIST, persist)
            c.load_instance(n, cl)
            c.init_uniform()
            c.evolve(0.02 * 50, 50)  # warm
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c.evolve(0.02 * K, K)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            st = c.stats()
        rows.append({"n": n, "persist": persist, "K": K, "us_per_step": ms * 1e3 / K, "steps_per_s": K / (ms / 1e3),
                     "persist_launches": st["persist_launches"], "pass_launches": st["pass_launches"]})
        print(json.dumps(rows[-1]), flush=True)
