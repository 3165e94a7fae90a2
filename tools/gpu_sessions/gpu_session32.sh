set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sweep" 2>&1 | tail -4
python - <<'PY'
import sys, time; sys.path.insert(0,'.')
import numpy as np, torch, paper_1103_1399_b200 as q
from inputs import cnf
for n in (8, 10, 12, 13, 14, 16):
    cl = cnf.load_instance(n)[0] if n in (8,10,12,13,14,16) else None
    with q.Context(0) as c:
        c.load_instance(n, cl)
        Ts = np.array([1, 2, 5, 10, 20, 50, 100, 200, 1, 2, 5, 10, 20, 50, 100, 200], dtype=float)
        Ks = (Ts / 0.05).astype(np.int64)
        c.sweep(Ts, Ks)
        torch.cuda.synchronize(); t0 = time.perf_counter(); p = c.sweep(Ts, Ks); t1 = time.perf_counter()
        print(f"n={n} sweep of {len(Ts)} replicas, {Ks.sum()} steps total: {1e3*(t1-t0):.2f} ms, {Ks.sum()/(t1-t0):.3e} steps/s, longest replica {Ks.max()} steps -> {1e6*(t1-t0)/Ks.max():.2f} us/step; P_succ(T=200) = {p[7]:.4f}")
PY
