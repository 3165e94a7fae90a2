set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super_pass_parity" 2>&1 | tail -2
for m in 1 17 1 17; do timeout 120 python tools/diag_super2.py $m 20 30; done
python - <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np, paper_1103_1399_b200 as q
from inputs import cnf
from oracle import oracle
n=24; cl=cnf.load_instance(n)[0]
for m in (17,):
    with q.Context(0) as c:
        c.set_option(q.OPT_SUPER, m); c.load_instance(n, cl); c.init_uniform(); c.evolve(1.3, 5); got=c.state()
    want=oracle.evolve(n, oracle.energy_table(n, cl), oracle.init_uniform(n), 1.3, 5)
    print("NG3 n=24 max|d|", np.abs(got-want).max())
PY
