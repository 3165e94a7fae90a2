timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "n30 or super or energy" 2>&1 | tail -2
python - <<'PY'
import sys, time; sys.path.insert(0,'.')
import torch, paper_1103_1399_b200 as q
from inputs import cnf
cl = cnf.load_instance(30)[0]
with q.Context(0) as c:
    for i in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter(); c.load_instance(30, cl); c.init_uniform(); torch.cuda.synchronize()
        print(f"load+init n=30: {1e3*(time.perf_counter()-t0):.1f} ms")
PY
timeout 900 python bench.py > gpurun_out/b35.json 2> gpurun_out/b35.err; python -c "
import json; d=json.load(open('gpurun_out/b35.json')); print(d['value'], d['e2e'], d['clocks'])"
