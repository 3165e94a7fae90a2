"""The CPU oracle (oracle/, as it stands) at the bench configuration with 1 thread
and with all host cores: one Trotter step of the n = 30 bench schedule each
(in place, table and state built outside the timing), with the CPU model.
Writes profiles/r02_oracle_threads.json (bench.py reports it as
cpu_baseline.single_thread). python tools/oracle_threads.py [n]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from inputs import cnf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cl, _ = cnf.load_instance(n)
t0 = time.perf_counter()
orc = bench.OracleAtConfig(n, cl)
setup = time.perf_counter() - t0
res = {"n": n, "cpu": bench.cpu_model(), "host_cores": os.cpu_count(), "setup_s_all_cores": setup,
       "how": "oracle_evolve in place, one Trotter step of the bench schedule (T=200, K=1e4) per timing"}
for threads in (os.cpu_count(), 1):
    k = bench.set_omp_threads(threads)
    dt = orc.step()
    res[f"threads_{k}"] = {"step_s": dt, "steps_per_s": 1.0 / dt}
    print(json.dumps(res), flush=True)
res["value"] = res["threads_1"]["steps_per_s"]
res["unit"] = "steps/s"
res["cores"] = 1
out = os.path.join(ROOT, "profiles", "r02_oracle_threads.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
