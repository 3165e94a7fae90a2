"""Regenerate inputs/instances/*.cnf (seed = 1000 + n). Calls only inputs/."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs.cnf import INSTANCE_DIR, generate_unique_instance, instance_path, write_dimacs  # noqa: E402


def main(ns):
    os.makedirs(INSTANCE_DIR, exist_ok=True)
    for n in ns:
        t0 = time.time()
        seed = 1000 + n
        clauses, sol, restarts = generate_unique_instance(n, seed)
        text = write_dimacs(n, clauses, comments=[
            f"unique-solution random 3-SAT, n={n}, m={len(clauses)}, ratio={len(clauses)/n:.3f}",
            f"generator: inputs/cnf.py generate_unique_instance(n={n}, seed={seed}); restarts={restarts}",
            f"solution_index={sol}",
        ])
        with open(instance_path(n, seed), "w") as f:
            f.write(text)
        print(f"n={n} m={len(clauses)} ratio={len(clauses)/n:.2f} sol={sol} restarts={restarts} {time.time()-t0:.1f}s", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [8, 12, 16, 20, 24])
