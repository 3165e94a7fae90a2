"""Dynamic instruction mix by SASS opcode (warp-level instructions executed) of the
first kernel in an ncu report. python tools/ncu_opmix.py rep [N]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')]
end = start[1] - 1 if len(start) > 1 else len(lines)
rows = list(csv.reader(io.StringIO("\n".join(lines[start[0]:end]))))
h = rows[0]
iS, iE = h.index("Source"), h.index("Instructions Executed")
by = defaultdict(int)
for r in rows[1:]:
    try:
        n = int(r[iE])
    except (ValueError, IndexError):
        continue
    src = r[iS].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    by[op.split(".")[0]] += n
tot = sum(by.values())
print(f"total {tot:.4g}")
for op, n in sorted(by.items(), key=lambda x: -x[1])[:N]:
    print(f"{op:10s} {n:14d} {100.0 * n / tot:5.1f}%")
