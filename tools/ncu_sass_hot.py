"""Top SASS instructions by warp-stall samples from an ncu report (first kernel),
with a per-opcode summary. python tools/ncu_sass_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# the report may hold several kernels; take the first table
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')]
end = start[1] - 1 if len(start) > 1 else len(lines)
rows = list(csv.reader(io.StringIO("\n".join(lines[start[0]:end]))))
h = rows[0]
iS, iA, iSmp = h.index("Source"), h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[1:]:
    try:
        data.append((int(r[iSmp]), r[iA], r[iS].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print(f"total samples {tot}")
byop = defaultdict(int)
for s, a, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    byop[op.split(".")[0]] += s
for op, s in sorted(byop.items(), key=lambda x: -x[1])[:25]:
    print(f"{op:12s} {s:8d} {100.0 * s / tot:5.1f}%")
print()
for s, a, src in sorted(data, key=lambda x: -x[0])[:N]:
    print(f"{s:7d} {100.0 * s / tot:5.1f}% {a[-5:]} {src[:110]}")
