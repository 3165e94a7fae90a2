"""Per-instruction stall reasons from an ncu report (first kernel of the source page):
top instructions for one stall column. python tools/ncu_stall_by_insn.py rep stall_long_sb [N]"""
import csv
import io
import subprocess
import sys

path, col = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')]
end = start[1] - 1 if len(start) > 1 else len(lines)
rows = list(csv.reader(io.StringIO("\n".join(lines[start[0]:end]))))
h = rows[0]
ic, iS, iA = h.index(col), h.index("Source"), h.index("Address")
data = []
for r in rows[1:]:
    try:
        data.append((int(r[ic]), r[iA][-5:], r[iS].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print(f"{col}: total {tot}")
for s, a, src in sorted(data, reverse=True)[:N]:
    print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}% {a} {src[:100]}")
