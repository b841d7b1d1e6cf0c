"""Instruction mix (warp-level SASS instructions executed, by opcode) of one
kernel of an ncu report.   python tools/ncu_opmix.py REPORT LAUNCH_INDEX [DIV]"""
import collections
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
st = 1 if rows[0] and rows[0][0] == "Kernel Name" else 0
h = rows[st]
ie, src = h.index("Instructions Executed"), h.index("Source")
c = collections.Counter()
tot = 0.0
for r in rows[st + 1:]:
    if r and r[0] == "Kernel Name":
        break
    try:
        n = float(r[ie])
    except ValueError:
        continue
    op = r[src].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    c[o] += n
    tot += n
print(f"total warp instructions {tot:.0f} ({tot / div:.0f} per unit)")
for o, n in c.most_common(25):
    print(f"{o:12s} {100 * n / tot:5.1f}% {n / div:9.0f}")
