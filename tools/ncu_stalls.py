"""Top SASS lines by warp-stall samples for one kernel of an ncu report, with
the dominant stall reasons of each line.

    python tools/ncu_stalls.py REPORT.ncu-rep LAUNCH_INDEX [TOP]
"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = 0
if rows[0] and rows[0][0] == "Kernel Name":
    print(rows[0][1][:120])
    start = 1
hdr = rows[start]
data = []
for r in rows[start + 1:]:
    if r and r[0] == "Kernel Name":
        break
    data.append(r)
col = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(num(r[col]) for r in data)
print(f"total samples {tot}")
agg = {}
for r in data:
    for i in stall_cols:
        agg[hdr[i]] = agg.get(hdr[i], 0.0) + num(r[i])
print("by reason:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
data.sort(key=lambda r: -num(r[col]))
for r in data[:top]:
    reasons = sorted(((num(r[i]), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
    rs = " ".join(f"{n}:{int(v)}" for v, n in reasons if v > 0)
    print(f"{100 * num(r[col]) / tot:5.1f}% {r[0][-5:]} {r[1][:60]:60s} {rs}")
