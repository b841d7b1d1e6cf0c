"""Top SASS lines by warp-stall samples for one kernel of an ncu report.

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
print(rows[0][1][:120])
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
ia, isrc = hdr.index("Address"), hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iall] or 0) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -float(r[iall] or 0))[:top]:
    print(f"{float(r[iall]) / tot * 100:5.1f}% {r[ia]} {r[isrc][:120]}")
if len(sys.argv) > 4:
    # context around addresses: --ctx ADDR[,ADDR]
    addrs = sys.argv[4].split(",")
    pos = {r[ia]: i for i, r in enumerate(data)}
    for a in addrs:
        i = pos.get(a)
        if i is None:
            continue
        print("----", a)
        for r in data[max(0, i - 6):i + 2]:
            print(f"   {float(r[iall] or 0) / tot * 100:5.1f}% {r[ia]} {r[isrc][:120]}")
