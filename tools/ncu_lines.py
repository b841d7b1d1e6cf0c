"""Top CUDA source lines by warp-stall samples for one kernel of an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep LAUNCH_INDEX [TOP]
"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
cur, hdr, si, agg, tot, fn = None, None, None, {}, 0.0, ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r[0]:
        continue
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    key = (cur, int(r[0]), r[1].strip()[:90])
    agg[key] = agg.get(key, 0.0) + v
    tot += v
print(fn[:100])
for (f, ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{ln} {src}")
