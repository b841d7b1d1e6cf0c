"""Rewrite the table in profiles/<round>/loadgen/README.md from its CSV reports."""
import csv
import sys
from pathlib import Path

P = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01b/loadgen")
rows = []
for f in sorted(P.glob("*.csv")):
    r = next(csv.DictReader(open(f)))
    rows.append(f"| {f.stem} | {float(r['throughput_pairs_per_s']) / 1e6:.2f} M | {float(r['overall_ms_mean']):.2f} / "
                f"{float(r['overall_ms_p99']):.2f} | {float(r['compute_ms_mean']):.2f} / {float(r['compute_ms_p99']):.2f} | "
                f"{float(r['cache_hit_rate']):.2f} | {r['steady_state_allocs']} |")
readme = P / "README.md"
s = readme.read_text()
head = "|---|---|---|---|---|---|\n"
a = s.index(head) + len(head)
b = s.index("\n\n", a)
readme.write_text(s[:a] + "\n".join(rows) + s[b:])
print("\n".join(rows))
