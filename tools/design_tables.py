"""Refresh DESIGN.md's results table, step-throughput sentence and GEMM kernel
times from profiles/<round>/ (bench_cfg*.json, ncu_kernels_cfg3.csv)."""
import csv
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
P = ROOT / (sys.argv[1] if len(sys.argv) > 1 else "profiles/r01b")
p = ROOT / "DESIGN.md"
s = p.read_text()
a = s.index("Results (`profiles/r01b/SUMMARY.md`)")
b = s.index("The target is 50 M cand/s on 8 GPUs at cfg3", a)
rows = []
for w in ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]:
    d = json.loads((P / f"bench_{w}.json").read_text())
    c = d.get("cpu_baseline") or {}
    name = f"**{w}**" if w == "cfg3" else (w + " (DSO, Zipf C)" if w == "cfg4" else w)
    v = f"**{d['value'] / 1e6:.2f} M**" if w == "cfg3" else f"{d['value'] / 1e6:.2f} M"
    tf = f"**{d['step_tflops']:.0f}**" if w == "cfg3" else f"{d['step_tflops']:.0f}"
    rows.append(f"| {name} | {v} | {d['e2e']['value'] / 1e6:.2f} M | {d['p99_ms']:.2f} | {tf} | "
                f"{c.get('value', 0) / 1e3:.1f} k |")
d3 = json.loads((P / "bench_cfg3.json").read_text())
new = (f"Results (`profiles/r01b/SUMMARY.md`), 1 × B200, SM clock {d3['clocks']['sm_mhz']} MHz median:\n\n"
       "| workload | cand/s (device) | e2e cand/s | p99 ms | step TFLOP/s | CPU oracle, 16 cores |\n"
       "|---|---|---|---|---|---|\n" + "\n".join(rows) + "\n\n")
s = s[:a] + new + s[b:]
s = re.sub(r"One B200 does\n[0-9.]+ M, and the requests shard with no collective. The p99 request\n"
           r"latency is [0-9.]+ ms against a 20 ms target. End to end, from numpy ids to\n"
           r"numpy scores through `BucketScheduler.score_stream`, cfg3 keeps\n[0-9]+ % of the (?:20-step )?device rate.",
           f"One B200 does\n{d3['value'] / 1e6:.2f} M, and the requests shard with no collective. The p99 request\n"
           f"latency is {d3['p99_ms']:.2f} ms against a 20 ms target. End to end, from numpy ids to\n"
           f"numpy scores through `BucketScheduler.score_stream`, cfg3 keeps\n"
           f"{100 * d3['e2e']['value'] / d3['value']:.0f} % of the 20-step device rate.", s)
s = re.sub(r"The measured step is [0-9.]+ ms, or\n[0-9]+ TFLOP/s\. That is [0-9]+ % of the measured sustained bf16 peak\n"
           r"\(1403 TF/s\) and [0-9]+ % of the burst peak \(1668 TF/s\)\.",
           f"The measured step is {d3['ms_per_step']:.3f} ms, or\n{d3['step_tflops']:.0f} TFLOP/s. That is "
           f"{100 * d3['step_tflops'] / 1403:.0f} % of the measured sustained bf16 peak\n(1403 TF/s) and "
           f"{100 * d3['step_tflops'] / 1668:.0f} % of the burst peak (1668 TF/s).", s)
k = {r["role"]: r for r in csv.DictReader(open(P / "ncu_kernels_cfg3.csv"))}
f = lambda n: f"{float(k[n]['duration_ms']):.3f}"
s = re.sub(r"\| KV [0-9.]+, QKV [0-9.]+, O-proj [0-9.]+, W1 [0-9.]+, W2 [0-9.]+, expert \(tf32\) [0-9.]+ ms;",
           f"| KV {f('gemm_kv_hist')}, QKV {f('gemm_qkv_cand')}, O-proj {f('gemm_oproj_cand')}, W1 {f('gemm_ffn_w1')}, "
           f"W2 {f('gemm_ffn_w2')}, expert (tf32) {f('gemm_expert_w1')} ms;", s)
s = re.sub(r"\| 4·dh per \(query, key\) pair: 138 GFLOP; 1.07 GB read \| [0-9.]+ ms, [0-9]+ % DRAM, [0-9]+ % tensor \|",
           f"| 4·dh per (query, key) pair: 138 GFLOP; 1.07 GB read | {f('attention_sumi')} ms, "
           f"{float(k['attention_sumi']['dram_pct']):.0f} % DRAM, {float(k['attention_sumi']['tensor_pct']):.0f} % tensor |", s)
p.write_text(s)
print("updated")
