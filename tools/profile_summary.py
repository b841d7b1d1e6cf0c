"""Write profiles/<round>/SUMMARY.md from the measurement files of one
dev/gpu_measure.sh call (bench_cfg*.json, reference_arm_cfg3.json,
ncu_kernels_cfg3.csv, parity.json).   python tools/profile_summary.py profiles/r01b"""
import csv
import json
import sys
from pathlib import Path

P = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01b")
desc = {"cfg1": "cfg1 d=64, 2 blocks, H=256, C=64", "cfg2": "cfg2 d=256, 4 blocks, H=1024, C=256",
        "cfg3": "**cfg3** d=512, 8 blocks, H=2048, C=512", "cfg4": "cfg4 DSO, Zipf C 16–2048, H=1024",
        "cfg5": "cfg5 d=768, 12 blocks, H=8184, C=1024"}
rows = []
for w in ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]:
    d = json.loads((P / f"bench_{w}.json").read_text())
    r, c = d["roofline"], d.get("cpu_baseline") or {}
    rows.append(f"| {desc[w]} | {d['value'] / 1e6:.2f} M | {d['ms_per_step']:.3f} | {d['e2e']['value'] / 1e6:.2f} M | "
                f"{d['p99_ms']:.2f} | {d['step_tflops']:.0f} | {r['kernel']} {r['frac']:.2f} | "
                f"{c.get('value', 0) / 1e3:.1f} k |")
k = list(csv.DictReader(open(P / "ncu_kernels_cfg3.csv")))
krows = [f"| {x['role']} | {float(x['duration_ms']):.3f} | {100 * float(x['share']):.0f} % | "
         f"{float(x['dram_read_MB']):.0f} / {float(x['dram_write_MB']):.0f} | {float(x['dram_pct']):.0f} | "
         f"{float(x['tensor_pct']):.0f} | {float(x['issue_pct']):.0f} |" for x in k]
att_mb = next(float(x["dram_read_MB"]) for x in k if x["role"] == "attention_sumi")
par = json.loads((P / "parity.json").read_text())
ref = json.loads((P / "reference_arm_cfg3.json").read_text())
d3 = json.loads((P / "bench_cfg3.json").read_text())
s = f"""# Round 1 measurements — 1 × B200

The tables come from one `gpurun` call of `dev/gpu_measure.sh` (the burst-vs-sustained
section at the end from a second call on one box). The call ran:
* the GPU parity tests (all pass);
* `smoke()`;
* `tools/parity_report.py`;
* `bench.py` on every workload;
* the reference (CPU) arm;
* an ncu launch list and one `ncu --set full` capture of a cfg3 pass.

During the cfg3 timed region the SM clock median was {d3['clocks']['sm_mhz']} MHz, with throttle
reasons {d3['clocks']['reasons']}.

## Bench lines (`bench_cfg*.json`)

| workload | cand/s (device) | ms/step | e2e cand/s | p99 ms | step TFLOP/s | roofline kernel, frac of sustained peak | CPU oracle (16 cores) |
|---|---|---|---|---|---|---|---|
""" + "\n".join(rows) + f"""

* `e2e` goes through the public streaming API, `BucketScheduler.score_stream`:
  * numpy ids are staged into pinned buffers, copied H2D, run as a graph replay per
    group, and copied D2H back to numpy;
  * the next batch is staged while the previous one runs.

  At cfg3 it reaches {d3['e2e']['value'] / d3['value'] * 100:.0f} % of the device-timed rate.
* The 8-GPU target is 50 M cand/s at cfg3, i.e. 6.25 M per GPU. Requests shard with no
  collective.
* The reference arm (`reference_arm_cfg3.json`) is the numpy fp64 port of the reference
  on the same host cores: {ref['value'] / 1e3:.1f} k cand/s.
* Box-to-box variation of the device rate is about ±3 %.

## Kernels of one cfg3 pass (`ncu_kernels_cfg3.csv`, `--set full`, cold, serialised)

| kernel | ms | share | DRAM R/W MB | DRAM % | tensor % | issue % |
|---|---|---|---|---|---|---|
""" + "\n".join(krows) + f"""

How to read the table:
* The gated fusion over the Climber blocks runs inside the FFN W2 epilogue. W2 writes
  64 MB, the fp32 fused rows (the tf32 expert operand), instead of 537 MB of fp32
  block outputs.
* The attention kernel's algorithmic read is 1.07 GB: the candidates' Q, K_self and
  V_self, plus each request-block's history K/V. The history K/V is read once per
  (request, block, head), never per candidate. In this cold, serialised capture it
  reads {att_mb / 1000:.2f} GB; the excess is tiles its L2 prefetch of the
  next-but-one job fetched and lost before use.
* The K = 512 projection GEMMs run as CTA pairs, which halves each CTA's W-tile L2
  traffic.
* PDA: the radix-sort dedup and the run-piece gather together take about 0.1 ms.

## Parity (`parity.json`, max |err| against the reference's own golden outputs)

""" + f"fp32 verification mode: at most {max(p['maxabs_fp32'] for p in par):.1e} (tolerance 1e-4).\n" + \
    f"bf16: at most {max(p['maxabs_bf16'] for p in par):.1e} (tolerance 2e-2).\n"
l2 = P / "bench_cfg3_l2.json"
if l2.exists():
    d = json.loads(l2.read_text())
    s += f"""
## Sensitivity row: cfg3 with 2 layers per block (`bench_cfg3_l2.json`)

SURVEY §8 asks for `L = 2` beside the L = 1 reading. Layer 1 of each block is a
non-final layer: Q/K/V on all rows, causal history attention, O-proj and FFN on
all rows, with an fp32 residual stream. This row measures that path at full size:

* {d['value'] / 1e6:.2f} M cand/s device ({d['ms_per_step']:.2f} ms/step);
* {d['e2e']['value'] / 1e6:.2f} M e2e;
* {d['step_tflops']:.0f} TFLOP/s algorithmic.
"""
su = P / "bench_cfg3_sustained.json"
bu = P / "bench_cfg3_burst_samebox.json"
if su.exists() and bu.exists():
    d, b = json.loads(su.read_text()), json.loads(bu.read_text())
    s += f"""
## Burst vs sustained (`bench_cfg3_burst_samebox.json`, `bench_cfg3_sustained.json`, `sustained_probe.txt`)

The bench lines above time 20 back-to-back steps (~45 ms). On one box, in one call:

* 20 steps: {b['value'] / 1e6:.2f} M cand/s ({b['ms_per_step']:.3f} ms/step), SM clock {b['clocks']['sm_mhz']:.0f} MHz, throttle reasons {b['clocks']['reasons']};
* 150 steps: {d['value'] / 1e6:.2f} M cand/s ({d['ms_per_step']:.3f} ms/step), SM clock median {d['clocks']['sm_mhz']:.0f} MHz
  (min {d['clocks']['sm_min_mhz']}), throttle reasons {d['clocks']['reasons']}.

`dev/sustained_probe.py` samples NVML every 5 ms over 700 replays: the software
power cap (reason 0x4) engages within ~150 ms of full load and pulls the SM clock
from 1965 MHz to 1.0–1.5 GHz, where it stays; NVML's averaged board power
settles at ~980 W against the 1000 W limit.
So sustained throughput on this pass is power-bound; energy per candidate (bytes
moved, instructions issued) is what moves it. The e2e figures are timed over
~0.3 s of device work and show the sustained rate.
"""
(P / "SUMMARY.md").write_text(s)
print(s[:1500])
