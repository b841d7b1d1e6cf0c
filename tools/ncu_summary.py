"""Summarise ncu captures of one forward pass into profiles/<round>/.

    python tools/ncu_summary.py --full gpurun_out/prof_full_cfg3.ncu-rep \
        --launches gpurun_out/launches_cfg3.csv --workload cfg3 --out profiles/r01

The capture command (run under gpurun, one GPU) is
    ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
        -k regex:5flame -c 10 -o gpurun_out/prof_full_cfg3 python tools/prof_step.py cfg3 1
Kernels are labelled by their position in the launch sequence of one pass
(paper_2509_22681_b200/csrc/flame.cu Pipe::run), which is fixed for a config.
Writes:
  ncu_kernels_<workload>.csv      per-kernel duration, DRAM bytes, pipe / SOL %
  ncu_dram_per_launch.json        {workload: {role: dram read+write bytes}} (bench traffic)
  launch_share_<workload>.csv     serialised cold-cache launch list with shares
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from pathlib import Path

# launch order of one id-input pass at L = 1 in bf16 mode
# (the gated fusion runs inside the FFN W2 epilogue of the last layer)
ROLES_L1 = ["pda_dedup", "pda_gather", "gemm_kv_hist", "gemm_qkv_cand", "attention_sumi",
            "gemm_oproj_cand", "gemm_ffn_w1", "gemm_ffn_w2", "gemm_expert_w1", "expert_combine"]
# the same with the candidate Q/K/V projection fused into the attention (hb <= 256)
ROLES_L1_FUSED = ["pda_dedup", "pda_gather", "gemm_kv_hist", "attention_fused",
                  "gemm_oproj_cand", "gemm_ffn_w1", "gemm_ffn_w2", "gemm_expert_w1", "expert_combine"]

METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}

OURS = re.compile(r"pda_|gemm_bf16|gemm_f32|sumi_attention|sumi_fused|gated_fusion|expert_|layer_norm_rows|scatter_emb")

UNIT_SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3,
              "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def ncu_raw(rep: Path) -> list[dict]:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    v = float("nan")
                d[k] = v * UNIT_SCALE.get(units[i], 1.0) if k in ("duration_ms", "dram_read", "dram_write") else v
        res.append(d)
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", type=Path, required=True)
    ap.add_argument("--launches", type=Path)
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--out", type=Path, required=True)
    args = ap.parse_args()
    args.out.mkdir(parents=True, exist_ok=True)
    ks = [k for k in ncu_raw(args.full) if OURS.search(k["kernel"])]
    roles = next((r for r in (ROLES_L1, ROLES_L1_FUSED) if len(r) == len(ks)), [f"k{i}" for i in range(len(ks))])
    total = sum(k["duration_ms"] for k in ks)
    with open(args.out / f"ncu_kernels_{args.workload}.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["role", "kernel", "duration_ms", "share", "dram_read_MB", "dram_write_MB", "dram_pct",
                    "sm_pct", "tensor_pct", "issue_pct", "regs", "l2_hit_pct"])
        for role, k in zip(roles, ks):
            w.writerow([role, k["kernel"][:90], f"{k['duration_ms']:.4f}", f"{k['duration_ms'] / total:.3f}",
                        f"{k['dram_read'] / 1e6:.1f}", f"{k['dram_write'] / 1e6:.1f}", f"{k.get('dram_pct', 0):.1f}",
                        f"{k.get('sm_pct', 0):.1f}", f"{k.get('tensor_pct', 0):.1f}", f"{k.get('issue_pct', 0):.1f}",
                        int(k.get("regs", 0)), f"{k.get('l2_hit_pct', 0):.1f}"])
    dram_path = args.out / "ncu_dram_per_launch.json"
    dram = json.loads(dram_path.read_text()) if dram_path.exists() else {}
    dram[args.workload] = {role: k["dram_read"] + k["dram_write"] for role, k in zip(roles, ks)}
    dram_path.write_text(json.dumps(dram, indent=1) + "\n")
    if args.launches and args.launches.exists():
        text = args.launches.read_text()
        text = text[text.index('"ID"'):] if '"ID"' in text else text
        rows = list(csv.DictReader(io.StringIO(text)))
        durs = [(r["Kernel Name"], float(r["Metric Value"].replace(",", "")) * UNIT_SCALE.get(r["Metric Unit"], 1.0))
                for r in rows if r.get("Metric Name") == "gpu__time_duration.sum" and OURS.search(r["Kernel Name"])]
        first = durs[:len(roles)]
        tot = sum(d for _, d in first)
        with open(args.out / f"launch_share_{args.workload}.csv", "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["role", "kernel", "duration_ms_cold_serialised", "share"])
            for role, (name, d) in zip(roles, first):
                w.writerow([role, name[:90], f"{d:.4f}", f"{d / tot:.3f}"])
    print((args.out / f"ncu_kernels_{args.workload}.csv").read_text())


if __name__ == "__main__":
    main()
