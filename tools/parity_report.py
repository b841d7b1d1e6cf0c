"""Max-abs error of the device path vs the reference's golden outputs
(tests/golden/forward_*.npz, produced by the reference itself), both precisions.

    python tools/parity_report.py [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import FORWARD_CASES, golden_forward  # noqa: E402

import paper_2509_22681_b200 as fb  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", type=Path)
    args = ap.parse_args()
    rows = []
    for name in FORWARD_CASES:
        cfg, params, hist, cand, blob = golden_forward(name)
        row = {"case": name, "d": cfg.hidden_dim, "blocks": cfg.num_blocks, "layers": cfg.layers_per_block,
               "H": int(blob["H"]), "C": int(blob["C"])}
        for prec in ("fp32", "bf16"):
            out = fb.model_forward(hist, cand, params, cfg, precision=prec)
            row[f"maxabs_{prec}"] = float(np.abs(out - blob["scores"]).max())
        rows.append(row)
        print(f"{name:14s} d={row['d']:4d} Nb={row['blocks']:2d} L={row['layers']} H={row['H']:5d} C={row['C']:5d}  "
              f"fp32 {row['maxabs_fp32']:.2e} (tol 1e-4)   bf16 {row['maxabs_bf16']:.2e} (tol 2e-2)", flush=True)
    if args.json:
        args.json.write_text(json.dumps(rows, indent=1) + "\n")


if __name__ == "__main__":
    main()
