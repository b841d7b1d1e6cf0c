"""Generate tests/golden/workload.json by running the REFERENCE load generator
(pkg/src/flameserve/bench.py) itself.  Test infrastructure only; run in the
build container, where the read-only reference lives at /root/reference:

    python oracle/gen_golden_workload.py

Pins ``paper_2509_22681_b200.loadgen`` to the reference: the request stream of
a seed (sha256 over user ids, history ids and candidate ids of the first
requests, per scenario / key distribution) and the exact CSV bytes that
reference ``emit_report`` writes for a sample report.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "workload.json"

STREAMS = [  # scenario, kind, exponent, seed, num_items, n
    ("base", "zipf", 1.0, 3, 5000, 20),
    ("long", "uniform", 1.0, 1, 100_000, 6),
    ("mixed", "zipf", 1.2, 7, 100_000, 40),
    ("mixed", "uniform", 1.0, 0, 1000, 40),
]

SAMPLE_REPORT = dict(scenario="mixed", cache=True, mem_opt=False, routing="explicit",
                     throughput_pairs_per_s=1234.5678901234, overall_ms_mean=1.23456789,
                     overall_ms_p99=9.87654321, compute_ms_mean=0.5, compute_ms_p99=2.25,
                     cache_hit_rate=0.7251, network_bytes=987654321, steady_state_allocs=0)


def stream_digest(requests) -> tuple[str, list]:
    h = hashlib.sha256()
    counts = []
    for r in requests:
        h.update(np.int64(r.user_id).tobytes())
        h.update(np.asarray(r.history_item_ids, dtype=np.int64).tobytes())
        h.update(np.asarray(r.candidate_item_ids, dtype=np.int64).tobytes())
        counts.append(len(r.candidate_item_ids))
    return h.hexdigest(), counts


def main() -> None:
    sys.path.insert(0, str(REF))
    from flameserve.bench import (KeyDistribution, RunReport, Scenario, WorkloadSpec, emit_report,
                                  generate_workload)

    out = {"streams": [], "report": {}}
    for scen, kind, expo, seed, items, n in STREAMS:
        spec = WorkloadSpec(scenario=Scenario(scen), duration_s=1.0, concurrency=1,
                            key_distribution=KeyDistribution(kind=kind, exponent=expo), seed=seed,
                            num_requests=n, num_items=items)
        reqs = list(generate_workload(spec))
        digest, counts = stream_digest(reqs)
        out["streams"].append({"scenario": scen, "kind": kind, "exponent": expo, "seed": seed,
                               "num_items": items, "n": n, "sha256": digest, "cand_counts": counts,
                               "first_user_id": reqs[0].user_id,
                               "first_hist_head": reqs[0].history_item_ids[:8].tolist()})
    with tempfile.TemporaryDirectory() as tmp:
        p = Path(tmp) / "r.csv"
        emit_report(RunReport(**SAMPLE_REPORT), p)
        out["report"] = {"fields": SAMPLE_REPORT, "csv": p.read_text()}
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
