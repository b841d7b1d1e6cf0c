"""Graph-replay step time of a bench workload (set up as bench.py) plus the
per-kernel eager profile: one line per process, for interleaved env A/B runs
(dev/step_ab.sh).   python dev/step_time.py [workload] [tag]"""
import statistics
import sys

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
import paper_2509_22681_b200 as fb  # noqa: E402
from paper_2509_22681_b200 import _lib  # noqa: E402
from paper_2509_22681_b200.pda import build_item_table  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
tag = sys.argv[2] if len(sys.argv) > 2 else ""
d, dh, nb, L, f, tasks, H, C, R, _ = bench.WORKLOADS[name]
cfg = bench.model_config(name)
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16")
eng.set_table(build_item_table(bench.NUM_ITEMS, d, bench.STORE_SEED), dtype="fp32")
ex = eng.executor(R, H // nb, C, with_ids=True)
ex.stage_ids(bench.make_requests(R, H, C, bench.WORKLOAD_SEED))
for _ in range(10):
    ex.run(_lib.INPUT_IDS, graph=True)
ex.stream.synchronize()
runs = [ex.profile(_lib.INPUT_IDS) for _ in range(5)]
prof = {rec["name"]: statistics.median(r[i]["ms"] for r in runs) for i, rec in enumerate(runs[0])}
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(3):
    ev[0].record(ex.stream)
    for _ in range(20):
        ex.run(_lib.INPUT_IDS, graph=True)
    ev[1].record(ex.stream)
    ex.stream.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) / 20)
print(f"{tag:>12s} step={statistics.median(ts):.4f} ms  " + " ".join(f"{k}={v:.3f}" for k, v in prof.items()),
      flush=True)
