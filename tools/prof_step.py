"""Eager forward passes (id path) of a bench workload, set up exactly as bench.py
sets it up: the 100k-item fp32 item table, bench.make_requests(R, H, C, 2509)
(rank 0's batch), the executor of the timed region.  For ncu captures:

    ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
        -k regex:5flame -c 10 -o gpurun_out/prof_full_cfg3 python tools/prof_step.py cfg3 1

    python tools/prof_step.py [workload] [passes] [profile reps]
"""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2509_22681_b200 as fb  # noqa: E402
from paper_2509_22681_b200 import _lib  # noqa: E402
from paper_2509_22681_b200.pda import build_item_table  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 0
d, dh, nb, L, f, tasks, H, C, R, _ = bench.WORKLOADS[name]
cfg = bench.model_config(name)
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16")
eng.set_table(build_item_table(bench.NUM_ITEMS, d, bench.STORE_SEED), dtype="fp32")
reqs = bench.make_requests(R, H, C, bench.WORKLOAD_SEED)
ex = eng.executor(R, H // nb, C, with_ids=True)
ex.stage_ids(reqs)
for _ in range(passes):
    ex.run(_lib.INPUT_IDS, graph=False)
ex.stream.synchronize()
print("launches per pass", ex.launch_count())
if reps:
    runs = [ex.profile(_lib.INPUT_IDS) for _ in range(reps)]
    tot = 0.0
    for i, rec in enumerate(runs[0]):
        ms = statistics.median(r[i]["ms"] for r in runs)
        tot += ms
        print(f"{rec['name']:>18s} {ms:8.3f} ms  {rec['flops'] / max(ms, 1e-9) / 1e9:8.1f} TF/s  "
              f"{rec['bytes'] / max(ms, 1e-9) / 1e6:8.1f} GB/s")
    print(f"{'sum':>18s} {tot:8.3f} ms")
