"""One eager forward pass (ids path) of a bench workload, for ncu captures."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import bench
import paper_2509_22681_b200 as fb
from paper_2509_22681_b200 import _lib
from paper_2509_22681_b200.pda import build_item_table

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
d, dh, nb, L, f, tasks, H, C, R, _ = bench.WORKLOADS[name]
cfg = bench.model_config(name)
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16")
eng.set_table(build_item_table(20000, d), dtype="bf16")
reqs = bench.make_requests(R, H, C, 7)
reqs = [(h % 20000, c % 20000) for h, c in reqs]
ex = eng.executor(R, H // nb, C, with_ids=True)
ex.stage_ids(reqs)
for _ in range(passes):
    ex.run(_lib.INPUT_IDS, graph=False)
ex.stream.synchronize()
print("launches per pass", ex.launch_count())
import statistics
try:
    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    hnd = None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 7
runs, clocks = [], []
for _ in range(reps):
    runs.append(ex.profile(_lib.INPUT_IDS))
    if hnd is not None:
        clocks.append(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM))
tot = 0.0
for i, rec in enumerate(runs[0]):
    ms = statistics.median(r[i]["ms"] for r in runs)
    tot += ms
    print(f"{rec['name']:>18s} {ms:8.3f} ms  {rec['flops']/max(ms,1e-9)/1e9:8.1f} TF/s  {rec['bytes']/max(ms,1e-9)/1e6:8.1f} GB/s")
print(f"{'sum':>18s} {tot:8.3f} ms   sm clocks {clocks}")
