"""Does the eager per-launch profile depend on what ran just before it?
Profile passes (median of 5) cold, after 40 graph replays, after 200 replays,
and per-kernel times from the graph itself (a profiled capture)."""
import statistics
import sys

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
import paper_2509_22681_b200 as fb  # noqa: E402
from paper_2509_22681_b200 import _lib  # noqa: E402
from paper_2509_22681_b200.pda import build_item_table  # noqa: E402

d, dh, nb, L, f, tasks, H, C, R, _ = bench.WORKLOADS["cfg3"]
cfg = bench.model_config("cfg3")
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16")
eng.set_table(build_item_table(bench.NUM_ITEMS, d, bench.STORE_SEED), dtype="fp32")
ex = eng.executor(R, H // nb, C, with_ids=True)
ex.stage_ids(bench.make_requests(R, H, C, bench.WORKLOAD_SEED))
ex.run(_lib.INPUT_IDS, graph=True)
ex.stream.synchronize()


def prof(tag):
    runs = [ex.profile(_lib.INPUT_IDS) for _ in range(5)]
    out = {rec["name"]: statistics.median(r[i]["ms"] for r in runs) for i, rec in enumerate(runs[0])}
    print(tag, " ".join(f"{k}={v:.3f}" for k, v in out.items()), f"sum={sum(out.values()):.3f}", flush=True)


prof("cold")
for n in (40, 200):
    for _ in range(n):
        ex.run(_lib.INPUT_IDS, graph=True)
    prof(f"after{n}")
    ex.stream.synchronize()
import torch  # noqa: E402
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(ex.stream)
for _ in range(20):
    ex.run(_lib.INPUT_IDS, graph=True)
ev[1].record(ex.stream)
ex.stream.synchronize()
print("graph step ms", ev[0].elapsed_time(ev[1]) / 20)
prof("end")
