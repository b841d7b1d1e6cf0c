"""cProfile of the cfg4 e2e loop (score_stream over 256-request batches)."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2509_22681_b200 as fb  # noqa: E402
from paper_2509_22681_b200.orchestrator import BucketScheduler  # noqa: E402
from paper_2509_22681_b200.pda import build_item_table  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
d, dh, nb, L, f, tasks, H, C, R, desc = bench.WORKLOADS[name]
cfg = bench.model_config(name)
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16", device=0)
eng.set_table(build_item_table(bench.NUM_ITEMS, d, bench.STORE_SEED), dtype="fp32")
reqs = bench.make_requests(R, H, C, bench.WORKLOAD_SEED, zipf_c=(name == "cfg4"))
n = sum(len(c) for _, c in reqs)
sched = BucketScheduler(eng, with_ids=True, executors_per_bucket=int(sys.argv[2]) if len(sys.argv) > 2 else 2)
print("groups", len(sched.plan([(len(h), len(c)) for h, c in reqs])))
for _ in sched.score_stream([reqs] * 3, ids=True):
    pass
for k in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in sched.score_stream([reqs] * 10, ids=True):
        pass
    print(f"e2e {n * 10 / (time.perf_counter() - t0) / 1e6:.2f} M/s")
pr = cProfile.Profile()
pr.enable()
for _ in sched.score_stream([reqs] * 10, ids=True):
    pass
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
