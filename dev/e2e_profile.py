"""Host-side profile of the DSO e2e stream (BucketScheduler.score_stream, ids) at
a bench workload: wall time per batch against the device step, and cProfile's
top functions.  Dev measurement only.   python dev/e2e_profile.py [cfg4] [steps]"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
import paper_2509_22681_b200 as fb  # noqa: E402
from paper_2509_22681_b200.orchestrator import BucketScheduler  # noqa: E402
from paper_2509_22681_b200.pda import build_item_table  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
d, dh, nb, L, f, tasks, H, C, R, _ = bench.WORKLOADS[name]
cfg = bench.model_config(name)
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16")
eng.set_table(build_item_table(bench.NUM_ITEMS, d, bench.STORE_SEED), dtype="fp32")
reqs = bench.make_requests(R, H, C, bench.WORKLOAD_SEED, zipf_c=name in bench.ZIPF_C)
n_cand = sum(len(c) for _, c in reqs)
sched = BucketScheduler(eng, with_ids=True)
sched.executors_per_bucket = 3
for _ in sched.score_stream([reqs] * 3, ids=True):
    pass
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in sched.score_stream([reqs] * steps, ids=True):
    pass
wall = time.perf_counter() - t0
print(f"{name}: {steps} batches, {1e3 * wall / steps:.3f} ms per batch, {n_cand * steps / wall / 1e6:.2f} M cand/s")
# host time alone: submit + collect with the device work already done is not separable,
# so profile the same loop and look at where the host spends its time
pr = cProfile.Profile()
pr.enable()
for _ in sched.score_stream([reqs] * steps, ids=True):
    pass
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(22)
