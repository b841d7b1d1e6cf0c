"""cProfile of the cfg4 e2e host path (BucketScheduler.score_stream)."""
import cProfile, pstats, sys
sys.path.insert(0, "/root/repo")
import torch, bench, paper_2509_22681_b200 as fb
from paper_2509_22681_b200.orchestrator import BucketScheduler
from paper_2509_22681_b200.pda import build_item_table
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
d, dh, nb, L, f, tasks, H, C, R, _ = bench.WORKLOADS[name]
cfg = bench.model_config(name)
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16")
eng.set_table(build_item_table(20000, d), dtype="fp32")
reqs = [(h % 20000, c % 20000) for h, c in bench.make_requests(R, H, C, 7, zipf_c=name in bench.ZIPF_C)]
sched = BucketScheduler(eng, with_ids=True, executors_per_bucket=3)
for _ in sched.score_stream([reqs] * 2, ids=True):
    pass
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in sched.score_stream([reqs] * 5, ids=True):
    pass
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
