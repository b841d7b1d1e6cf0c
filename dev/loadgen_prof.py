"""Host-side profile of the service path at the cfg3 model: one thread calling
handle_batch with B mixed requests (cProfile), then a concurrent loadgen run
reporting the mean coalesced batch size."""
import cProfile
import json
import pstats
import sys
import time

from paper_2509_22681_b200.loadgen import (AblationConfig, KeyDistribution, Scenario, WorkloadSpec,
                                           generate_workload, _drive, scenario_shapes)
from paper_2509_22681_b200.service import DeviceService, ServiceConfig

cfg = ServiceConfig.from_dict(json.load(open("dev/configs/service_cfg3.json")))
svc = DeviceService.from_config(cfg)
spec = WorkloadSpec(Scenario.MIXED, 10.0, 32, KeyDistribution("zipf", 1.0), 0, 400, 100_000)
svc.warm(scenario_shapes(spec))
reqs = list(generate_workload(spec))
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
for k in range(3):
    svc.handle_batch(reqs[:B])
t0 = time.perf_counter()
n = 0
for k in range(0, len(reqs) - B, B):
    svc.handle_batch(reqs[k:k + B])
    n += sum(len(r.candidate_item_ids) for r in reqs[k:k + B])
dt = time.perf_counter() - t0
print(f"single-thread handle_batch({B}): {n / dt / 1e6:.2f} M pairs/s")
pr = cProfile.Profile()
pr.enable()
for k in range(0, len(reqs) - B, B):
    svc.handle_batch(reqs[k:k + B])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
d0 = svc.metrics_snapshot()["dispatches"]
r0 = svc.requests_total
spec2 = WorkloadSpec(Scenario.MIXED, 8.0, 32, KeyDistribution("zipf", 1.0), 1, None, 100_000)
t0 = time.perf_counter()
active = _drive(spec2, svc.handle_request)
m = svc.metrics_snapshot()
print(f"concurrent c32: {(svc.requests_total - r0) / (m['dispatches'] - d0):.1f} requests per dispatch, "
      f"{(svc.requests_total - r0) / active:.0f} req/s")
svc.close()
