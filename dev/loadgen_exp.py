"""Where does the concurrent service path spend its time?  (cfg3 model)"""
import json
import sys
import time

from paper_2509_22681_b200.loadgen import KeyDistribution, Scenario, WorkloadSpec, generate_workload, _drive, scenario_shapes
from paper_2509_22681_b200.service import DeviceService, ServiceConfig

cfg = ServiceConfig.from_dict(json.load(open("dev/configs/service_cfg3.json")))
svc = DeviceService.from_config(cfg)
spec = WorkloadSpec(Scenario.MIXED, 5.0, 32, KeyDistribution("zipf", 1.0), 0, 2000, 100_000)
svc.warm(scenario_shapes(spec))
t0 = time.perf_counter()
reqs = list(generate_workload(spec))
print(f"generate: {len(reqs) / (time.perf_counter() - t0):.0f} req/s")
for r in reqs[:20]:
    svc.handle_request(r)
t0 = time.perf_counter()
for r in reqs[:500]:
    svc.handle_request(r)
print(f"sequential handle_request: {500 / (time.perf_counter() - t0):.0f} req/s")


def run(conc, label, pregenerated=False):
    d0, r0 = svc.dispatches, svc.requests_total
    s = WorkloadSpec(Scenario.MIXED, 5.0, conc, KeyDistribution("zipf", 1.0), 1, None, 100_000)
    if pregenerated:
        import itertools
        it = itertools.cycle(reqs)
        import paper_2509_22681_b200.loadgen as lg
        orig = lg.generate_workload
        lg.generate_workload = lambda spec: it
    active = _drive(s, svc.handle_request)
    if pregenerated:
        lg.generate_workload = orig
    n = svc.requests_total - r0
    print(f"{label}: {n / active:.0f} req/s, {n / max(1, svc.dispatches - d0):.1f} req/dispatch")


run(32, "c32")
run(32, "c32 pregenerated", True)
sys.setswitchinterval(0.0002)
run(32, "c32 switchinterval 0.2ms")
run(32, "c32 pregenerated switchinterval 0.2ms", True)
svc.close()
