"""cfg3 replays back to back for ~1.5 s while NVML samples SM / memory clocks,
power and throttle reasons every 5 ms; prints per-200 ms windows."""
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2509_22681_b200 as fb  # noqa: E402
from paper_2509_22681_b200 import _lib  # noqa: E402
from paper_2509_22681_b200.pda import build_item_table  # noqa: E402

d, dh, nb, L, f, tasks, H, C, R, desc = bench.WORKLOADS["cfg3"]
cfg = bench.model_config("cfg3")
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16", device=0)
eng.set_table(build_item_table(bench.NUM_ITEMS, d, bench.STORE_SEED), dtype="fp32")
reqs = bench.make_requests(R, H, C, bench.WORKLOAD_SEED)
ex = eng.executor(R, H // nb, C, with_ids=True)
ex.stage_ids(reqs)
for _ in range(5):
    ex.run(_lib.INPUT_IDS, graph=True)
torch.cuda.synchronize()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = False


def sampler():
    while not stop:
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.005)


th = threading.Thread(target=sampler)
th.start()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(701)]
t0 = time.perf_counter()
with torch.cuda.stream(ex.stream):
    evs[0].record(ex.stream)
    for k in range(700):
        ex.run(_lib.INPUT_IDS, graph=True)
        evs[k + 1].record(ex.stream)
ex.stream.synchronize()
stop = True
th.join()
ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(700)]
for w in range(0, 700, 70):
    print(f"steps {w:3d}-{w + 69}: {sum(ms[w:w + 70]) / 70:.3f} ms/step")
lim = pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
print("power limit W", lim)
tb = samples[0][0]
for k in range(0, len(samples), max(1, len(samples) // 12)):
    t, sm, mem, pw, rs = samples[k]
    print(f"t={1000 * (t - tb):6.0f} ms sm={sm} mem={mem} power={pw:.0f} W reasons=0x{rs:x}")
