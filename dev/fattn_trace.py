"""Per-event timeline of CTA 0 of the fused projection + attention kernel
(needs a FLAME_DEBUG_TRACE build: dev/build_variant.sh trace -DFLAME_DEBUG_TRACE,
run with FLAME_B200_LIB=dev/var_trace.so).  Slots: 0/1 = warpgroups, 2 = MMA
issuer, 3 = A/W ring producer."""
import ctypes
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
import paper_2509_22681_b200 as fb  # noqa: E402
from paper_2509_22681_b200 import _lib  # noqa: E402
from paper_2509_22681_b200.pda import build_item_table  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
d, dh, nb, L, f, tasks, H, C, R, _ = bench.WORKLOADS[name]
cfg = bench.model_config(name)
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16")
eng.set_table(build_item_table(5000, d), dtype="fp32")
reqs = [(h % 5000, c % 5000) for h, c in bench.make_requests(R, H, C, 7)]
ex = eng.executor(R, H // nb, C, with_ids=True)
ex.stage_ids(reqs)
ex.run(_lib.INPUT_IDS, graph=False)
ex.stream.synchronize()
lib = _lib.load()
lib.flame_debug_attn_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(4 * 4096, dtype=torch.int64, device="cuda")
lib.flame_debug_attn_trace(ctypes.c_void_p(buf.data_ptr()))
ex.run(_lib.INPUT_IDS, graph=False)
ex.stream.synchronize()
lib.flame_debug_attn_trace(None)
t = buf.cpu().numpy().astype(np.uint64).reshape(4, 4096)
names = {21: "P:stage", 31: "M:full", 32: "M:projc", 33: "M:qrdy", 35: "M:pfull",
         41: "projfull", 42: "qready", 43: "s_full", 44: "p_arr", 45: "o_full", 46: "out"}
t0 = min(int(x >> 8) for row in t for x in row if x)
for slot in range(4):
    ev = [(int(x >> 8) - t0, int(x & 0xff)) for x in t[slot] if x]
    if not ev:
        continue
    print(f"slot {slot}: {len(ev)} events, span {ev[-1][0]} cycles")
    print("  ", " ".join(f"{names.get(c, c)}@{c0}" for c0, c in ev[:60]))
    gaps = defaultdict(list)
    for (a, ca), (b, cb) in zip(ev, ev[1:]):
        gaps[(names.get(ca, ca), names.get(cb, cb))].append(b - a)
    for k, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1]))[:10]:
        print(f"   {k[0]:>8s} -> {k[1]:<8s} n={len(v):5d} mean={np.mean(v):8.0f} total={sum(v):9d}")
