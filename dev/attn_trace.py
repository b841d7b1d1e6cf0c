import sys, ctypes, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench, paper_2509_22681_b200 as fb
from paper_2509_22681_b200 import _lib
from paper_2509_22681_b200.pda import build_item_table
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
d, dh, nb, L, f, tasks, H, C, R, _ = bench.WORKLOADS[name]
cfg = bench.model_config(name)
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16")
eng.set_table(build_item_table(5000, d), dtype="fp32")
reqs = [(h % 5000, c % 5000) for h, c in bench.make_requests(R, H, C, 7)]
ex = eng.executor(R, H // nb, C, with_ids=True)
ex.stage_ids(reqs); ex.run(_lib.INPUT_IDS, graph=False); ex.stream.synchronize()
lib = _lib.load()  # needs a FLAME_DEBUG_TRACE build: FLAME_B200_LIB=dev/var_trace.so (dev/build_variant.sh trace -DFLAME_DEBUG_TRACE)
lib.flame_debug_attn_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(4 * 4096, dtype=torch.int64, device="cuda")
lib.flame_debug_attn_trace(ctypes.c_void_p(buf.data_ptr()))
ex.run(_lib.INPUT_IDS, graph=False); ex.stream.synchronize()
lib.flame_debug_attn_trace(None)
t = buf.cpu().numpy().astype(np.uint64).reshape(4, 4096)
names = {1: "job", 2: "q_ok", 3: "s_ok", 4: "p_arr", 5: "o_ok", 6: "s_ld", 7: "max", 8: "exp", 9: "pv_ok", 11: "C:job", 12: "C:q_ok", 13: "C:S", 14: "C:p_ok", 15: "C:PV"}
t0 = min(int(x >> 8) for row in t for x in row if x)
for slot in range(4):
    ev = [(int(x >> 8) - t0, int(x & 0xff)) for x in t[slot] if x]
    print(f"slot {slot}: {len(ev)} events, span {ev[-1][0] if ev else 0} cycles")
    print("  ", " ".join(f"{names[c]}@{c0}" for c0, c in ev[:40]))
    # per-code average interval to next event
    from collections import defaultdict
    gaps = defaultdict(list)
    for (a, ca), (b, cb) in zip(ev, ev[1:]):
        gaps[(names[ca], names[cb])].append(b - a)
    for k, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1]))[:8]:
        print(f"   {k[0]:>7s} -> {k[1]:<7s} n={len(v):4d} mean={np.mean(v):8.0f} total={sum(v):9d}")
