"""Per-tile timeline of one GEMM of a cfg pass (CTA 0): MMA issue vs epilogue.
    python dev/gemm_trace.py cfg3 WHICH   (WHICH = GEMM launch index in the pass: 0 kv_hist,
    1 qkv_cand, 2 oproj, 3 ffn_w1, 4 ffn_w2, 5 expert)"""
import ctypes, sys
from collections import defaultdict
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench, paper_2509_22681_b200 as fb
from paper_2509_22681_b200 import _lib
from paper_2509_22681_b200.pda import build_item_table
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
which = int(sys.argv[2]) if len(sys.argv) > 2 else 3
d, dh, nb, L, f, tasks, H, C, R, _ = bench.WORKLOADS[name]
cfg = bench.model_config(name)
eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16")
eng.set_table(build_item_table(5000, d), dtype="fp32")
reqs = [(h % 5000, c % 5000) for h, c in bench.make_requests(R, H, C, 7)]
ex = eng.executor(R, H // nb, C, with_ids=True)
ex.stage_ids(reqs); ex.run(_lib.INPUT_IDS, graph=False); ex.stream.synchronize()
lib = _lib.load()  # needs a FLAME_DEBUG_TRACE build: FLAME_B200_LIB=dev/var_trace.so (dev/build_variant.sh trace -DFLAME_DEBUG_TRACE)
lib.flame_debug_gemm_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = torch.zeros(4 * 4096 + 2 * 1024, dtype=torch.int64, device="cuda")
lib.flame_debug_gemm_trace(ctypes.c_void_p(buf.data_ptr()), which)
ex.run(_lib.INPUT_IDS, graph=False); ex.stream.synchronize()
lib.flame_debug_gemm_trace(None, -1)
allb = buf.cpu().numpy().astype(np.uint64)
t = allb[:4 * 4096].reshape(4, 4096)
se = allb[4 * 4096:].reshape(-1, 2)
se = se[(se[:, 0] > 0) & (se[:, 1] > 0)].astype(np.int64)
if len(se):
    g0 = se[:, 0].min()
    st, en = (se[:, 0] - g0) / 1e3, (se[:, 1] - g0) / 1e3
    print(f"CTAs {len(se)}: start us min/max {st.min():.1f}/{st.max():.1f}; end us min/p10/p50/p90/max "
          f"{en.min():.1f}/{np.percentile(en, 10):.1f}/{np.median(en):.1f}/{np.percentile(en, 90):.1f}/{en.max():.1f}")
    order = np.argsort(en)
    print("  slowest CTAs (index: end us):", " ".join(f"{i}:{en[i]:.0f}" for i in order[-8:]))
    print("  fastest CTAs (index: end us):", " ".join(f"{i}:{en[i]:.0f}" for i in order[:8]))
names = {1: "M:acc_free", 2: "M:data", 3: "M:commit", 4: "E:full", 5: "E:chunk", 6: "E:free", 7: "P:stage", 8: "E:resid", 9: "E:staged", 10: "M:kb_data", 11: "M:kb_wait"}
t0 = min(int(x >> 8) for row in t for x in row if x)
for slot in range(4):
    ev = [(int(x >> 8) - t0, int(x & 0xff)) for x in t[slot] if x]
    if not ev:
        continue
    print(f"slot {slot}: {len(ev)} events, span {ev[-1][0] - ev[0][0]} cycles")
    print("  ", " ".join(f"{names[c]}@{c0}" for c0, c in ev[:24]))
    gaps = defaultdict(list)
    for (a, ca), (b, cb) in zip(ev, ev[1:]):
        gaps[(names[ca], names[cb])].append(b - a)
    for k, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1]))[:9]:
        print(f"   {k[0]:>10s} -> {k[1]:<10s} n={len(v):4d} mean={np.mean(v):8.0f} total={sum(v):9d}")
