"""gemm_bf16_tcgen05 epilogue variants vs cuBLAS on the cfg3 FFN shapes (dev
measurement: where does W2's time over cuBLAS go?).  Needs a GPU."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2509_22681_b200 import _lib

lib = _lib.load()
f = lib.flame_debug_gemm
f.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 7 + [ctypes.c_int] * 4 + [ctypes.c_void_p] * 3 + [ctypes.c_int]
f.restype = ctypes.c_int
E = dict(BIAS=1, GELU=2, RESID=4, OUT_F32=8, LNSTATS=128, RESID_BF16=256, GATED=512)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(n):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


G = 8
res = {}
ONLY = sys.argv[2] if len(sys.argv) > 2 else None  # e.g. w2_gated: that variant alone (ncu captures)
for shape, (M, N, K) in {"w1": (32768, 2048, 512), "w2": (32768, 512, 2048)}.items():
    a = torch.randn(G, M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(G, N, K, device="cuda", dtype=torch.bfloat16) * 0.05
    out = torch.empty(G, M, N, device="cuda", dtype=torch.float32)
    bias = torch.randn(G, N, device="cuda")
    rb = torch.randn(G, M, N, device="cuda", dtype=torch.bfloat16)
    gw = torch.randn(G, N, device="cuda")
    gb = torch.randn(G, N, device="cuda")
    parts = 4  # folded-LN partials per row (cfg3 O-proj: 2 column tiles x 2 warp shares)
    lns = torch.rand(G, M, parts, 2, device="cuda") + 1.0
    colsum = torch.randn(G, N, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    variants = {"plain": 0, "bias_gelu": E["BIAS"] | E["GELU"],
                "bias_resid_f32": E["BIAS"] | E["RESID"] | E["RESID_BF16"] | E["OUT_F32"],
                "gated": E["BIAS"] | E["RESID"] | E["RESID_BF16"] | E["GATED"],
                "ln_bias_gelu": E["LNSTATS"] | E["BIAS"] | E["GELU"]}
    for vn, epi in variants.items():
        if (shape == "w1" and vn in ("gated", "bias_resid_f32")) or (shape == "w2" and vn == "ln_bias_gelu"):
            continue
        if ONLY and f"{shape}_{vn}" != ONLY:
            continue

        def run(epi=epi):
            rc = f(epi, a.data_ptr(), w.data_ptr(), out.data_ptr(), bias.data_ptr(), rb.data_ptr(), gw.data_ptr(),
                   gb.data_ptr(), M, N, K, G, s, lns.data_ptr(), colsum.data_ptr(), parts)
            assert rc == 0, lib.flame_last_error()
        ms = t(run)
        res[f"{shape}_{vn}"] = {"ms": round(ms, 4), "tflops": round(2 * G * M * N * K / ms / 1e9, 1)}
    if ONLY:
        continue
    wt = w.transpose(1, 2)
    c = torch.empty(G, M, N, device="cuda", dtype=torch.bfloat16)
    ms = t(lambda: torch.bmm(a, wt, out=c))
    res[f"{shape}_cublas"] = {"ms": round(ms, 4), "tflops": round(2 * G * M * N * K / ms / 1e9, 1)}
    # correctness of the plain variant against cuBLAS (bf16 out)
    outb = torch.empty(G, M, N, device="cuda", dtype=torch.bfloat16)
    f(0, a.data_ptr(), w.data_ptr(), outb.data_ptr(), None, None, None, None, M, N, K, G, s, None, None, 0)
    torch.cuda.synchronize()
    res[f"{shape}_plain_maxdiff"] = float((outb.float() - c.float()).abs().max())
    del a, w, out, rb, c, outb, lns
print(json.dumps(res, indent=1))
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gemm_ab.json", "w"))
