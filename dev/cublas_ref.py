"""cuBLAS (torch.bmm) on the cfg3 FFN / projection shapes, for comparison with
gemm_bf16_tcgen05 (plain GEMM, no epilogue): dev measurement only."""
import json
import sys

import torch


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


out = {}
G = 8
for name, (M, N, K) in {"w1": (32768, 2048, 512), "w2": (32768, 512, 2048), "qkv": (32768, 1536, 512),
                        "oproj": (32768, 512, 512), "square8k": (8192, 8192, 8192)}.items():
    g = 1 if name == "square8k" else G
    a = torch.randn(g, M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(g, K, N, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(g, M, N, device="cuda", dtype=torch.bfloat16)
    ms = t(lambda: torch.bmm(a, b, out=c))
    out[name] = {"ms": round(ms, 4), "tflops": round(2 * g * M * N * K / ms / 1e9, 1)}
print(json.dumps(out))
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cublas_ref.json", "w"))
