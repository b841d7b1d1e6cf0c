"""FFN W1 -> GELU -> W2 with the hidden activations (Hf) L2-resident vs through HBM
(dev measurement for the on-chip-FFN question).  Needs a GPU.

"full":    W1 over all G x 32768 rows writes Hf (1.07 GB) to HBM, W2 reads it back.
"chunk m": rows laid out chunk-major ([M/m][G][m][K]); per chunk W1 writes a
           G x m x F Hf buffer that is reused by every chunk (m = 2048: 64 MB,
           L2-resident) and W2 consumes it at once.
Both use the production epilogues of the non-final layer (W1: bias + GELU, bf16
out; W2: bias + bf16 residual, fp32 out).  Reported: burst time (median of 20
single passes) and a sustained rate over ~1.5 s of back-to-back passes with the
NVML SM clock and board power sampled during it (the power-capped regime the
e2e number lives in).

    python dev/ffn_chunk_ab.py [out.json]
"""
import ctypes
import json
import sys
import threading
import time

import torch

sys.path.insert(0, "/root/repo")
from paper_2509_22681_b200 import _lib  # noqa: E402

lib = _lib.load()
f = lib.flame_debug_gemm
f.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 7 + [ctypes.c_int] * 4 + [ctypes.c_void_p] * 3 + [ctypes.c_int]
f.restype = ctypes.c_int
BIAS, GELU, RESID, OUT_F32, RESID_BF16 = 1, 2, 4, 8, 256

G, M, D, F = 8, 32768, 512, 2048
x = torch.randn(G, M, D, device="cuda", dtype=torch.bfloat16)  # FFN input (also the W2 residual)
w1 = torch.randn(G, F, D, device="cuda", dtype=torch.bfloat16) * 0.05
w2 = torch.randn(G, D, F, device="cuda", dtype=torch.bfloat16) * 0.02
b1 = torch.randn(G, F, device="cuda")
b2 = torch.randn(G, D, device="cuda")
out = torch.empty(G, M, D, device="cuda", dtype=torch.float32)


def gemm(epi, a, w, o, bias, rb, m, n, k):
    st = torch.cuda.current_stream().cuda_stream  # the capture stream inside graphed()
    rc = f(epi, a, w, o, bias, rb, None, None, m, n, k, G, st, None, None, 0)
    assert rc == 0, lib.flame_last_error()


def make(m):
    if m == M:
        hf = torch.empty(G, M, F, device="cuda", dtype=torch.bfloat16)

        def run():
            gemm(BIAS | GELU, x.data_ptr(), w1.data_ptr(), hf.data_ptr(), b1.data_ptr(), None, M, F, D)
            gemm(BIAS | RESID | RESID_BF16 | OUT_F32, hf.data_ptr(), w2.data_ptr(), out.data_ptr(), b2.data_ptr(),
                 x.data_ptr(), M, D, F)
        return run, hf
    n = M // m
    xc = x.view(n, G, m, D)  # chunk-major layout (same bytes)
    oc = out.view(n, G, m, D)
    hf = torch.empty(G, m, F, device="cuda", dtype=torch.bfloat16)

    def run():
        for c in range(n):
            gemm(BIAS | GELU, xc[c].data_ptr(), w1.data_ptr(), hf.data_ptr(), b1.data_ptr(), None, m, F, D)
            gemm(BIAS | RESID | RESID_BF16 | OUT_F32, hf.data_ptr(), w2.data_ptr(), oc[c].data_ptr(),
                 b2.data_ptr(), xc[c].data_ptr(), m, D, F)
    return run, hf


def burst(run, n=20):
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(n):
        time.sleep(0.02)  # let the clock recover: a burst figure
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def sustained(run, seconds=1.5):
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.01)

    run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # size the loop from one pass
    e0.record(); run(); e1.record(); e1.synchronize()
    iters = max(10, int(seconds * 1000 / e0.elapsed_time(e1)))
    th = threading.Thread(target=sampler)
    th.start()
    e0.record()
    for _ in range(iters):
        run()
    e1.record()
    e1.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / iters
    half = samples[len(samples) // 3:]  # after the power cap engages
    clk = sorted(c for c, _ in half)[len(half) // 2] if half else None
    pw = sorted(p for _, p in half)[len(half) // 2] if half else None
    _ = t0
    return ms, iters, clk, pw


def graphed(m):
    """One pass captured as a CUDA graph, so 2 x M/m launches cost no host time."""
    run, hf = make(m)
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    return g.replay, hf


res = {}
for m in (M, 4096, 2048, 1024):
    run, hf = graphed(m)
    b = burst(run)
    ms, iters, clk, pw = sustained(run)
    flops = 2 * 2 * G * M * D * F
    res[f"m{m}"] = {"hf_mb": round(hf.numel() * 2 / 2**20, 1), "burst_ms": round(b, 4),
                    "burst_tflops": round(flops / b / 1e9, 1), "sustained_ms": round(ms, 4), "iters": iters,
                    "sustained_sm_mhz": clk, "sustained_power_w": pw}
    print(m, res[f"m{m}"], flush=True)
    del hf, run
    torch.cuda.synchronize()
    time.sleep(1.0)
# second pass in reverse order (power / thermal drift)
for m in (1024, 2048, 4096, M):
    run, hf = graphed(m)
    ms, iters, clk, pw = sustained(run)
    res[f"m{m}"]["sustained_ms_2"] = round(ms, 4)
    res[f"m{m}"]["sustained_sm_mhz_2"] = clk
    print(m, "repeat", round(ms, 4), clk, pw, flush=True)
    del hf, run
    time.sleep(1.0)
print(json.dumps(res, indent=1))
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ffn_chunk_ab.json", "w"), indent=1)
