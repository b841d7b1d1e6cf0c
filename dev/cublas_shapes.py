"""cuBLAS (torch.matmul bf16) on the same GEMM shapes as one cfg3 pass, for comparison."""
import sys
sys.path.insert(0, "/root/repo")
import torch
shapes = {"gemm_kv_hist": (1024, 512), "gemm_qkv_cand": (1536, 512), "gemm_oproj_cand": (512, 512),
          "gemm_ffn_w1": (2048, 512), "gemm_ffn_w2": (512, 2048)}
flops = {k: float(v) for k, v in (a.split("=") for a in sys.argv[1:])}
for name, (N, K) in shapes.items():
    M = 131072 if name == "gemm_kv_hist" else 262144
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = torch.randn(K, N, device="cuda").bfloat16()
    for _ in range(3):
        A @ W
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        A @ W
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cublas {name:>16s} M={M} N={N} K={K}: {ms:.3f} ms {2*M*N*K/ms/1e9:.1f} TF/s")
