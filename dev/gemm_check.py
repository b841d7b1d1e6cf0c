import ctypes, torch, time, sys
lib = ctypes.CDLL("/root/repo/dev/dbg.so")
f = lib.flame_debug_gemm
f.restype = ctypes.c_int
L = ctypes.c_longlong; P = ctypes.c_void_p; I = ctypes.c_int
f.argtypes = [P, L, L, I, P, L, L, I, I, I, I, P, L, L, P, L, P, L, L, I, P]
torch.manual_seed(0)
dev = "cuda"
def run(M, N, K, G, epi, a_shared=0, out_f32=False):
    A = (torch.randn(1 if a_shared else G, M, K, device=dev) ).bfloat16()
    W = (torch.randn(G, N, K, device=dev) * 0.1).bfloat16()
    bias = torch.randn(G, N, device=dev)
    resid = torch.randn(G, M, N, device=dev)
    of32 = bool(epi & 8)
    out = torch.zeros(G, M, N, device=dev, dtype=torch.float32 if of32 else torch.bfloat16)
    rc = f(A.data_ptr(), K, 0 if a_shared else M*K, a_shared, W.data_ptr(), K, N*K, M, N, K, G,
           out.data_ptr(), N, M*N, bias.data_ptr(), N, resid.data_ptr(), N, M*N, epi, None)
    torch.cuda.synchronize()
    assert rc == 0, rc
    ref = torch.einsum("gmk,gnk->gmn", A.float().expand(G, M, K), W.float())
    if epi & 1: ref = ref + bias[:, None, :]
    if epi & 2: ref = torch.nn.functional.gelu(ref, approximate="tanh")
    if epi & 4: ref = ref + resid
    err = (out.float() - ref).abs().max().item()
    rel = err / ref.abs().max().item()
    print(f"M={M} N={N} K={K} G={G} epi={epi} shared={a_shared}: maxabs={err:.3e} rel={rel:.3e}", flush=True)
    return rel
ok = True
for args in [(128,128,64,1,8),(128,256,64,1,8),(256,512,128,2,8),(300,200,192,3,0),(1000,576,512,2,3),
             (513,512,512,4,12),(777,256,1024,2,13),(4096,1536,512,8,0,1),(100,64,64,1,8)]:
    rel = run(*args)
    ok &= rel < 2e-2
# perf
M,N,K,G = 32768, 2048, 512, 8
A = torch.randn(G, M, K, device=dev).bfloat16(); W = (torch.randn(G, N, K, device=dev)*0.1).bfloat16()
bias = torch.randn(G, N, device=dev); out = torch.empty(G, M, N, device=dev, dtype=torch.bfloat16)
def call():
    return f(A.data_ptr(), K, M*K, 0, W.data_ptr(), K, N*K, M, N, K, G, out.data_ptr(), N, M*N, bias.data_ptr(), N, None, 0, 0, 3, None)
for _ in range(3): call()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): call()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)/10
print(f"perf W1-like G={G} M={M} N={N} K={K}: {ms:.3f} ms  {2*M*N*K*G/ms/1e9:.1f} TFLOP/s", flush=True)
# torch reference perf
Af = A; Wf = W
e0.record()
for _ in range(10): torch.baddbmm(bias[:,None,:].bfloat16(), Af, Wf.transpose(1,2))
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)/10
print(f"torch bmm same: {ms:.3f} ms  {2*M*N*K*G/ms/1e9:.1f} TFLOP/s", flush=True)
print("ALLOK" if ok else "FAIL")
