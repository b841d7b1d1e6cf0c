// Host launchers for the tcgen05 GEMM (template dispatch over tile width and
// fused epilogue) — shared by the model pipeline and the debug entry points.
#pragma once
#include <cuda_runtime.h>
#include <cstdlib>
#include "gemm_tcgen05.cuh"
#include "tmap.cuh"
#include "device_once.cuh"

namespace flame {

struct GemmProblem {
  // A: bf16 (fp32 with EPI_TF32) [G or 1][M][lda], K-major; W: same type [G][N][ldw]
  // (transposed weight)
  const void* A;
  long long lda, a_gstride;
  int a_shared;  // 1: every group reads the same A
  const void* W;
  long long ldw, w_gstride;
  int M, N, K, G;
  GemmEpilogue ep;
  int epi;  // EPI_* flags
};

// Programmatic dependent launch for the kernels of a forward pass (FLAME_PDL=1;
// off by default: measured neutral): each such kernel runs its
// prologue (barrier init, TMEM allocation, tensor-map prefetch) while its
// predecessor drains, then waits in ptx::griddep_wait() for the predecessor's
// results.  Only kernels that execute griddep_wait() before touching predecessor
// data may be launched this way.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("FLAME_PDL");
    return v && atoi(v) == 1;
  }();
  return on;
}

inline void pdl_attr(cudaLaunchAttribute& at) {
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t q = {};
  cudaLaunchAttribute at[1];
  q.gridDim = grid;
  q.blockDim = block;
  q.dynamicSmemBytes = smem;
  q.stream = s;
  if (pdl_enabled()) {
    pdl_attr(at[0]);
    q.attrs = at;
    q.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&q, kernel, args...);
}

// Gated-fusion W2 tile width: BN = 256 (running sum in registers, balanced
// hand-over schedule) for N = 256 / 512, BN = 128 (sum in TMEM) otherwise.
// Measured at cfg3 (N = 512): W2 0.505 -> 0.447 ms, step 2.02 -> 1.95 ms; cfg2
// (N = 256) step -0.9 %; cfg5 (N = 768) W2 0.44 -> 0.47 ms, so it keeps BN = 128
// (profiles/r02h/sched_fence_ab).  FLAME_GATED_BN=128 / 256 forces one (A/B).
// Executors allocate the hand-over scratch only when BN = 256 can be chosen.
inline int gated_bn_env() {
  static const int force = [] {
    const char* v = getenv("FLAME_GATED_BN");
    return v ? atoi(v) : 0;
  }();
  return force;
}
inline bool gated_bn_forced() { return gated_bn_env() == 256; }
inline bool gated_bn256(int N) {
  if (N < 256 || N % 32 != 0) return false;
  if (gated_bn_env() == 256) return true;
  if (gated_bn_env() == 128) return false;
  return N % 256 == 0 && N <= 512;
}

// CTA pairs (cta_group::2, 256-row tiles) unless FLAME_GEMM_CLUSTER=1
static int gemm_cluster_pref() {
  static int v = [] {
    const char* e = getenv("FLAME_GEMM_CLUSTER");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  return v;
}

template <int BN, int EPI>
static cudaError_t launch_gemm_t(const GemmProblem& p, cudaStream_t s, int num_sms) {
  using C1 = gemm::Cfg<BN, EPI, 1>;
  using C = gemm::Cfg<BN, EPI, 2>;
  static DeviceOnce once;
  static int max_clusters_dev[kMaxDevices];  // co-resident CTA pairs at this smem size, per device
  cudaError_t setup = once.run([&](int dev) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tcgen05<BN, EPI, 1>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C1::kSmemBytes);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(gemm_bf16_tcgen05<BN, EPI, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::kSmemBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t q = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    q.gridDim = dim3(2 * ((num_sms + 1) / 2));
    q.blockDim = dim3(C::kThreads);
    q.dynamicSmemBytes = C::kSmemBytes;
    q.attrs = at;
    q.numAttrs = 1;
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, gemm_bf16_tcgen05<BN, EPI, 2>, &q) != cudaSuccess) {
      cudaGetLastError();
      mc = 0;
    }
    max_clusters_dev[dev] = mc;
    return cudaSuccess;
  });
  if (setup != cudaSuccess) return setup;
  const int max_clusters = max_clusters_dev[current_device()];
  const int m_tiles = (p.M + gemm::BM - 1) / gemm::BM;
  const int n_tiles = (p.N + BN - 1) / BN;
  // CTA pairs halve each CTA's W-tile traffic from L2, which is what paces the
  // K = 512 GEMMs (measured at cfg3: QKV 0.367 -> 0.323 ms, K/V of the history
  // 0.136 -> 0.120 ms), and, since the residual loader decodes once per tile, also
  // O-proj + LN2 statistics (0.175 -> 0.165 ms) and the tf32 expert (0.131 ->
  // 0.120 ms).  FFN W1 (bf16 GELU epilogue) gains too since the epilogue moved to
  // fp32 pairs: 0.513 -> 0.459 ms for bias + GELU alone (dev/gemm_ab.py, cfg3
  // shape), 0.504 -> 0.500 ms in the step, where the folded-LN epilogue is its
  // limit.  GEMMs with K < 512 keep single CTAs.
  static const int pair_min_k_env = [] {  // FLAME_GEMM_PAIR_MINK overrides (A/B)
    const char* e = getenv("FLAME_GEMM_PAIR_MINK");
    return e ? atoi(e) : 0;
  }();
  const int pair_min_k = pair_min_k_env > 0 ? pair_min_k_env : 512;
  const int ncl = (gemm_cluster_pref() == 2 && m_tiles >= 2 && max_clusters > 0 && p.K >= pair_min_k) ? 2 : 1;
  CUtensorMap ta, tb;
  const int ga = p.a_shared ? 1 : p.G;
  constexpr bool kTF32 = (EPI & EPI_TF32) != 0;
  constexpr int kEs = kTF32 ? 4 : 2;                     // operand element bytes
  constexpr int kBKe = kTF32 ? 32 : gemm::BK;            // K elements per 128-byte row
  auto in_map = kTF32 ? make_tmap_f32_3d : make_tmap_bf16_3d;
  if (!in_map(&ta, p.A, p.K, p.M, ga, p.lda * kEs, p.a_gstride * kEs, kBKe, gemm::BM))
    return cudaErrorInvalidValue;
  if (!in_map(&tb, p.W, p.K, p.N, p.G, p.ldw * kEs, p.w_gstride * kEs, kBKe, BN / ncl))
    return cudaErrorInvalidValue;
  CUtensorMap to;
  constexpr int ob = (EPI & EPI_OUT_F32) ? 4 : 2;
  if constexpr ((EPI & EPI_ROWDOT) != 0) {
    // row-dot epilogue writes its partials directly; the map is a valid placeholder
    if (!make_tmap_out_3d(&to, p.ep.out, 4, 32, p.M, 1, 128, 0)) return cudaErrorInvalidValue;
  } else if constexpr (C::kGated) {
    // one [M][N] fp32 output (the gated sum) shared by all groups
    if (!make_tmap_out_3d(&to, p.ep.out, 4, p.N, p.M, 1, p.ep.out_ld * 4, 0)) return cudaErrorInvalidValue;
  } else if (!make_tmap_out_3d(&to, p.ep.out, ob, static_cast<uint64_t>(p.ep.out_col0) + p.N, p.M, p.G,
                               p.ep.out_ld * ob, p.ep.out_gstride * ob)) {
    return cudaErrorInvalidValue;
  }
  CUtensorMap to2 = to, tr = to;
  if constexpr (C::kResidTma) {
    constexpr int rb = (EPI & EPI_RESID_BF16) ? 2 : 4;
    void* rbase = (EPI & EPI_RESID_BF16) ? const_cast<__nv_bfloat16*>(p.ep.resid_b)
                                         : static_cast<void*>(const_cast<float*>(p.ep.resid));
    if (!make_tmap_out_3d(&tr, rbase, rb, p.N, p.M, p.ep.resid_gstride ? p.G : 1, p.ep.resid_ld * rb,
                          p.ep.resid_gstride * rb))
      return cudaErrorInvalidValue;
  }
  if constexpr (C::kDual && !C::kGated) {
    if (!make_tmap_out_3d(&to2, p.ep.out2, 2, p.N, p.M, p.G, p.ep.out2_ld * 2, p.ep.out2_gstride * 2))
      return cudaErrorInvalidValue;
  }
  GemmEpilogue ep = p.ep;
  ep.M = p.M;
  ep.N = p.N;
  if (ncl == 1) {
    const int total = p.G * m_tiles * n_tiles;
    const int grid = total < num_sms ? total : num_sms;
    return launch_pdl(gemm_bf16_tcgen05<BN, EPI, 1>, dim3(grid), dim3(C1::kThreads), C1::kSmemBytes, s, ta, tb,
                      to, to2, tr, p.K / kBKe, m_tiles, n_tiles, p.G, p.a_shared, ep);
  }
  const int total_pairs = p.G * ((m_tiles + 1) / 2) * n_tiles;
  const int clusters = total_pairs < max_clusters ? total_pairs : max_clusters;
  cudaLaunchConfig_t q = {};
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  q.gridDim = dim3(2 * clusters);
  q.blockDim = dim3(C::kThreads);
  q.dynamicSmemBytes = C::kSmemBytes;
  q.stream = s;
  q.attrs = at;
  q.numAttrs = 1;
  if (pdl_enabled()) pdl_attr(at[q.numAttrs++]);
  return cudaLaunchKernelEx(&q, gemm_bf16_tcgen05<BN, EPI, 2>, ta, tb, to, to2, tr, p.K / kBKe, m_tiles, n_tiles,
                            p.G, p.a_shared, ep);
}

template <int BN>
static cudaError_t launch_gemm_bn(const GemmProblem& p, cudaStream_t s, int num_sms) {
  switch (p.epi) {
    case 0: return launch_gemm_t<BN, 0>(p, s, num_sms);
    case EPI_OUT_F32: return launch_gemm_t<BN, EPI_OUT_F32>(p, s, num_sms);
    case EPI_BIAS: return launch_gemm_t<BN, EPI_BIAS>(p, s, num_sms);
    case EPI_BIAS | EPI_GELU: return launch_gemm_t<BN, EPI_BIAS | EPI_GELU>(p, s, num_sms);
    case EPI_RESID | EPI_OUT_F32: return launch_gemm_t<BN, EPI_RESID | EPI_OUT_F32>(p, s, num_sms);
    case EPI_BIAS | EPI_RESID | EPI_OUT_F32:
      return launch_gemm_t<BN, EPI_BIAS | EPI_RESID | EPI_OUT_F32>(p, s, num_sms);
    case EPI_BIAS | EPI_GELU | EPI_OUT_F32:
      return launch_gemm_t<BN, EPI_BIAS | EPI_GELU | EPI_OUT_F32>(p, s, num_sms);
    case EPI_ROWSCALE | EPI_BIAS: return launch_gemm_t<BN, EPI_ROWSCALE | EPI_BIAS>(p, s, num_sms);
    case EPI_ROWSCALE | EPI_BIAS | EPI_GELU:
      return launch_gemm_t<BN, EPI_ROWSCALE | EPI_BIAS | EPI_GELU>(p, s, num_sms);
    case EPI_RESID | EPI_OUT_F32 | EPI_STATS:
      return launch_gemm_t<BN, EPI_RESID | EPI_OUT_F32 | EPI_STATS>(p, s, num_sms);
    case EPI_RESID | EPI_STATS: return launch_gemm_t<BN, EPI_RESID | EPI_STATS>(p, s, num_sms);
    case EPI_BIAS | EPI_RESID | EPI_RESID_BF16 | EPI_OUT_F32:
      return launch_gemm_t<BN, EPI_BIAS | EPI_RESID | EPI_RESID_BF16 | EPI_OUT_F32>(p, s, num_sms);
    case EPI_LNSTATS | EPI_BIAS:
      return launch_gemm_t<BN, EPI_LNSTATS | EPI_BIAS>(p, s, num_sms);
    case EPI_BIAS | EPI_RESID | EPI_RESID_BF16 | EPI_OUT_F32 | EPI_STATS:
      return launch_gemm_t<BN, EPI_BIAS | EPI_RESID | EPI_RESID_BF16 | EPI_OUT_F32 | EPI_STATS>(p, s, num_sms);
    case EPI_LNSTATS | EPI_BIAS | EPI_GELU:
      return launch_gemm_t<BN, EPI_LNSTATS | EPI_BIAS | EPI_GELU>(p, s, num_sms);
    case EPI_BIAS | EPI_GELU | EPI_ROWDOT:
      return launch_gemm_t<BN, EPI_BIAS | EPI_GELU | EPI_ROWDOT>(p, s, num_sms);
    case EPI_BIAS | EPI_GELU | EPI_ROWDOT | EPI_TF32:
      return launch_gemm_t<BN, EPI_BIAS | EPI_GELU | EPI_ROWDOT | EPI_TF32>(p, s, num_sms);
    case EPI_BIAS | EPI_GELU | EPI_OUT_F32 | EPI_TF32:
      return launch_gemm_t<BN, EPI_BIAS | EPI_GELU | EPI_OUT_F32 | EPI_TF32>(p, s, num_sms);
    default: return cudaErrorInvalidValue;
  }
}

// Per-row partial count written by the STATS / ROWDOT epilogues of a GEMM with
// N output columns: one per (column tile, epilogue-warp share).
static int gemm_row_parts(int N, int epi) {
  const int bn = N >= 256 ? 256 : 128;
  return ((N + bn - 1) / bn) * (gemm::gemm_epi_warps(epi) / 4);
}

// debug: trace (g_gemm_trace) only the which-th GEMM launched after flame_debug_gemm_trace
static unsigned long long* g_gemm_trace_buf = nullptr;
static int g_gemm_trace_which = -1, g_gemm_trace_count = 0;

static cudaError_t launch_gemm(const GemmProblem& p, cudaStream_t s, int num_sms) {
  if (p.K % ((p.epi & EPI_TF32) ? 32 : gemm::BK) != 0 || p.M < 1 || p.N < 1 || p.G < 1) return cudaErrorInvalidValue;
  if (g_gemm_trace_buf != nullptr) {
    unsigned long long* v = g_gemm_trace_count++ == g_gemm_trace_which ? g_gemm_trace_buf : nullptr;
    cudaError_t e = cudaMemcpyToSymbolAsync(g_gemm_trace, &v, sizeof(v), 0, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    cudaStreamSynchronize(s);  // the host copy source is a local
  }
  constexpr int kGatedW2 = EPI_BIAS | EPI_RESID | EPI_RESID_BF16 | EPI_GATED;
  if (p.epi & EPI_GATED) {
    if (p.epi != kGatedW2 || p.N % 32 != 0) return cudaErrorInvalidValue;
    // BN = 256 chains are twice as long: only when there are enough of them to
    // occupy every CTA pair (small DSO groups keep BN = 128's parallelism)
    const long long chains256 = (static_cast<long long>(p.M) + 255) / 256 * (p.N / 256);
    if (gated_bn256(p.N) && (chains256 >= num_sms / 2 || gated_bn_forced()))
      return launch_gemm_t<256, kGatedW2>(p, s, num_sms);
    return launch_gemm_t<128, kGatedW2>(p, s, num_sms);
  }
  if (p.N >= 256) return launch_gemm_bn<256>(p, s, num_sms);
  return launch_gemm_bn<128>(p, s, num_sms);
}

}  // namespace flame
