// Host launchers for the tcgen05 GEMM (template dispatch over tile width and
// fused epilogue) — shared by the model pipeline and the debug entry points.
#pragma once
#include <cuda_runtime.h>
#include "gemm_tcgen05.cuh"
#include "tmap.cuh"

namespace flame {

struct GemmProblem {
  // A: bf16 [G or 1][M][lda], K-major; W: bf16 [G][N][ldw] (transposed weight)
  const __nv_bfloat16* A;
  long long lda, a_gstride;
  int a_shared;  // 1: every group reads the same A
  const __nv_bfloat16* W;
  long long ldw, w_gstride;
  int M, N, K, G;
  GemmEpilogue ep;
  int epi;  // EPI_* flags
};

template <int BN, int EPI>
static cudaError_t launch_gemm_t(const GemmProblem& p, cudaStream_t s, int num_sms) {
  using C = gemm::Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tcgen05<BN, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  CUtensorMap ta, tb;
  const int ga = p.a_shared ? 1 : p.G;
  if (!make_tmap_bf16_3d(&ta, p.A, p.K, p.M, ga, p.lda * 2, p.a_gstride * 2, gemm::BK, gemm::BM))
    return cudaErrorInvalidValue;
  if (!make_tmap_bf16_3d(&tb, p.W, p.K, p.N, p.G, p.ldw * 2, p.w_gstride * 2, gemm::BK, BN))
    return cudaErrorInvalidValue;
  CUtensorMap to;
  constexpr int ob = (EPI & EPI_OUT_F32) ? 4 : 2;
  if (!make_tmap_out_3d(&to, p.ep.out, ob, static_cast<uint64_t>(p.ep.out_col0) + p.N, p.M, p.G,
                        p.ep.out_ld * ob, p.ep.out_gstride * ob))
    return cudaErrorInvalidValue;
  const int m_tiles = (p.M + gemm::BM - 1) / gemm::BM;
  const int n_tiles = (p.N + BN - 1) / BN;
  const int total = p.G * m_tiles * n_tiles;
  const int grid = total < num_sms ? total : num_sms;
  GemmEpilogue ep = p.ep;
  ep.M = p.M;
  ep.N = p.N;
  gemm_bf16_tcgen05<BN, EPI><<<grid, gemm::kThreads, C::kSmemBytes, s>>>(
      ta, tb, to, p.K / gemm::BK, m_tiles, n_tiles, p.G, p.a_shared, ep);
  return cudaGetLastError();
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
    default: return cudaErrorInvalidValue;
  }
}

static cudaError_t launch_gemm(const GemmProblem& p, cudaStream_t s, int num_sms) {
  if (p.K % gemm::BK != 0 || p.M < 1 || p.N < 1 || p.G < 1) return cudaErrorInvalidValue;
  if (p.N >= 256) return launch_gemm_bn<256>(p, s, num_sms);
  return launch_gemm_bn<128>(p, s, num_sms);
}

}  // namespace flame
