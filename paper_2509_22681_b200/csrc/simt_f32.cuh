// fp32 verification path (north star: "within 1e-4 with an fp32 verification
// mode").  tcgen05 has no fp32 MMA kind (tf32 keeps 10 mantissa bits), so this
// mode runs true-fp32 FFMA kernels with the same data layout, the same fused
// epilogues and the same SUMI online-softmax formulation as the bf16 path.
#pragma once
#include "common.cuh"
#include "gemm_tcgen05.cuh"  // GemmEpilogue, EPI_* flags

namespace flame {

// D[g][m][n] = epi( sum_k A[g][m][k] * W[g][n][k] ), 128x128 CTA tile, 8x8 per
// thread, BK = 16 through shared memory.  K-reduction order is fixed per row.
template <int EPI>
__global__ void __launch_bounds__(256) gemm_f32_simt(const float* __restrict__ A, long long lda,
                                                     long long a_gstride,
                                                     const float* __restrict__ W, long long ldw,
                                                     long long w_gstride, int M, int N, int K,
                                                     GemmEpilogue ep) {
  constexpr int BMs = 128, BNs = 128, BKs = 16;
  __shared__ float sA[BKs][BMs + 4];
  __shared__ float sW[BKs][BNs + 4];
  const int g = blockIdx.z;
  const int m0 = blockIdx.y * BMs, n0 = blockIdx.x * BNs;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const float* Ag = A + g * a_gstride;
  const float* Wg = W + g * w_gstride;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += BKs) {
    // 128 rows x 16 k of A and W: 2048 elements each, 8 per thread
    for (int e = threadIdx.x; e < BMs * BKs; e += 256) {
      const int rr = e / BKs, kk = e % BKs;
      const int gm = m0 + rr, gn = n0 + rr, gk = k0 + kk;
      sA[kk][rr] = (gm < M && gk < K) ? Ag[static_cast<long long>(gm) * lda + gk] : 0.f;
      sW[kk][rr] = (gn < N && gk < K) ? Wg[static_cast<long long>(gn) * ldw + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BKs; ++kk) {
      float a[8], w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = sA[kk][ty * 8 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = sW[kk][tx * 8 + j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = m0 + ty * 8 + i;
    const int col0 = n0 + tx * 8;
    if (row < M && col0 < N) {
      epilogue_math<EPI, 8, false>(acc[i], ep, g, row, col0);
      epilogue_store_direct<EPI, 8>(acc[i], ep, g, row, col0);
    }
  }
}

template <typename T>
struct AttnArgsSimt {
  const T* qkv;  // [G][rows][3*DA]
  T* out;        // [G][rows][out_ld]
  long long qkv_gstride, out_ld, out_gstride;
  int DA, R, hb_bkt, c_bkt, num_blocks;
  const int* hist_len;
  const int* cand_len;
  const float* scale;  // [G] 1 / (tau_g * sqrt(head_dim))  (natural-exp domain)
};

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// One thread = one query row; KC-key chunks of K/V staged in shared memory (fp32).
// Same SUMI state update as the tcgen05 kernel: candidates start from the self
// term (m = s_self, l = 1, o = v_self); history rows start empty and are causal.
// T = float: the fp32 verification mode; T = bf16 with DH = 128: the head slots
// wider than the tcgen05 kernel's 64 lanes (64 < head_dim <= 128), fp32 math.
template <typename T, int DH, bool kHist>
__global__ void __launch_bounds__(128) sumi_attention_simt(AttnArgsSimt<T> a) {
  constexpr int KC = DH > 64 ? 32 : 64;
  __shared__ float sK[KC][DH + 1];
  __shared__ float sV[KC][DH + 1];
  const int h = blockIdx.y;
  const int g = blockIdx.z % a.num_blocks;
  const int r = blockIdx.z / a.num_blocks;
  const int hb = a.hist_len[r] / a.num_blocks;
  const int qi = blockIdx.x * 128 + threadIdx.x;
  const int bkt = kHist ? a.hb_bkt : a.c_bkt;
  const int q_valid = kHist ? hb : a.cand_len[r];
  const bool row_ok = qi < q_valid;
  const long long grow = kHist ? static_cast<long long>(r) * a.hb_bkt + qi
                               : static_cast<long long>(a.R) * a.hb_bkt + static_cast<long long>(r) * a.c_bkt + qi;
  const long long ld = 3LL * a.DA;
  const T* G0 = a.qkv + g * a.qkv_gstride;
  const float sc = a.scale[g];
  float q[DH], o[DH];
  float m, l;
  if (qi < bkt) {
    const T* qrow = G0 + grow * ld + h * DH;
#pragma unroll
    for (int e = 0; e < DH; ++e) q[e] = to_f32(qrow[e]);
  } else {
#pragma unroll
    for (int e = 0; e < DH; ++e) q[e] = 0.f;
  }
  if (!kHist && qi < bkt) {
    const T* krow = G0 + grow * ld + a.DA + h * DH;
    const T* vrow = G0 + grow * ld + 2 * a.DA + h * DH;
    float dot = 0.f;
#pragma unroll
    for (int e = 0; e < DH; ++e) dot = fmaf(q[e], to_f32(krow[e]), dot);
#pragma unroll
    for (int e = 0; e < DH; ++e) o[e] = to_f32(vrow[e]);
    m = dot * sc;
    l = 1.f;
  } else {
#pragma unroll
    for (int e = 0; e < DH; ++e) o[e] = 0.f;
    m = -INFINITY;
    l = 0.f;
  }
  int n_keys = hb;
  if (kHist) n_keys = min(hb, (blockIdx.x + 1) * 128);
  const long long hist0 = static_cast<long long>(r) * a.hb_bkt;
  for (int k0 = 0; k0 < n_keys; k0 += KC) {
    __syncthreads();
    for (int e = threadIdx.x; e < KC * DH; e += 128) {
      const int kk = e / DH, dd = e % DH;
      const bool ok = k0 + kk < n_keys;
      const T* rowp = G0 + (hist0 + k0 + kk) * ld;
      sK[kk][dd] = ok ? to_f32(rowp[a.DA + h * DH + dd]) : 0.f;
      sV[kk][dd] = ok ? to_f32(rowp[2 * a.DA + h * DH + dd]) : 0.f;
    }
    __syncthreads();
    int lim = min(KC, n_keys - k0);
    if (kHist) lim = min(lim, qi - k0 + 1);
    for (int kk = 0; kk < lim; ++kk) {
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < DH; ++e) s = fmaf(q[e], sK[kk][e], s);
      s *= sc;
      const float m_new = fmaxf(m, s);
      const float alpha = (m == -INFINITY) ? 0.f : expf(m - m_new);
      const float p = expf(s - m_new);
      l = l * alpha + p;
#pragma unroll
      for (int e = 0; e < DH; ++e) o[e] = fmaf(o[e], alpha, p * sV[kk][e]);
      m = m_new;
    }
  }
  if (row_ok) {
    T* dst = a.out + g * a.out_gstride + grow * a.out_ld + h * DH;
    const float inv = 1.f / l;
#pragma unroll
    for (int e = 0; e < DH; ++e) dst[e] = from_f32<T>(o[e] * inv);
  }
}

}  // namespace flame
