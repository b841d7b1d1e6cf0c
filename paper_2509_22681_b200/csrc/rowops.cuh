// Row-wise HBM-bound kernels of the FLAME forward pass: LayerNorm (feeding the
// projection GEMMs), the per-block sigmoid-gated fusion, the final expert dot +
// sigmoid, and the history scatter into the block-major row space.
#pragma once
#include <cuda_bf16.h>
#include <type_traits>
#include "common.cuh"

namespace flame {

template <typename T>
__device__ __forceinline__ void store4(T* p, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void store4<float>(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, float a, float b, float c,
                                                     float d) {
  uint2 w;
  w.x = pack_bf16x2(a, b);
  w.y = pack_bf16x2(c, d);
  *reinterpret_cast<uint2*>(p) = w;
}

// LayerNorm, reference forward.py:43-47: mean, biased variance of the
// deviations, (x - mean) / sqrt(var + 1e-5) * scale + shift.  Statistics run
// over the first d_true columns; padded columns have scale = shift = 0 and
// come out as 0.  One warp per row; rows of group g use gamma/beta of block g.
template <typename TOut, int kMaxPerLane = 8>  // float4 chunks per lane: D <= 32*4*kMaxPerLane
__global__ void layer_norm_rows(const float* __restrict__ src, long long src_ld,
                                long long src_gstride, TOut* __restrict__ out, long long out_ld,
                                long long out_gstride, const float* __restrict__ gamma,
                                const float* __restrict__ beta, int rows, int D, int d_true) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int g = blockIdx.y;
  if (warp >= rows) return;
  const float* x = src + g * src_gstride + static_cast<long long>(warp) * src_ld;
  float4 v[kMaxPerLane];
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < kMaxPerLane; ++k) {
    const int c = (k * 32 + lane) * 4;
    v[k] = c < D ? *reinterpret_cast<const float4*>(x + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    sum += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / d_true;
  float sq = 0.f;
#pragma unroll
  for (int k = 0; k < kMaxPerLane; ++k) {
    const int c = (k * 32 + lane) * 4;
    const float e[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float dv = e[q] - mean;
      if (c + q < d_true) sq = fmaf(dv, dv, sq);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const float rstd = rsqrtf(sq / d_true + 1e-5f);
  const float* ga = gamma + g * D;
  const float* be = beta + g * D;
  TOut* y = out + g * out_gstride + static_cast<long long>(warp) * out_ld;
#pragma unroll
  for (int k = 0; k < kMaxPerLane; ++k) {
    const int c = (k * 32 + lane) * 4;
    if (c < D) {
      const float4 gg = *reinterpret_cast<const float4*>(ga + c);
      const float4 bb = *reinterpret_cast<const float4*>(be + c);
      store4<TOut>(y + c, (v[k].x - mean) * rstd * gg.x + bb.x, (v[k].y - mean) * rstd * gg.y + bb.y,
                   (v[k].z - mean) * rstd * gg.z + bb.z, (v[k].w - mean) * rstd * gg.w + bb.w);
    }
  }
}

// Gated fusion, reference forward.py:143-156:
//   fused = sum_b sigmoid(h_b * w_b + c_b) * h_b, accumulated in block order.
template <typename TOut>
__global__ void gated_fusion_rows(const float* __restrict__ xc, long long x_ld, long long x_gstride,
                                  int G, const float* __restrict__ gate_w,
                                  const float* __restrict__ gate_b, TOut* __restrict__ out,
                                  long long out_ld, int rows, int D) {
  const int per_row = D / 4;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(rows) * per_row) return;
  const int row = static_cast<int>(idx / per_row);
  const int c = static_cast<int>(idx % per_row) * 4;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  // the block outputs are read exactly once: issue 8 streaming loads before
  // consuming any, then accumulate strictly in block order
  constexpr int kBatch = 8;
  for (int g0 = 0; g0 < G; g0 += kBatch) {
    float4 hv[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q)
      if (g0 + q < G) hv[q] = __ldcs(reinterpret_cast<const float4*>(xc + (g0 + q) * x_gstride + row * x_ld + c));
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      if (g0 + q >= G) break;
      const int g = g0 + q;
      const float4 h = hv[q];
      const float4 w = __ldg(reinterpret_cast<const float4*>(gate_w + g * D + c));
      const float4 b = __ldg(reinterpret_cast<const float4*>(gate_b + g * D + c));
      acc[0] = acc[0] + sigmoid_f(h.x * w.x + b.x) * h.x;
      acc[1] = acc[1] + sigmoid_f(h.y * w.y + b.y) * h.y;
      acc[2] = acc[2] + sigmoid_f(h.z * w.z + b.z) * h.z;
      acc[3] = acc[3] + sigmoid_f(h.w * w.w + b.w) * h.w;
    }
  }
  store4<TOut>(out + row * out_ld + c, acc[0], acc[1], acc[2], acc[3]);
}

// Expert output, reference forward.py:165-166: sigmoid(hidden @ w2 + b2).
// One warp per candidate row; lane-strided dot over F in a fixed order, then a
// fixed butterfly reduction (deterministic, batch-position invariant).
// Padded rows (c >= C_r) are skipped; real rows go to the compact output
// out[out_offset[r] + c][t].
template <typename TIn>
__global__ void expert_out_rows(const TIn* __restrict__ hidden, long long h_ld,
                                const float* __restrict__ w2, const float* __restrict__ b2,
                                int F, int tasks, int c_bkt, const int* __restrict__ cand_len,
                                const int* __restrict__ out_offset, float* __restrict__ out,
                                int rows) {
  constexpr int kGroup = 8;  // tasks per pass over the hidden row
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (warp >= rows) return;
  const int r = warp / c_bkt, c = warp % c_bkt;
  if (c >= cand_len[r]) return;
  const TIn* hrow = hidden + static_cast<long long>(warp) * h_ld;
  float* dst = out + static_cast<long long>(out_offset[r] + c) * tasks;
  for (int t0 = 0; t0 < tasks; t0 += kGroup) {
    float acc[kGroup];
#pragma unroll
    for (int t = 0; t < kGroup; ++t) acc[t] = 0.f;
    for (int k = lane; k < F; k += 32) {
      const float hv = static_cast<float>(hrow[k]);
#pragma unroll
      for (int t = 0; t < kGroup; ++t)
        if (t0 + t < tasks) acc[t] = fmaf(hv, w2[k * tasks + t0 + t], acc[t]);
    }
#pragma unroll
    for (int t = 0; t < kGroup; ++t) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
    }
    if (lane == 0)
      for (int t = 0; t < kGroup && t0 + t < tasks; ++t) dst[t0 + t] = sigmoid_f(acc[t] + b2[t0 + t]);
  }
}

}  // namespace flame

namespace flame {

// ---------------------------------------------------------- folded LayerNorm
// LN(x) W = rstd * ((x - mean) (gamma . W)) + beta W, so a row only needs its
// centered values (bf16, padded columns 0) and rstd; gamma / beta live in the
// folded weights and the GEMM epilogue (EPI_ROWSCALE | EPI_BIAS).  Statistics
// follow reference forward.py:43-47 (biased variance of the deviations).
struct RowStats {
  float mean, rstd;
};

template <int kChunks>
__device__ __forceinline__ RowStats warp_row_stats(const float4 (&v)[kChunks], int lane, int D,
                                                   int d_true) {
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < kChunks; ++k) sum += (v[k].x + v[k].y) + (v[k].z + v[k].w);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / d_true;
  float sq = 0.f;
#pragma unroll
  for (int k = 0; k < kChunks; ++k) {
    const int c = (k * 32 + lane) * 4;
    const float e[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (c + q < d_true) sq = fmaf(e[q] - mean, e[q] - mean, sq);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  (void)D;
  return {mean, rsqrtf(sq / d_true + 1e-5f)};
}

template <int kChunks>
__device__ __forceinline__ void store_centered(__nv_bfloat16* y, const float4 (&v)[kChunks], float mean,
                                               int lane, int D, int d_true) {
#pragma unroll
  for (int k = 0; k < kChunks; ++k) {
    const int c = (k * 32 + lane) * 4;
    if (c < D) {
      const float a0 = c + 0 < d_true ? v[k].x - mean : 0.f;
      const float a1 = c + 1 < d_true ? v[k].y - mean : 0.f;
      const float a2 = c + 2 < d_true ? v[k].z - mean : 0.f;
      const float a3 = c + 3 < d_true ? v[k].w - mean : 0.f;
      store4<__nv_bfloat16>(y + c, a0, a1, a2, a3);
    }
  }
}

// Expert head combine: score = sigmoid(sum_p partial[row][p][t] + b2[t]) over the
// row-dot partials of the expert GEMM, summed in fixed order; compact output.
__global__ void expert_combine(const float* __restrict__ partial, int n_parts, int tasks,
                               const float* __restrict__ b2, int c_bkt, const int* __restrict__ cand_len,
                               const int* __restrict__ out_offset, float* __restrict__ out, int rows) {
  ptx::griddep_wait();  // PDL: the expert GEMM's row-dot partials
  ptx::griddep_launch();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int r = row / c_bkt, c = row % c_bkt;
  if (c >= cand_len[r]) return;
  const float* p = partial + static_cast<long long>(row) * n_parts * tasks;
  float* dst = out + static_cast<long long>(out_offset[r] + c) * tasks;
  for (int t = 0; t < tasks; ++t) {
    float acc = 0.f;
    for (int k = 0; k < n_parts; ++k) acc += p[k * tasks + t];
    dst[t] = sigmoid_f(acc + b2[t]);
  }
}

}  // namespace flame

namespace flame {

// Embedding rows given by the caller ([R][H_bkt][d] history, [R][C_bkt][d]
// candidates, fp32, width d) -> the padded row space: history goes to the
// block-major layout row (g, r*hb_bkt + i) = hist[r][g*hb_r + i] (the contiguous
// Climber split of the ACTUAL length H_r, forward.py:50-62), candidates to row
// r*c_bkt + c.  Each row is written as fp32 (optional: residual input) and as
// mean-centered bf16 + rstd (folded LN1 input).  Padding rows / cols are zero.
struct AssembleOut {
  float* Eh;                 // [G][R*hb_bkt][D] fp32 or null
  float* Ec;                 // [R*c_bkt][D] fp32 or null
  __nv_bfloat16* Ehc;        // [G][R*hb_bkt][D] centered bf16 or null
  __nv_bfloat16* Ecc;        // [R*c_bkt][D]
  float* rs_h;               // [G][R*hb_bkt]
  float* rs_c;               // [R*c_bkt]
};

template <int kChunks>
__device__ __forceinline__ void assemble_row(const AssembleOut& o, bool hist, long long row,
                                             const float4 (&v)[kChunks], int lane, int D, int d_true, bool valid) {
  float* f = hist ? o.Eh : o.Ec;
  if (f != nullptr) {
    float* dst = f + row * D;
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      const int c = (k * 32 + lane) * 4;
      if (c < D) *reinterpret_cast<float4*>(dst + c) = v[k];
    }
  }
  __nv_bfloat16* y = hist ? o.Ehc : o.Ecc;
  if (y != nullptr) {
    const RowStats st = valid ? warp_row_stats<kChunks>(v, lane, D, d_true) : RowStats{0.f, 0.f};
    store_centered<kChunks>(y + row * D, v, st.mean, lane, D, d_true);
    if (lane == 0) (hist ? o.rs_h : o.rs_c)[row] = st.rstd;
  }
}

template <int kChunks>  // float4 chunks per lane: D <= 128 * kChunks
__global__ void scatter_embeddings(const float* __restrict__ hist, const float* __restrict__ cand,
                                   int d, int D, int R, int H_bkt, int C_bkt, int G, int hb_bkt,
                                   const int* __restrict__ hist_len, const int* __restrict__ cand_len,
                                   AssembleOut o) {
  // one warp per destination row; rows [0, G*R*hb_bkt) history, then R*C_bkt candidates
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const long long n_hist = static_cast<long long>(G) * R * hb_bkt;
  const long long n_cand = static_cast<long long>(R) * C_bkt;
  if (warp >= n_hist + n_cand) return;
  const float* src = nullptr;
  const bool is_hist = warp < n_hist;
  long long row;
  if (is_hist) {
    const int g = static_cast<int>(warp / (static_cast<long long>(R) * hb_bkt));
    const int rem = static_cast<int>(warp % (static_cast<long long>(R) * hb_bkt));
    const int r = rem / hb_bkt, i = rem % hb_bkt;
    const int hb = hist_len[r] / G;
    if (i < hb) src = hist + (static_cast<long long>(r) * H_bkt + g * hb + i) * d;
    row = warp;
  } else {
    row = warp - n_hist;
    const int r = static_cast<int>(row / C_bkt), c = static_cast<int>(row % C_bkt);
    if (c < cand_len[r]) src = cand + row * d;
  }
  float4 v[kChunks];
#pragma unroll
  for (int k = 0; k < kChunks; ++k) {
    const int c = (k * 32 + lane) * 4;
    float e[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) e[q] = (src != nullptr && c + q < d) ? src[c + q] : 0.f;
    v[k] = make_float4(e[0], e[1], e[2], e[3]);
  }
  assemble_row<kChunks>(o, is_hist, row, v, lane, D, d, src != nullptr);
}

}  // namespace flame
