// Shared device helpers: activation functions (reference forms), bf16 packing,
// and the fused GEMM epilogue used by both the tcgen05 and the fp32 paths.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace flame {

// tanh-form GELU, reference forward.py:34-36:
//   0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
template <bool kFast>
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f;  // sqrt(2/pi)
  const float u = k0 * (x + 0.044715f * x * x * x);
  float t;
  if constexpr (kFast) {
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  } else {
    t = tanhf(u);
  }
  return 0.5f * x * (1.0f + t);
}

// reference forward.py:39-40  1 / (1 + exp(-x))
__device__ __forceinline__ float sigmoid_f(float x) { return 1.0f / (1.0f + expf(-x)); }

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <typename GemmEpilogueT>
__device__ __forceinline__ void store_row_segment_bf16(const GemmEpilogueT& ep, int g, int row,
                                                       int col0, const float* v, int n) {
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(ep.out) + g * ep.out_gstride +
                       static_cast<long long>(row) * ep.out_ld + ep.out_col0 + col0;
  if (n == 32 && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w;
      w.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
      w.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
      w.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
      w.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
      reinterpret_cast<uint4*>(out)[q] = w;
    }
  } else {
    for (int j = 0; j < n; ++j) out[j] = __float2bfloat16_rn(v[j]);
  }
}

template <typename GemmEpilogueT>
__device__ __forceinline__ void store_row_segment_f32(const GemmEpilogueT& ep, int g, int row,
                                                      int col0, const float* v, int n) {
  float* out = reinterpret_cast<float*>(ep.out) + g * ep.out_gstride +
               static_cast<long long>(row) * ep.out_ld + ep.out_col0 + col0;
  if (n == 32 && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      reinterpret_cast<float4*>(out)[q] =
          make_float4(v[q * 4 + 0], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]);
  } else {
    for (int j = 0; j < n; ++j) out[j] = v[j];
  }
}

// Apply bias -> GELU -> residual (that order matches the reference:
// gelu(y@w1+b1) and x + (...)@w2 + b2) to NV consecutive columns of one row.
template <int EPI, int NV, bool kFastMath = true, typename GemmEpilogueT>
__device__ __forceinline__ void epilogue_apply(float* v, const GemmEpilogueT& ep, int g, int row,
                                               int col0) {
  constexpr bool kBias = (EPI & 1) != 0;
  constexpr bool kGelu = (EPI & 2) != 0;
  constexpr bool kResid = (EPI & 4) != 0;
  constexpr bool kF32 = (EPI & 8) != 0;
  const int n = min(NV, ep.N - col0);
  if constexpr (kBias) {
    const float* b = ep.bias + g * ep.bias_gstride + col0;
    if (n == NV) {
#pragma unroll
      for (int j = 0; j < NV; j += 4) {
        const float4 bb = *reinterpret_cast<const float4*>(b + j);
        v[j] += bb.x; v[j + 1] += bb.y; v[j + 2] += bb.z; v[j + 3] += bb.w;
      }
    } else {
      for (int j = 0; j < n; ++j) v[j] += b[j];
    }
  }
  if constexpr (kGelu) {
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = gelu_tanh<kFastMath>(v[j]);
  }
  if constexpr (kResid) {
    const float* rp = ep.resid + g * ep.resid_gstride + static_cast<long long>(row) * ep.resid_ld + col0;
    if (n == NV) {
#pragma unroll
      for (int j = 0; j < NV; j += 4) {
        const float4 rr = *reinterpret_cast<const float4*>(rp + j);
        v[j] += rr.x; v[j + 1] += rr.y; v[j + 2] += rr.z; v[j + 3] += rr.w;
      }
    } else {
      for (int j = 0; j < n; ++j) v[j] += rp[j];
    }
  }
  if constexpr (kF32) {
    store_row_segment_f32(ep, g, row, col0, v, n);
  } else {
    store_row_segment_bf16(ep, g, row, col0, v, n);
  }
}

}  // namespace flame
