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
// two MUFU ops (ex2, rcp), ~2 ulp: the bf16 path's gated-fusion epilogue
__device__ __forceinline__ float sigmoid_fast(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * -1.4426950408889634f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return r;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Fused epilogue math on NV consecutive columns of one row, kept in registers
// (every index is a compile-time constant): bias -> GELU -> residual, the order
// of the reference (gelu(y@w1+b1), x + (...)@w2 + b2).  Columns >= ep.N are
// left untouched (the store clips them).
template <int EPI, int NV, bool kFastMath, typename GemmEpilogueT>
__device__ __forceinline__ void epilogue_math(float (&v)[NV], const GemmEpilogueT& ep, int g,
                                              int row, int col0) {
  constexpr bool kBias = (EPI & 1) != 0;
  constexpr bool kGelu = (EPI & 2) != 0;
  constexpr bool kResid = (EPI & 4) != 0;
  const bool full = col0 + NV <= ep.N;
  if constexpr (kBias) {
    const float* b = ep.bias + g * ep.bias_gstride + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < NV; j += 4) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(b + j));
        v[j] += bb.x; v[j + 1] += bb.y; v[j + 2] += bb.z; v[j + 3] += bb.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (col0 + j < ep.N) v[j] += b[j];
    }
  }
  if constexpr (kGelu) {
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = gelu_tanh<kFastMath>(v[j]);
  }
  if constexpr (kResid && (EPI & 256) != 0) {
    // bf16 residual (EPI_RESID_BF16): 8 values per 16-byte load
    const __nv_bfloat16* rp = ep.resid_b + g * ep.resid_gstride + static_cast<long long>(row) * ep.resid_ld + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < NV; j += 8) {
        const uint4 u = *reinterpret_cast<const uint4*>(rp + j);
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(h2[q]);
          v[j + 2 * q] += f.x;
          v[j + 2 * q + 1] += f.y;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (col0 + j < ep.N) v[j] += __bfloat162float(rp[j]);
    }
  } else if constexpr (kResid) {
    const float* rp = ep.resid + g * ep.resid_gstride + static_cast<long long>(row) * ep.resid_ld + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < NV; j += 4) {
        const float4 rr = *reinterpret_cast<const float4*>(rp + j);
        v[j] += rr.x; v[j + 1] += rr.y; v[j + 2] += rr.z; v[j + 3] += rr.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (col0 + j < ep.N) v[j] += rp[j];
    }
  }
}

// Direct (non-TMA) store of NV columns of one row, predicated on ep.N.
template <int EPI, int NV, typename GemmEpilogueT>
__device__ __forceinline__ void epilogue_store_direct(const float (&v)[NV], const GemmEpilogueT& ep,
                                                      int g, int row, int col0) {
  constexpr bool kF32 = (EPI & 8) != 0;
  const long long off = g * ep.out_gstride + static_cast<long long>(row) * ep.out_ld + ep.out_col0 + col0;
  if constexpr (kF32) {
    float* out = reinterpret_cast<float*>(ep.out) + off;
    if (col0 + NV <= ep.N && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < NV; j += 4)
        *reinterpret_cast<float4*>(out + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (col0 + j < ep.N) out[j] = v[j];
    }
  } else {
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(ep.out) + off;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (col0 + j < ep.N) out[j] = __float2bfloat16_rn(v[j]);
  }
}

// Write 32 columns of one row into a 32x32 TMA staging box (row = lane).
// bf16: 64-byte rows, SWIZZLE_64B (16-byte chunk c -> c ^ ((r >> 1) & 3));
// fp32: 128-byte rows, SWIZZLE_128B (chunk c -> c ^ (r & 7)).  Both patterns
// are bank-conflict free for a warp writing one row per lane.
template <bool kF32>
__device__ __forceinline__ void stage_row32(uint8_t* box, int r, const float (&v)[32]) {
  if constexpr (kF32) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int cc = c ^ (r & 7);
      *reinterpret_cast<float4*>(box + r * 128 + cc * 16) =
          make_float4(v[c * 4 + 0], v[c * 4 + 1], v[c * 4 + 2], v[c * 4 + 3]);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int cc = c ^ ((r >> 1) & 3);
      uint4 w;
      w.x = pack_bf16x2(v[c * 8 + 0], v[c * 8 + 1]);
      w.y = pack_bf16x2(v[c * 8 + 2], v[c * 8 + 3]);
      w.z = pack_bf16x2(v[c * 8 + 4], v[c * 8 + 5]);
      w.w = pack_bf16x2(v[c * 8 + 6], v[c * 8 + 7]);
      *reinterpret_cast<uint4*>(box + r * 64 + cc * 16) = w;
    }
  }
}

}  // namespace flame

// ------------------------------------------------------------ fp32 pairs
// fma.rn.f32x2 (FFMA2) does two fp32 FMAs per lane per instruction at the
// issue rate of one scalar FFMA.  A pair lives in a 64-bit register pair.
namespace f2 {
__device__ __forceinline__ uint64_t make(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void split(uint64_t r, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ uint64_t fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// tanh-form GELU on a pair: hx (1 + tanh(x (k0 + k1 x^2))), hx = x / 2
// TWICE the tanh-form GELU, x (1 + tanh(x (k0 + k1 x^2))): the 1/2 is folded
// into every consumer's weights at pack time (FFN W2, expert W2 — exact, a power
// of two), saving one multiply per element in the GELU epilogues; bf16(2 g) =
// 2 bf16(g) and (2 g)(w / 2) = g w, so the results are bit-identical.
__device__ __forceinline__ uint64_t gelu2x(uint64_t x) {
  const uint64_t k0 = make(0.7978845608028654f, 0.7978845608028654f);
  const uint64_t k1 = make(0.7978845608028654f * 0.044715f, 0.7978845608028654f * 0.044715f);
  const uint64_t z = mul(x, fma(mul(x, x), k1, k0));
  float z0, z1;
  split(z, z0, z1);
  asm("tanh.approx.f32 %0, %0;" : "+f"(z0));
  asm("tanh.approx.f32 %0, %0;" : "+f"(z1));
  return fma(x, make(z0, z1), x);
}
}  // namespace f2
