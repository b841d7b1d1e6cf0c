// SUMI attention on tcgen05 (reference model/attention.py:118-146 for the
// candidate rows, :168-173 for the causal history rows of non-final layers).
//
// One CTA = (Climber block g, request r, head h, 128-row query tile).  All
// candidates of a request read the SAME history K/V rows of that request-block
// (never replicated per candidate).  The candidate's own key/value (the
// diagonal of the SUMI mask) seeds the online-softmax state:
//     m = s_self, l = 1, o = v_self
// and every 128-key history chunk then updates (m, l, o) exactly like the
// streaming softmax of attention_tiled (attention.py:72-115).  With H = 0 the
// loop is empty and the output is v_self (attention.py:131-133).
//
// Per chunk:  S = Q K^T  (tcgen05, M=128 N=128 K=dh, fp32 in TMEM)
//             softmax rows (1 thread = 1 row, tcgen05.ld) -> P bf16 -> smem (SW128)
//             O_j = P V  (tcgen05, M=128 N=dh K=128, V consumed MN-major)
//             o = o * alpha + O_j  in registers.
// Threads 0..127 own TMEM lanes 0..127 (= query rows); warp 4 is the control
// warp (TMA + MMA issue + TMEM allocation).
#pragma once
#include "ptx.cuh"
#include "common.cuh"

namespace flame {

struct AttnArgs {
  const __nv_bfloat16* qkv;  // [G][rows][3*DA]
  __nv_bfloat16* out;        // [G][rows][out_ld]
  long long qkv_gstride;     // elements per group
  long long out_ld, out_gstride;
  int DA;                    // attention width (heads * 64)
  int R;                     // requests in the batch
  int hb_bkt;                // history rows per (request, block) in the row space
  int c_bkt;                 // candidate rows per request in the row space
  int num_blocks;            // N_b (history length split)
  const int* hist_len;       // [R] actual history length H_r
  const int* cand_len;       // [R] actual candidate count C_r
  const float* scale_log2;   // [G] log2(e) / (tau_g * sqrt(head_dim))
};

namespace attn {
constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int DH = 64;
constexpr int kThreads = 160;
constexpr int kTileBytes = kRows * DH * 2;  // 16 KB (Q, K chunk, V chunk)
constexpr int kPBytes = kRows * kKeys * 2;  // 32 KB (two SW128 sub-tiles)
constexpr int kSmemBytes = 3 * kTileBytes + kPBytes + 1024 + 256;
constexpr uint32_t kTmemCols = 256;  // S: cols [0,128), O: cols [128, 128+DH)
}  // namespace attn

// kHist = false : candidate rows (history keys + self)
// kHist = true  : history rows, causal over the request-block's history
template <bool kHist>
__global__ void __launch_bounds__(attn::kThreads, 2) sumi_attention_tcgen05(
    const __grid_constant__ CUtensorMap tm_qkv, AttnArgs a) {
  using namespace attn;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kTileBytes;
  uint8_t* sV = smem + 2 * kTileBytes;
  uint8_t* sP = smem + 3 * kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 3 * kTileBytes + kPBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = bars + 2;
  uint64_t* s_full = bars + 3;
  uint64_t* o_full = bars + 4;
  uint64_t* s_free = bars + 5;
  uint64_t* p_full = bars + 6;
  uint64_t* o_free = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int tile = blockIdx.x;
  const int h = blockIdx.y;
  const int g = blockIdx.z % a.num_blocks;
  const int r = blockIdx.z / a.num_blocks;
  const int hb = a.hist_len[r] / a.num_blocks;  // actual history rows of this request-block
  const int hist_row0 = r * a.hb_bkt;
  const int q_local0 = tile * kRows;
  const int q_row0 = kHist ? hist_row0 + q_local0 : a.R * a.hb_bkt + r * a.c_bkt + q_local0;
  const int q_valid = kHist ? hb : a.cand_len[r];  // rows with local index < q_valid are real
  if (q_local0 >= (kHist ? a.hb_bkt : a.c_bkt)) return;
  int nk = (hb + kKeys - 1) / kKeys;
  if (kHist) nk = min(nk, tile + 1);  // causal: keys <= last query row of the tile

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int qx = h * DH, kx = a.DA + h * DH, vx = 2 * a.DA + h * DH;

  if (threadIdx.x == 128) {
    ptx::tma_prefetch_desc(&tm_qkv);
    for (int i = 0; i < 5; ++i) ptx::mbar_init(&bars[i], 1);
    for (int i = 5; i < 8; ++i) ptx::mbar_init(&bars[i], 128);
    ptx::fence_barrier_init();
  }
  if (warp == 4) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + kKeys;

  if (threadIdx.x == 128) {
    // ------------------------------------------------------- control thread
    ptx::mbar_arrive_expect_tx(q_full, kTileBytes);
    ptx::tma_load_3d(sQ, &tm_qkv, q_full, qx, q_row0, g);
    if (nk > 0) {
      ptx::mbar_arrive_expect_tx(k_full, kTileBytes);
      ptx::tma_load_3d(sK, &tm_qkv, k_full, kx, hist_row0, g);
      ptx::mbar_arrive_expect_tx(v_full, kTileBytes);
      ptx::tma_load_3d(sV, &tm_qkv, v_full, vx, hist_row0, g);
    }
    constexpr uint32_t idesc_s = ptx::make_idesc_bf16(kRows, kKeys, 0, 0);
    constexpr uint32_t idesc_o = ptx::make_idesc_bf16(kRows, DH, 0, 1);
    const uint32_t aQ = ptx::smem_u32(sQ), aK = ptx::smem_u32(sK), aV = ptx::smem_u32(sV),
                   aP = ptx::smem_u32(sP);
    ptx::mbar_wait(q_full, 0);
    for (int j = 0; j < nk; ++j) {
      const uint32_t par = j & 1;
      ptx::mbar_wait(k_full, par);
      if (j > 0) ptx::mbar_wait(s_free, par ^ 1);
      ptx::tc_fence_after();
#pragma unroll
      for (int k = 0; k < DH / 16; ++k)
        ptx::mma_bf16_ss(tS, ptx::make_desc_sw128(aQ + k * 32, 16, 1024),
                         ptx::make_desc_sw128(aK + k * 32, 16, 1024), idesc_s, k != 0);
      ptx::mma_commit(s_full);
      ptx::mbar_wait(p_full, par);  // softmax consumed S_j (so K_j is free) and wrote P_j
      if (j + 1 < nk) {
        ptx::mbar_arrive_expect_tx(k_full, kTileBytes);
        ptx::tma_load_3d(sK, &tm_qkv, k_full, kx, hist_row0 + (j + 1) * kKeys, g);
      }
      ptx::mbar_wait(v_full, par);
      if (j > 0) ptx::mbar_wait(o_free, par ^ 1);
      ptx::tc_fence_after();
#pragma unroll
      for (int k = 0; k < kKeys / 16; ++k) {
        const uint64_t ad = ptx::make_desc_sw128(aP + (k >> 2) * (kRows * 128) + (k & 3) * 32, 16, 1024);
        const uint64_t bd = ptx::make_desc_sw128(aV + k * 16 * 128, kRows * 128, 1024);
        ptx::mma_bf16_ss(tO, ad, bd, idesc_o, k != 0);
      }
      ptx::mma_commit(o_full);
      if (j + 1 < nk) {
        ptx::mbar_wait(o_full, par);  // PV_j done: V_j (and P_j) are free
        ptx::mbar_arrive_expect_tx(v_full, kTileBytes);
        ptx::tma_load_3d(sV, &tm_qkv, v_full, vx, hist_row0 + (j + 1) * kKeys, g);
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------- softmax / epilogue rows
    const int i = threadIdx.x;  // query row within the tile == TMEM lane
    const int qi = q_local0 + i;
    const bool row_ok = qi < q_valid;
    // rows past this request's region (c_bkt < 128) belong to a neighbour or
    // lie past the buffer: never touch their global memory
    const bool in_region = qi < (kHist ? a.hb_bkt : a.c_bkt);
    const long long grow = q_row0 + (in_region ? i : 0);
    const __nv_bfloat16* base = a.qkv + g * a.qkv_gstride + grow * (3LL * a.DA);
    const float sl2 = a.scale_log2[g];
    float o[DH];
    float m, l;
    if (!kHist) {
      // self term: s_self = q . k_self (attention.py:134), seeds the state
      ptx::mbar_wait(q_full, 0);
      float dot = 0.f;
#pragma unroll
      for (int c = 0; c < DH / 8; ++c) {
        const uint4 qv = *reinterpret_cast<const uint4*>(sQ + ptx::sw128_offset(i, c * 16));
        const uint4 kv = in_region ? *reinterpret_cast<const uint4*>(base + kx + c * 8) : make_uint4(0, 0, 0, 0);
        const uint4 vv = in_region ? *reinterpret_cast<const uint4*>(base + vx + c * 8) : make_uint4(0, 0, 0, 0);
        const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&qv);
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
        const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 qf = __bfloat1622float2(q2[e]);
          const float2 kf = __bfloat1622float2(k2[e]);
          const float2 vf = __bfloat1622float2(v2[e]);
          dot = fmaf(qf.x, kf.x, dot);
          dot = fmaf(qf.y, kf.y, dot);
          o[c * 8 + e * 2] = vf.x;
          o[c * 8 + e * 2 + 1] = vf.y;
        }
      }
      m = dot * sl2;
      l = 1.f;
    } else {
      m = -INFINITY;
      l = 0.f;
#pragma unroll
      for (int e = 0; e < DH; ++e) o[e] = 0.f;
    }
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    for (int j = 0; j < nk; ++j) {
      const uint32_t par = j & 1;
      const int key0 = j * kKeys;
      int key_lim = hb - key0;  // keys with local index < key_lim are valid
      if (kHist) key_lim = min(key_lim, qi - key0 + 1);
      ptx::mbar_wait(s_full, par);
      ptx::tc_fence_after();
      // pass 1: chunk max
      float cmax = -INFINITY;
#pragma unroll 1
      for (int c = 0; c < kKeys / 32; ++c) {
        uint32_t s[32];
        ptx::tmem_ld_32x32b_x32(tS + lane_base + c * 32, s);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (c * 32 + e < key_lim) cmax = fmaxf(cmax, __uint_as_float(s[e]));
      }
      const float m_new = fmaxf(m, cmax * sl2);
      const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
      const float alpha = (m == -INFINITY) ? 0.f : ptx::exp2_approx(m - m_use);
      // pass 2: p = exp2(s*scale - m) -> bf16 P tile (SW128 K-major, 2 sub-tiles of 64 keys)
      float psum = 0.f;
#pragma unroll 1
      for (int c = 0; c < kKeys / 32; ++c) {
        uint32_t s[32];
        ptx::tmem_ld_32x32b_x32(tS + lane_base + c * 32, s);
        ptx::tmem_ld_wait();
        uint32_t packed[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float p0 = (c * 32 + e < key_lim) ? ptx::exp2_approx(fmaf(__uint_as_float(s[e]), sl2, -m_use)) : 0.f;
          float p1 = (c * 32 + e + 1 < key_lim) ? ptx::exp2_approx(fmaf(__uint_as_float(s[e + 1]), sl2, -m_use)) : 0.f;
          // accumulate the normaliser from the bf16-rounded weights actually used in P.V
          const uint32_t pk = pack_bf16x2(p0, p1);
          const float2 pr = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk));
          psum += pr.x + pr.y;
          packed[e / 2] = pk;
        }
        uint8_t* sub = sP + (c >> 1) * (kRows * 128);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t byte_in_row = (c & 1) * 64 + q * 16;
          *reinterpret_cast<uint4*>(sub + ptx::sw128_offset(i, byte_in_row)) =
              make_uint4(packed[q * 4], packed[q * 4 + 1], packed[q * 4 + 2], packed[q * 4 + 3]);
        }
      }
      ptx::tc_fence_before();
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(s_free);
      ptx::mbar_arrive(p_full);
      l = l * alpha + psum;
      m = m_new;
      // O_j = P V
      ptx::mbar_wait(o_full, par);
      ptx::tc_fence_after();
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld_32x32b_x32(tO + lane_base + c * 32, ov);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) o[c * 32 + e] = fmaf(o[c * 32 + e], alpha, __uint_as_float(ov[e]));
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(o_free);
    }
    if (row_ok) {
      const float inv = 1.f / l;
      __nv_bfloat16* dst = a.out + g * a.out_gstride + grow * a.out_ld + h * DH;
#pragma unroll
      for (int c = 0; c < DH / 8; ++c) {
        uint4 w;
        w.x = pack_bf16x2(o[c * 8 + 0] * inv, o[c * 8 + 1] * inv);
        w.y = pack_bf16x2(o[c * 8 + 2] * inv, o[c * 8 + 3] * inv);
        w.z = pack_bf16x2(o[c * 8 + 4] * inv, o[c * 8 + 5] * inv);
        w.w = pack_bf16x2(o[c * 8 + 6] * inv, o[c * 8 + 7] * inv);
        reinterpret_cast<uint4*>(dst)[c] = w;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem);
  }
}

}  // namespace flame
