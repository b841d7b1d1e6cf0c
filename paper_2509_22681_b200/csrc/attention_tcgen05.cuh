// SUMI attention on tcgen05 (reference model/attention.py:118-146 for the
// candidate rows, :168-173 for the causal history rows of non-final layers).
//
// One CTA = (Climber block g, request r, head h) and up to kMaxTiles 128-row
// query tiles of that request.  All candidates of a request read the SAME
// history K/V of that request-block: it is loaded into shared memory once per
// CTA (hb <= 256: resident for every tile; longer histories stream through a
// two-slot ring) and never replicated per candidate.
//
// The candidate's own key/value (the diagonal of the SUMI mask) seeds the
// online-softmax state  m = s_self, l = 1, o = v_self;  every 128-key history
// chunk then updates (m, l, o) as in the streaming softmax of attention_tiled
// (attention.py:72-115).  H = 0 leaves the loop empty: out = v_self
// (attention.py:131-133).
//
// Roles (288 threads):
//   warps 0-3  softmax warpgroup 0 (TMEM lanes 0..127 = its query rows)
//   warps 4-7  softmax warpgroup 1 (same lanes, second TMEM column range)
//   warp 8     control: TMEM allocation, TMA loads, tcgen05.mma issue
// The two warpgroups take alternating query tiles, so the MMAs of one overlap
// the softmax of the other.  Per chunk and warpgroup:
//   S = Q K^T (M=128 N=128 K=64) -> TMEM;  softmax rows (tcgen05.ld) -> P bf16
//   in SW128 K-major smem;  O_j = P V (M=128 N=64 K=128, V consumed MN-major)
//   -> TMEM;  o = o * alpha + O_j in registers.
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
constexpr int kMaxTiles = 4;  // query tiles per CTA
constexpr int kThreads = 288;
constexpr int kTileBytes = kRows * DH * 2;  // 16 KB: Q tile, K chunk, V chunk
constexpr int kPBytes = kRows * kKeys * 2;  // 32 KB: two SW128 sub-tiles
constexpr int kSmemBytes = 2 * kTileBytes + 4 * kTileBytes + 2 * kPBytes + 1024 + 512;
constexpr uint32_t kTmemCols = 512;  // per WG i: S at i*256 + [0,128), O at i*256 + [128,192)
}  // namespace attn

template <bool kHist>
__global__ void __launch_bounds__(attn::kThreads, 1) sumi_attention_tcgen05(
    const __grid_constant__ CUtensorMap tm_qkv, AttnArgs a) {
  using namespace attn;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  uint8_t* sQ = smem;                       // [2] per warpgroup
  uint8_t* sK = smem + 2 * kTileBytes;      // [2] slots
  uint8_t* sV = smem + 4 * kTileBytes;      // [2] slots
  uint8_t* sP = smem + 6 * kTileBytes;      // [2] per warpgroup
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * kTileBytes + 2 * kPBytes);
  uint64_t* q_full = bars + 0;    // [2] per WG (TMA)
  uint64_t* q_empty = bars + 2;   // [2] per WG (MMA commit)
  uint64_t* k_full = bars + 4;    // [2] per slot (TMA)
  uint64_t* v_full = bars + 6;    // [2] per slot (TMA)
  uint64_t* kv_empty = bars + 8;  // [2] per slot (MMA commit)
  uint64_t* s_full = bars + 10;   // [2] per WG (MMA commit)
  uint64_t* o_full = bars + 12;   // [2] per WG (MMA commit)
  uint64_t* p_full = bars + 14;   // [2] per WG (128 softmax threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int h = blockIdx.y;
  const int g = blockIdx.z % a.num_blocks;
  const int r = blockIdx.z / a.num_blocks;
  const int hb = a.hist_len[r] / a.num_blocks;  // actual history rows of this request-block
  const int hist_row0 = r * a.hb_bkt;
  const int bkt = kHist ? a.hb_bkt : a.c_bkt;
  const int n_tiles_total = (bkt + kRows - 1) / kRows;
  const int tile0 = blockIdx.x * kMaxTiles;
  const int n_tiles = min(kMaxTiles, n_tiles_total - tile0);
  const int q_valid = kHist ? hb : a.cand_len[r];  // rows with local index < q_valid are real
  const int q_base = kHist ? hist_row0 : a.R * a.hb_bkt + r * a.c_bkt;
  const int nk_all = (hb + kKeys - 1) / kKeys;
  const bool resident = nk_all <= 2;
  auto chunks_of = [&](int tile) { return kHist ? min(nk_all, tile + 1) : nk_all; };

  const int warp = threadIdx.x / 32;
  const int qx = h * DH, kx = a.DA + h * DH, vx = 2 * a.DA + h * DH;

  if (threadIdx.x == 256) {
    ptx::tma_prefetch_desc(&tm_qkv);
    for (int i = 0; i < 14; ++i) ptx::mbar_init(&bars[i], 1);
    for (int i = 14; i < 16; ++i) ptx::mbar_init(&bars[i], 128);
    ptx::fence_barrier_init();
  }
  if (warp == 8) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (threadIdx.x == 256) {
    // ------------------------------------------------------- control thread
    constexpr uint32_t idesc_s = ptx::make_idesc_bf16(kRows, kKeys, 0, 0);
    constexpr uint32_t idesc_o = ptx::make_idesc_bf16(kRows, DH, 0, 1);
    uint32_t kv_loads[2] = {0, 0};  // loads issued into each K/V slot
    uint32_t kv_frees[2] = {0, 0};  // kv_empty completions consumed per slot
    auto load_kv = [&](int j, int slot) {
      ptx::mbar_arrive_expect_tx(&k_full[slot], kTileBytes);
      ptx::tma_load_3d(sK + slot * kTileBytes, &tm_qkv, &k_full[slot], kx, hist_row0 + j * kKeys, g);
      ptx::mbar_arrive_expect_tx(&v_full[slot], kTileBytes);
      ptx::tma_load_3d(sV + slot * kTileBytes, &tm_qkv, &v_full[slot], vx, hist_row0 + j * kKeys, g);
      ++kv_loads[slot];
    };
    auto load_q = [&](int i, int tile) {
      ptx::mbar_arrive_expect_tx(&q_full[i], kTileBytes);
      ptx::tma_load_3d(sQ + i * kTileBytes, &tm_qkv, &q_full[i], qx, q_base + tile * kRows, g);
    };
    const int rounds = nk_all > 0 ? (n_tiles + 1) / 2 : 0;  // H = 0: no MMA work at all
    for (int i = 0; i < 2 && i < n_tiles && rounds > 0; ++i) load_q(i, tile0 + i);
    if (resident)
      for (int j = 0; j < nk_all; ++j) load_kv(j, j);
    uint32_t chunk_cnt[2] = {0, 0};  // chunks processed per WG (barrier phases)
    for (int k = 0; k < rounds; ++k) {
      const bool has_b = 2 * k + 1 < n_tiles;
      const int nk[2] = {chunks_of(tile0 + 2 * k), has_b ? chunks_of(tile0 + 2 * k + 1) : 0};
      const int nkr = max(nk[0], nk[1]);
      if (!resident) {
        for (int j = 0; j < 2 && j < nkr; ++j) {
          if (kv_loads[j] > kv_frees[j]) {  // slot still read by the previous round's MMAs
            ptx::mbar_wait(&kv_empty[j], kv_frees[j] & 1);
            ++kv_frees[j];
          }
          load_kv(j, j);
        }
      }
      for (int j = 0; j < nkr; ++j) {
        const int slot = j & 1;
        if (j == 0) {
          ptx::mbar_wait(&q_full[0], k & 1);
          if (has_b) ptx::mbar_wait(&q_full[1], k & 1);
        }
        ptx::mbar_wait(&k_full[slot], (kv_loads[slot] - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t aK = ptx::smem_u32(sK + slot * kTileBytes);
        for (int i = 0; i < 2; ++i) {
          if (j >= nk[i]) continue;
          const uint32_t aQ = ptx::smem_u32(sQ + i * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            ptx::mma_bf16_ss(tmem + i * 256, ptx::make_desc_sw128(aQ + kk * 32, 16, 1024),
                             ptx::make_desc_sw128(aK + kk * 32, 16, 1024), idesc_s, kk != 0);
          ptx::mma_commit(&s_full[i]);
          if (j == nk[i] - 1) ptx::mma_commit(&q_empty[i]);  // Q_i no longer read this round
        }
        // prefetch the next round's Q as soon as this round's last S MMAs are done
        for (int i = 0; i < 2; ++i) {
          const int next = 2 * (k + 1) + i;
          if (j == nk[i] - 1 && next < n_tiles) {
            ptx::mbar_wait(&q_empty[i], k & 1);
            load_q(i, tile0 + next);
          }
        }
        ptx::mbar_wait(&v_full[slot], (kv_loads[slot] - 1) & 1);
        const uint32_t aV = ptx::smem_u32(sV + slot * kTileBytes);
        for (int i = 0; i < 2; ++i) {
          if (j >= nk[i]) continue;
          ptx::mbar_wait(&p_full[i], chunk_cnt[i] & 1);  // S_i consumed, P_i written, O_i read
          ptx::tc_fence_after();
          const uint32_t aP = ptx::smem_u32(sP + i * kPBytes);
#pragma unroll
          for (int kk = 0; kk < kKeys / 16; ++kk) {
            const uint64_t ad = ptx::make_desc_sw128(aP + (kk >> 2) * (kRows * 128) + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = ptx::make_desc_sw128(aV + kk * 16 * 128, kRows * 128, 1024);
            ptx::mma_bf16_ss(tmem + i * 256 + kKeys, ad, bd, idesc_o, kk != 0);
          }
          ptx::mma_commit(&o_full[i]);
          ++chunk_cnt[i];
        }
        if (!resident) {
          ptx::mma_commit(&kv_empty[slot]);
          if (j + 2 < nkr) {
            ptx::mbar_wait(&kv_empty[slot], kv_frees[slot] & 1);
            ++kv_frees[slot];
            load_kv(j + 2, slot);
          }
        }
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------- softmax / epilogue rows
    const int wg = warp >> 2;
    const int i = threadIdx.x & 127;  // query row within the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + wg * 256 + lane_base, tO = tS + kKeys;
    uint8_t* myP = sP + wg * kPBytes;
    const float sl2 = a.scale_log2[g];
    uint32_t cnt = 0;
    for (int t = wg; t < n_tiles; t += 2) {
      const int tile = tile0 + t;
      const int qi = tile * kRows + i;
      const bool in_region = qi < bkt;  // rows past the request's region are never touched
      const bool row_ok = qi < q_valid;
      const long long grow = q_base + (in_region ? qi : 0);
      const __nv_bfloat16* base = a.qkv + g * a.qkv_gstride + grow * (3LL * a.DA);
      float o[DH];
      float m, l;
      if (!kHist) {
        // self term: s_self = q . k_self (attention.py:134) seeds the state
        float dot = 0.f;
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) {
          uint4 qv = make_uint4(0, 0, 0, 0), kv = qv, vv = qv;
          if (in_region) {
            qv = *reinterpret_cast<const uint4*>(base + qx + c * 8);
            kv = *reinterpret_cast<const uint4*>(base + kx + c * 8);
            vv = *reinterpret_cast<const uint4*>(base + vx + c * 8);
          }
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
      const int nk = chunks_of(tile);
      for (int j = 0; j < nk; ++j, ++cnt) {
        const int key0 = j * kKeys;
        int key_lim = hb - key0;  // keys with local index < key_lim are valid
        if (kHist) key_lim = min(key_lim, qi - key0 + 1);
        const bool full = key_lim >= kKeys;
        ptx::mbar_wait(&s_full[wg], cnt & 1);
        ptx::tc_fence_after();
        // pass 1: chunk max
        float cmax = -INFINITY;
#pragma unroll
        for (int c = 0; c < kKeys / 32; ++c) {
          uint32_t s[32];
          ptx::tmem_ld_32x32b_x32(tS + c * 32, s);
          ptx::tmem_ld_wait();
          if (full) {
#pragma unroll
            for (int e = 0; e < 32; ++e) cmax = fmaxf(cmax, __uint_as_float(s[e]));
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c * 32 + e < key_lim) cmax = fmaxf(cmax, __uint_as_float(s[e]));
          }
        }
        const float m_new = fmaxf(m, cmax * sl2);
        const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
        const float alpha = (m == -INFINITY) ? 0.f : ptx::exp2_approx(m - m_use);
        // pass 2: p = exp2(s*scale - m) -> bf16 P (SW128 K-major, 2 sub-tiles of 64 keys)
        float psum = 0.f;
#pragma unroll
        for (int c = 0; c < kKeys / 32; ++c) {
          uint32_t s[32];
          ptx::tmem_ld_32x32b_x32(tS + c * 32, s);
          ptx::tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float p0 = ptx::exp2_approx(fmaf(__uint_as_float(s[e]), sl2, -m_use));
            float p1 = ptx::exp2_approx(fmaf(__uint_as_float(s[e + 1]), sl2, -m_use));
            if (!full) {
              p0 = (c * 32 + e < key_lim) ? p0 : 0.f;
              p1 = (c * 32 + e + 1 < key_lim) ? p1 : 0.f;
            }
            psum += p0 + p1;
            packed[e / 2] = pack_bf16x2(p0, p1);
          }
          uint8_t* sub = myP + (c >> 1) * (kRows * 128);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(sub + ptx::sw128_offset(i, (c & 1) * 64 + q * 16)) =
                make_uint4(packed[q * 4], packed[q * 4 + 1], packed[q * 4 + 2], packed[q * 4 + 3]);
        }
        ptx::tc_fence_before();
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive(&p_full[wg]);
        l = l * alpha + psum;
        m = m_new;
        // O_j = P V
        ptx::mbar_wait(&o_full[wg], cnt & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < DH / 32; ++c) {
          uint32_t ov[32];
          ptx::tmem_ld_32x32b_x32(tO + c * 32, ov);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[c * 32 + e] = fmaf(o[c * 32 + e], alpha, __uint_as_float(ov[e]));
        }
        ptx::tc_fence_before();
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
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem);
  }
}

}  // namespace flame
