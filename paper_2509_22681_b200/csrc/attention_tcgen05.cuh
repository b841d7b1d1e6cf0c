// SUMI attention on tcgen05 (reference model/attention.py:118-146 for the
// candidate rows, :168-173 for the causal history rows of non-final layers).
//
// Persistent kernel: each CTA walks units u = (request r, block g, head h) and
// their 128-row query tiles ("jobs").  Jobs alternate between two softmax
// warpgroups; each warpgroup has its OWN control thread that issues its TMA
// loads and tcgen05 MMAs in a linear schedule, so the two pipelines run
// independently: while one warpgroup computes a softmax, the tensor core works
// on the other's QK^T / PV.
//
// All candidates of a request read the SAME history K/V of that request-block
// (never replicated per candidate): with hb <= 256 the whole K/V of the unit
// stays resident in the warpgroup's two smem slots for all of its tiles of
// that unit; longer histories stream 128-key chunks through the two slots.
// The candidate's own key/value (the diagonal of the SUMI mask) arrives as TMA
// tiles and seeds the online-softmax state  m = s_self, l = 1, o = v_self;
// every history chunk then updates (m, l, o) like attention_tiled
// (attention.py:72-115).  H = 0: no chunks, out = v_self (attention.py:131-133).
//
// Per chunk and warpgroup (TMEM columns of WG i: S [i*256, +128), P [+128, +64),
// O [+192, +64)):
//   S = Q K^T      tcgen05.mma SS, M=128 N=128 K=64          -> TMEM S
//   softmax        1 thread = 1 query row (tcgen05.ld), exp2 -> bf16 P
//   P -> TMEM      tcgen05.st (P never touches shared memory)
//   O_j = P V      tcgen05.mma TS (A = P from TMEM, B = V MN-major smem), N=64
//   o = o*alpha + O_j in registers.
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
  int nh;                    // heads
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
constexpr int kThreads = 320;  // WG0: warps 0-3, WG1: warps 4-7, control: warp 8 (WG0), warp 9 (WG1)
constexpr int kTile = kRows * DH * 2;  // 16 KB
// per warpgroup: Q, K_self, V_self, K[2], V[2]
constexpr int kWGBytes = 7 * kTile;
constexpr int kSmemBytes = 2 * kWGBytes + 1024 + 512;
constexpr uint32_t kTmemCols = 512;
}  // namespace attn

template <bool kHist>
__global__ void __launch_bounds__(attn::kThreads, 1) sumi_attention_tcgen05(
    const __grid_constant__ CUtensorMap tm_qkv, AttnArgs a) {
  using namespace attn;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kWGBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);

  const int warp = threadIdx.x / 32;
  const int G = a.num_blocks;
  const int n_units = a.R * G * a.nh;
  const int bkt = kHist ? a.hb_bkt : a.c_bkt;
  const int n_tiles = (bkt + kRows - 1) / kRows;

  // barriers of warpgroup i: 11 each
  auto B = [&](int i, int k) { return bars + i * 12 + k; };
  // 0 q_full (tx)  1 qs_free (128 WG + 1 control)  2,3 k_full  4,5 v_full
  // 6,7 kv_free (commit)  8 s_full (commit)  9 p_full (128)  10 o_full (commit)
  if (threadIdx.x == 256) {
    ptx::tma_prefetch_desc(&tm_qkv);
    for (int i = 0; i < 2; ++i) {
      for (int k = 0; k < 11; ++k) ptx::mbar_init(B(i, k), 1);
      ptx::mbar_init(B(i, 1), 129);
      ptx::mbar_init(B(i, 9), 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 8) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // job q (per CTA) -> unit u = blockIdx.x + (q / n_tiles) * gridDim.x, tile t = q % n_tiles;
  // warpgroup i takes jobs q = i, i + 2, ...
  struct Job {
    bool valid;
    int u, r, g, h, t, hb, nk_all, nk, q_valid;
    int hist_row0, q_row0;
  };
  auto job_at = [&](int q) {
    Job j{};
    j.u = blockIdx.x + (q / n_tiles) * gridDim.x;
    j.valid = j.u < n_units;
    if (!j.valid) return j;
    j.t = q % n_tiles;
    j.h = j.u % a.nh;
    j.g = (j.u / a.nh) % G;
    j.r = j.u / (a.nh * G);
    j.hb = a.hist_len[j.r] / G;
    j.nk_all = (j.hb + kKeys - 1) / kKeys;
    j.nk = kHist ? min(j.nk_all, j.t + 1) : j.nk_all;
    j.q_valid = kHist ? j.hb : a.cand_len[j.r];
    j.hist_row0 = j.r * a.hb_bkt;
    j.q_row0 = (kHist ? j.hist_row0 : a.R * a.hb_bkt + j.r * a.c_bkt) + j.t * kRows;
    return j;
  };

  if (warp >= 8 && (threadIdx.x & 31) == 0) {
    // --------------------------------------------- control thread of WG i
    const int i = warp - 8;
    uint8_t* base = smem + i * kWGBytes;
    uint8_t *sQ = base, *sKs = base + kTile, *sVs = base + 2 * kTile;
    uint8_t *sK = base + 3 * kTile, *sV = base + 5 * kTile;
    const uint32_t tS = tmem + i * 256, tP = tS + 128, tO = tS + 192;
    constexpr uint32_t idesc_s = ptx::make_idesc_bf16(kRows, kKeys, 0, 0);
    constexpr uint32_t idesc_o = ptx::make_idesc_bf16(kRows, DH, 0, 1);
    uint32_t kv_loads[2] = {0, 0}, kv_frees[2] = {0, 0};
    int res_unit = -1;  // unit whose K/V is resident in the slots (hb <= 256)
    auto load_qs = [&](const Job& j) {
      ptx::mbar_arrive_expect_tx(B(i, 0), (kHist ? 1 : 3) * kTile);
      const int h = j.h;
      ptx::tma_load_3d(sQ, &tm_qkv, B(i, 0), h * DH, j.q_row0, j.g);
      if (!kHist) {
        ptx::tma_load_3d(sKs, &tm_qkv, B(i, 0), a.DA + h * DH, j.q_row0, j.g);
        ptx::tma_load_3d(sVs, &tm_qkv, B(i, 0), 2 * a.DA + h * DH, j.q_row0, j.g);
      }
    };
    auto load_kv = [&](const Job& j, int chunk, int slot) {
      if (kv_loads[slot] > kv_frees[slot]) {  // slot still read by earlier MMAs
        ptx::mbar_wait(B(i, 6 + slot), kv_frees[slot] & 1);
        ++kv_frees[slot];
      }
      const int row = j.hist_row0 + chunk * kKeys;
      ptx::mbar_arrive_expect_tx(B(i, 2 + slot), kTile);
      ptx::tma_load_3d(sK + slot * kTile, &tm_qkv, B(i, 2 + slot), a.DA + j.h * DH, row, j.g);
      ptx::mbar_arrive_expect_tx(B(i, 4 + slot), kTile);
      ptx::tma_load_3d(sV + slot * kTile, &tm_qkv, B(i, 4 + slot), 2 * a.DA + j.h * DH, row, j.g);
      ++kv_loads[slot];
    };
    // K/V needed at the start of a job
    auto prepare_kv = [&](const Job& j) {
      if (j.nk_all <= 2) {
        if (res_unit != j.u)
          for (int c = 0; c < j.nk_all; ++c) load_kv(j, c, c);
        res_unit = j.u;
      } else {
        res_unit = -1;
        for (int c = 0; c < 2 && c < j.nk; ++c) load_kv(j, c, c);
      }
    };
    Job cur = job_at(i);
    if (cur.valid) {
      load_qs(cur);
      prepare_kv(cur);
    }
    uint32_t n = 0, cc = 0;  // jobs / chunks processed by this warpgroup
    for (int q = i; cur.valid; q += 2, ++n) {
      const Job nxt = job_at(q + 2);
      const bool resident = cur.nk_all <= 2;
      ptx::mbar_wait(B(i, 0), n & 1);  // Q (+ self tiles) landed
      for (int c = 0; c < cur.nk; ++c, ++cc) {
        const int slot = resident ? c : (c & 1);
        ptx::mbar_wait(B(i, 2 + slot), (kv_loads[slot] - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t aQ = ptx::smem_u32(sQ), aK = ptx::smem_u32(sK + slot * kTile);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          ptx::mma_bf16_ss(tS, ptx::make_desc_sw128(aQ + kk * 32, 16, 1024),
                           ptx::make_desc_sw128(aK + kk * 32, 16, 1024), idesc_s, kk != 0);
        ptx::mma_commit(B(i, 8));
        if (c == cur.nk - 1) {
          // last S of this job: once it completes (and the WG has read its
          // q / self rows) the Q and self tiles can take the next job
          ptx::mma_commit(B(i, 1));
          if (nxt.valid) {
            ptx::mbar_wait(B(i, 1), n & 1);
            load_qs(nxt);
          }
        }
        ptx::mbar_wait(B(i, 9), cc & 1);  // WG consumed S, stored P, read previous O
        ptx::mbar_wait(B(i, 4 + slot), (kv_loads[slot] - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t aV = ptx::smem_u32(sV + slot * kTile);
#pragma unroll
        for (int kk = 0; kk < kKeys / 16; ++kk)
          ptx::mma_bf16_ts(tO, tP + kk * 8, ptx::make_desc_sw128(aV + kk * 16 * 128, kRows * 128, 1024),
                           idesc_o, kk != 0);
        ptx::mma_commit(B(i, 10));
        if (!resident) {
          ptx::mma_commit(B(i, 6 + slot));
          if (c + 2 < cur.nk) load_kv(cur, c + 2, slot);
        } else if (c == cur.nk - 1 && !(nxt.valid && nxt.u == cur.u)) {
          // unit done: every resident chunk's TMA must have landed (a causal tile
          // may not have used all of them) before its slot can be recycled
          for (int s = 0; s < cur.nk_all; ++s) {
            ptx::mbar_wait(B(i, 2 + s), (kv_loads[s] - 1) & 1);
            ptx::mbar_wait(B(i, 4 + s), (kv_loads[s] - 1) & 1);
            ptx::mma_commit(B(i, 6 + s));
          }
        }
      }
      if (cur.nk == 0) {
        ptx::mbar_arrive(B(i, 1));
        if (nxt.valid) {
          ptx::mbar_wait(B(i, 1), n & 1);
          load_qs(nxt);
        }
        if (resident && !(nxt.valid && nxt.u == cur.u)) res_unit = -1;
      }
      if (nxt.valid) prepare_kv(nxt);
      cur = nxt;
    }
  } else if (warp < 8) {
    // ------------------------------------------------- softmax / epilogue rows
    const int i = warp >> 2;
    const int row = threadIdx.x & 127;  // query row within the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + i * 256 + lane_base, tP = tS + 128, tO = tS + 192;
    const uint8_t* base = smem + i * kWGBytes;
    const uint8_t *sQ = base, *sKs = base + kTile, *sVs = base + 2 * kTile;
    uint32_t n = 0, cc = 0;
    for (int q = i;; q += 2, ++n) {
      const Job j = job_at(q);
      if (!j.valid) break;
      const int qi = j.t * kRows + row;
      const bool row_ok = qi < j.q_valid;
      const float sl2 = a.scale_log2[j.g];
      float o[DH];
      float m, l;
      ptx::mbar_wait(B(i, 0), n & 1);
      if (!kHist) {
        // self term: s_self = q . k_self (attention.py:134) seeds the state
        float dot = 0.f;
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) {
          const uint32_t off = ptx::sw128_offset(row, c * 16);
          const uint4 qv = *reinterpret_cast<const uint4*>(sQ + off);
          const uint4 kv = *reinterpret_cast<const uint4*>(sKs + off);
          const uint4 vv = *reinterpret_cast<const uint4*>(sVs + off);
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
      ptx::mbar_arrive(B(i, 1));  // q / self rows read
      for (int c = 0; c < j.nk; ++c, ++cc) {
        const int key0 = c * kKeys;
        int key_lim = j.hb - key0;  // keys with local index < key_lim are valid
        if (kHist) key_lim = min(key_lim, qi - key0 + 1);
        const bool full = key_lim >= kKeys;
        ptx::mbar_wait(B(i, 8), cc & 1);
        ptx::tc_fence_after();
        float cmax = -INFINITY;
#pragma unroll
        for (int k = 0; k < kKeys / 32; ++k) {
          uint32_t s[32];
          ptx::tmem_ld_32x32b_x32(tS + k * 32, s);
          ptx::tmem_ld_wait();
          if (full) {
#pragma unroll
            for (int e = 0; e < 32; ++e) cmax = fmaxf(cmax, __uint_as_float(s[e]));
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (k * 32 + e < key_lim) cmax = fmaxf(cmax, __uint_as_float(s[e]));
          }
        }
        const float m_new = fmaxf(m, cmax * sl2);
        const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
        const float alpha = (m == -INFINITY) ? 0.f : ptx::exp2_approx(m - m_use);
        float psum = 0.f;
#pragma unroll
        for (int k = 0; k < kKeys / 32; ++k) {
          uint32_t s[32];
          ptx::tmem_ld_32x32b_x32(tS + k * 32, s);
          ptx::tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float p0 = ptx::exp2_approx(fmaf(__uint_as_float(s[e]), sl2, -m_use));
            float p1 = ptx::exp2_approx(fmaf(__uint_as_float(s[e + 1]), sl2, -m_use));
            if (!full) {
              p0 = (k * 32 + e < key_lim) ? p0 : 0.f;
              p1 = (k * 32 + e + 1 < key_lim) ? p1 : 0.f;
            }
            psum += p0 + p1;
            packed[e / 2] = pack_bf16x2(p0, p1);
          }
          ptx::tmem_st_32x32b_x16(tP + k * 16, packed);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(B(i, 9));
        l = l * alpha + psum;
        m = m_new;
        ptx::mbar_wait(B(i, 10), cc & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < DH / 32; ++k) {
          uint32_t ov[32];
          ptx::tmem_ld_32x32b_x32(tO + k * 32, ov);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[k * 32 + e] = fmaf(o[k * 32 + e], alpha, __uint_as_float(ov[e]));
        }
        ptx::tc_fence_before();
      }
      if (row_ok) {
        const float inv = 1.f / l;
        __nv_bfloat16* dst = a.out + j.g * a.out_gstride + static_cast<long long>(j.q_row0 + row) * a.out_ld + j.h * DH;
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
