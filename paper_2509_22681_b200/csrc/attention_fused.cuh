// Fused candidate projection + SUMI attention on tcgen05 (last layer, layer 0,
// bf16 folded-LN path).  Reference: model/forward.py:111-115 (qc = LN1(x_c) W_q,
// k/v of the candidate rows) feeding model/attention.py:118-146
// (attention_sumi_candidates).
//
// The separate path writes the candidates' Q, K_self and V_self to HBM (one
// [rows][3*DA] bf16 tensor per block: 0.8 GB per cfg3 step) and the attention
// kernel reads them straight back.  Here they never leave the SM: each job
// projects one 128-row candidate tile for one (request, block, head) into TMEM,
// the softmax warps turn it into the S-MMA's Q operand (bf16, in TMEM), the
// self score q.k_self and the V_self rows (smem), and the attention over the
// request-block's history K/V follows in the same CTA.
//
// Work unit u = (request r, block g, head h); a CTA walks units
// blockIdx.x + k * gridDim.x and, inside a unit, PAIRS of 128-row candidate
// tiles (t0 = 2p, t1 = 2p + 1): warpgroup 0 owns t0, warpgroup 1 owns t1.
// Both tiles use the same W_{g,h} k-blocks, so one ring stage holds
//   A_t0 [128 x 32] | A_t1 [128 x 32] | W_q,k,v [192 x 32]   (28 KB, 64-byte swizzle)
// and feeds two M = 128, N = 192 MMAs (6.7 KB of L2 reads per MFLOP instead of
// 9.5 for one tile per W load; the K = 512 GEMMs of this pass are L2-bound).
// The ring holds 4 such 32-deep stages rather than 2 of 64: the same 112 KB, but
// a slot is refilled as soon as its half-sized stage is consumed, so more bytes
// are in flight (measured per-stage period at 2 x 64: 1188 cycles for 768 cycles
// of MMA work, L2-latency-bound).
// The unit's history K/V (hb <= 256 keys: <= 2 chunks of 128) stays resident
// for all its pairs and is read from HBM once per (request, block, head).
//
// TMEM (512 columns), warpgroup i at base i * 256:
//   [0, 192)   projection accumulator q | k | v (fp32); after the epilogue read
//              it, S = Q K^T lives in [0, 128) and P (bf16) in [128, 192)
//   [192, 256) O = P V; its first 32 columns hold Q (bf16) until the last S MMA
//              of the job was issued: every MMA of a job is issued by one thread
//              in the order proj -> S_0 .. S_{nk-1} -> PV_0 .., and tcgen05.mma
//              executes in issue order, so the S MMAs have read Q before PV_0
//              overwrites those columns (accumulate = 0).
//
// Warps: 0-3 warpgroup 0, 4-7 warpgroup 1 (one candidate row per thread: the
// projection epilogue, the softmax, the output), 8 = A / W ring producer
// (TMA), 9 = MMA issuer, 10 = history K/V producer (TMA).
#pragma once
#include "ptx.cuh"
#include "common.cuh"
#include "attention_tcgen05.cuh"

namespace flame {

struct FusedAttnArgs {
  __nv_bfloat16* out;        // [G][rows][out_ld] attention output (candidate rows)
  long long out_ld, out_gstride;
  int DA;                    // attention width (heads * 64)
  int nh;                    // heads
  int R;                     // requests in the batch
  int hb_bkt;                // history rows per (request, block) in the row space
  int c_bkt;                 // candidate rows per request
  int num_blocks;            // G
  int k_blocks;              // D / 64 (projection K steps)
  const int* hist_len;       // [R]
  const int* cand_len;       // [R]
  const float* scale_log2;   // [G]
  const float* rs_c;         // [R * c_bkt] rstd of the centered candidate rows
  const float* cqkv;         // [G][3 * DA] folded-LN column bias (beta @ W)
  int store_tma;             // c_bkt % 128 == 0: output tiles by TMA
  const int* active;         // [1] requests in use (null: all R)
};

namespace fattn {
constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int DH = 64;
// 12 warps.  setmaxnreg moves registers from warpgroup 2 (producer, MMA, K/V
// loader, one idle warp) to the two softmax warpgroups: 2 x 224 + 56 = 504 =
// 3 x 168, the CTA's launch allocation (the pool setmaxnreg.inc draws from; a
// larger sum blocks forever).  Measured at cfg3: 0.609 -> 0.596 ms, the spills
// of the 168-register build (108 bytes) gone.
constexpr int kThreads = 384;
constexpr int kRegsSoftmax = 224, kRegsOther = 56;
static_assert(2 * kRegsSoftmax + kRegsOther <= 3 * 168, "setmaxnreg budget above the launch allocation");
constexpr int kTile = kRows * DH * 2;           // 16 KB: 128 rows x 64 bf16
constexpr int kKB = 32;                         // projection k-block depth (64-byte rows)
constexpr int kATile = kRows * kKB * 2;         // 8 KB: 128 rows x 32 bf16
constexpr int kWPart = DH * kKB * 2;            // 4 KB: 64 rows of W x 32 bf16
constexpr int kWBytes = 3 * kWPart;             // 12 KB: q | k | v rows of W, 32 k
constexpr int kStageBytes = 2 * kATile + kWBytes;  // 28 KB
#ifndef FLAME_FATTN_STAGES
#define FLAME_FATTN_STAGES 4
#endif
constexpr int kStages = FLAME_FATTN_STAGES;
constexpr int kKOff = kStages * kStageBytes;    // history K chunks [2]
constexpr int kVOff = kKOff + 2 * kTile;        // history V chunks [2]
constexpr int kStgOff = kVOff + 2 * kTile;      // per-WG V_self / output staging [2]
constexpr int kBarOff = kStgOff + 2 * kTile;
constexpr int kSmemBytes = kBarOff + 256 + 1024;
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;
// barrier slots
constexpr int RING_FULL = 0, RING_EMPTY = kStages, KV_FULL = 2 * kStages, KV_FREE = 2 * kStages + 2;
constexpr int WGB = 2 * kStages + 3;  // per-WG block of 6: proj_full, q_ready, s_full, s_free, p_full, o_full
constexpr int PROJ_FULL = 0, Q_READY = 1, S_FULL = 2, S_FREE = 3, P_FULL = 4, O_FULL = 5;
constexpr int kBars = WGB + 2 * 6;
}  // namespace fattn

__global__ void __launch_bounds__(fattn::kThreads, 1) sumi_fused_tcgen05(
    const __grid_constant__ CUtensorMap tm_a,    // Ecc [Rc][D] bf16, box 32 x 128, 64-byte swizzle
    const __grid_constant__ CUtensorMap tm_w,    // Wqkv [G][3DA][D] bf16, box 32 x 64, 64-byte swizzle
    const __grid_constant__ CUtensorMap tm_qkv,  // QKV [G][rows][3DA] (history K / V), box 64 x 128
    const __grid_constant__ CUtensorMap tm_out,  // AO [G][rows][DA], box 64 x 128
    FusedAttnArgs a) {
  using namespace fattn;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kBars);

  const int warp = threadIdx.x / 32;
  const int G = a.num_blocks;
  const int R_eff = a.active != nullptr ? min(a.R, __ldg(a.active)) : a.R;
  const int n_units = R_eff * G * a.nh;
  const int KB = a.k_blocks;
  auto WB = [&](int i, int k) { return bars + WGB + i * 6 + k; };

  if (threadIdx.x == 0) {
    for (int k = 0; k < kBars; ++k) ptx::mbar_init(bars + k, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(WB(i, Q_READY), 128);
      ptx::mbar_init(WB(i, S_FREE), 128);
      ptx::mbar_init(WB(i, P_FULL), 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 9) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  if (threadIdx.x == 256) {
    ptx::tma_prefetch_desc(&tm_a);
    ptx::tma_prefetch_desc(&tm_w);
    ptx::tma_prefetch_desc(&tm_qkv);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::griddep_wait();  // PDL: previous kernel's outputs visible from here on
  ptx::griddep_launch();

  // Unit k of this CTA: u = blockIdx.x + k * gridDim.x -> (r, g, h); its work:
  // pairs of 128-row tiles over the request's REAL candidates (C_r), history
  // chunks over its real history (H_r / G).  Every role derives the same list.
  struct Unit {
    bool valid;
    int r, g, h, hb, nk, n_tiles, n_pairs;
  };
  auto unit_at = [&](int k) {
    Unit un{};
    const int u = blockIdx.x + k * gridDim.x;
    un.valid = u < n_units;
    if (!un.valid) return un;
    un.h = u % a.nh;
    un.g = (u / a.nh) % G;
    un.r = u / (a.nh * G);
    un.hb = __ldg(a.hist_len + un.r) / G;
    un.nk = (un.hb + kKeys - 1) / kKeys;
    const int cl = min(__ldg(a.cand_len + un.r), a.c_bkt);
    un.n_tiles = (cl + kRows - 1) / kRows;
    un.n_pairs = (un.n_tiles + 1) / 2;
    return un;
  };
  const int cand_row0 = a.R * a.hb_bkt;  // first candidate row of the QKV / AO row space

  if (warp >= 8) {
    ptx::setmaxnreg_dec<kRegsOther>();
    if (warp == 8) {
      // ------------------------------------------------ A / W ring producer
      const bool leader = ptx::elect_one();
      uint32_t rk = 0;
      unsigned trace_k = 0;
      for (int k = 0;; ++k) {
        const Unit un = unit_at(k);
        if (!un.valid) break;
        for (int p = 0; p < un.n_pairs; ++p) {
          const int t0 = 2 * p;
          const bool has1 = t0 + 1 < un.n_tiles;
          const int arow = un.r * a.c_bkt + t0 * kRows;
          for (int kb = 0; kb < KB; ++kb, ++rk) {
            const int s = rk % kStages;
            if (rk >= kStages) ptx::mbar_wait(bars + RING_EMPTY + s, ((rk / kStages) - 1) & 1);
            ATTN_TRACE(3, 21);
            if (leader) {
              uint8_t* st = smem + s * kStageBytes;
              uint64_t* fb = bars + RING_FULL + s;
#ifdef FLAME_FATTN_DBG_SKIP_W
              // timing experiment only (wrong results): load FLAME_FATTN_DBG_SKIP_W fewer W parts
              constexpr int kWLoads = 3 - FLAME_FATTN_DBG_SKIP_W;
#else
              constexpr int kWLoads = 3;
#endif
              ptx::mbar_arrive_expect_tx(fb, (has1 ? 2 : 1) * kATile + kWLoads * kWPart);
              ptx::tma_load_3d(st, &tm_a, fb, kb * kKB, arow, 0);
              if (has1) ptx::tma_load_3d(st + kATile, &tm_a, fb, kb * kKB, arow + kRows, 0);
              uint8_t* w = st + 2 * kATile;
#pragma unroll
              for (int part = 0; part < kWLoads; ++part)
                ptx::tma_load_3d(w + part * kWPart, &tm_w, fb, kb * kKB, part * a.DA + un.h * DH, un.g);
            }
            __syncwarp();
          }
        }
      }
    } else if (warp == 10) {
      // ---------------------------------------------- history K / V producer
      const bool leader = ptx::elect_one();
      uint32_t ku = 0;
      for (int k = 0;; ++k) {
        const Unit un = unit_at(k);
        if (!un.valid) break;
        if (un.nk == 0 || un.n_pairs == 0) continue;
        if (ku > 0) ptx::mbar_wait(bars + KV_FREE, (ku - 1) & 1);  // previous unit's last PV done
        if (leader) {
          for (int c = 0; c < un.nk; ++c) {
            uint64_t* fb = bars + KV_FULL + c;
            const int row = un.r * a.hb_bkt + c * kKeys;
            ptx::mbar_arrive_expect_tx(fb, 2 * kTile);
            ptx::tma_load_3d(smem + kKOff + c * kTile, &tm_qkv, fb, a.DA + un.h * DH, row, un.g);
            ptx::tma_load_3d(smem + kVOff + c * kTile, &tm_qkv, fb, 2 * a.DA + un.h * DH, row, un.g);
          }
        }
        __syncwarp();
        ++ku;
      }
    } else if (warp == 9) {
      // ------------------------------------------------------ MMA issuer
      const bool leader = ptx::elect_one();
      constexpr uint32_t idesc_p = ptx::make_idesc_bf16(kRows, 3 * DH, 0, 0);
      constexpr uint32_t idesc_s = ptx::make_idesc_bf16(kRows, kKeys, 0, 0);
      constexpr uint32_t idesc_o = ptx::make_idesc_bf16(kRows, DH, 0, 1);
      uint32_t rk = 0, ku = 0;
      uint32_t nj[2] = {0, 0}, cc[2] = {0, 0};
      unsigned trace_k = 0;
      for (int k = 0;; ++k) {
        const Unit un = unit_at(k);
        if (!un.valid) break;
        const bool kv = un.nk > 0 && un.n_pairs > 0;
        for (int p = 0; p < un.n_pairs; ++p) {
          const bool has1 = 2 * p + 1 < un.n_tiles;
          const int nw = has1 ? 2 : 1;
          // projection: proj_i = A_ti (128 x D) . W_{g,h}^T (D x 192) for both tiles
          for (int kb = 0; kb < KB; ++kb, ++rk) {
            const int s = rk % kStages;
            ptx::mbar_wait(bars + RING_FULL + s, (rk / kStages) & 1);
            ATTN_TRACE(2, 31);
            ptx::tc_fence_after();
            if (leader) {
              const uint32_t st = ptx::smem_u32(smem + s * kStageBytes);
              const uint32_t aw = st + 2 * kATile;
#pragma unroll
              for (int kk = 0; kk < kKB / 16; ++kk) {
                const uint64_t bd = ptx::make_desc_sw64(aw + kk * 32, 512);
                ptx::mma_bf16_ss(tmem, ptx::make_desc_sw64(st + kk * 32, 512), bd, idesc_p, (kb | kk) != 0);
                if (has1)
                  ptx::mma_bf16_ss(tmem + 256, ptx::make_desc_sw64(st + kATile + kk * 32, 512), bd, idesc_p,
                                   (kb | kk) != 0);
              }
              ptx::mma_commit(bars + RING_EMPTY + s);
            }
            __syncwarp();
          }
          if (leader) {
            ptx::mma_commit(WB(0, PROJ_FULL));
            if (has1) ptx::mma_commit(WB(1, PROJ_FULL));
          }
          __syncwarp();
          // each warpgroup stored its Q (bf16) into TMEM: its first S MMA starts at once
          ATTN_TRACE(2, 32);
          auto issue_s = [&](int i, int c) {
            if (p == 0) ptx::mbar_wait(bars + KV_FULL + c, ku & 1);  // first use of chunk c in this unit
            ptx::tc_fence_after();
            const uint32_t aK = ptx::smem_u32(smem + kKOff + c * kTile);
            const uint32_t tS = tmem + i * 256, tQ = tS + 192;
            if (leader) {
#pragma unroll
              for (int kk = 0; kk < DH / 16; ++kk)
                ptx::mma_bf16_ts(tS, tQ + kk * 8, ptx::make_desc_sw128(aK + kk * 32, 16, 1024), idesc_s, kk != 0);
              ptx::mma_commit(WB(i, S_FULL));
            }
            __syncwarp();
          };
          for (int i = 0; i < nw; ++i) {
            ptx::mbar_wait(WB(i, Q_READY), nj[i] & 1);
            if (un.nk > 0) issue_s(i, 0);
          }
          ATTN_TRACE(2, 33);
          if (un.nk > 0) {
            for (int c = 0; c < un.nk; ++c) {
              for (int i = 0; i < nw; ++i) {
                ptx::mbar_wait(WB(i, S_FREE), cc[i] & 1);  // S_c in the WG's registers
                if (c + 1 < un.nk) {
                  // S_{c+1} runs under the softmax of chunk c (waits for chunk c+1's K only on first use)
                  if (p == 0) ptx::mbar_wait(bars + KV_FULL + c + 1, ku & 1);
                  ptx::tc_fence_after();
                  const uint32_t aK = ptx::smem_u32(smem + kKOff + (c + 1) * kTile);
                  const uint32_t tS = tmem + i * 256, tQ = tS + 192;
                  if (leader) {
#pragma unroll
                    for (int kk = 0; kk < DH / 16; ++kk)
                      ptx::mma_bf16_ts(tS, tQ + kk * 8, ptx::make_desc_sw128(aK + kk * 32, 16, 1024), idesc_s, kk != 0);
                    ptx::mma_commit(WB(i, S_FULL));
                  }
                  __syncwarp();
                }
              }
              for (int i = 0; i < nw; ++i) {
                ptx::mbar_wait(WB(i, P_FULL), cc[i] & 1);  // P_c stored (and O rescaled)
                ATTN_TRACE(2, 35);
                ptx::tc_fence_after();
                const uint32_t aV = ptx::smem_u32(smem + kVOff + c * kTile);
                const uint32_t tP = tmem + i * 256 + 128, tO = tmem + i * 256 + 192;
                if (leader) {
#pragma unroll
                  for (int kk = 0; kk < kKeys / 16; ++kk)
                    ptx::mma_bf16_ts(tO, tP + kk * 8, ptx::make_desc_sw128(aV + kk * 16 * 128, kRows * 128, 1024),
                                     idesc_o, (c | kk) != 0);
                  ptx::mma_commit(WB(i, O_FULL));
                }
                __syncwarp();
                ++cc[i];
              }
            }
          }
          for (int i = 0; i < nw; ++i) ++nj[i];
        }
        if (kv) {
          if (leader) ptx::mma_commit(bars + KV_FREE);  // the unit's last PV done -> K / V slots free
          __syncwarp();
          ++ku;
        }
      }
    }
  } else {
    ptx::setmaxnreg_inc<kRegsSoftmax>();
    // ---------------------------------- projection epilogue, softmax, output
    const int i = warp >> 2;
    const int row = threadIdx.x & 127;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tW = tmem + i * 256 + lane_base;
    const uint32_t tS = tW, tP = tW + 128, tO = tW + 192, tQ = tW + 192;
    uint8_t* stage = smem + kStgOff + i * kTile;
    uint32_t nj = 0, cc = 0;
    bool store_pending = false;
    unsigned trace_k = 0;
    for (int k = 0;; ++k) {
      const Unit un = unit_at(k);
      if (!un.valid) break;
      const float sl2 = __ldg(a.scale_log2 + un.g);
      const float* cq = a.cqkv + static_cast<long long>(un.g) * 3 * a.DA + un.h * DH;
      const float* ck = cq + a.DA;
      const float* cv = cq + 2 * a.DA;
      for (int p = 0; p < un.n_pairs; ++p) {
        const int t = 2 * p + i;
        if (t >= un.n_tiles) continue;  // odd tile count: warpgroup 1 sits this pair out
        const int cidx = un.r * a.c_bkt + t * kRows + row;  // candidate row index
        const bool row_ok = t * kRows + row < min(__ldg(a.cand_len + un.r), a.c_bkt);
        const float rs = row_ok ? __ldg(a.rs_c + cidx) : 0.f;
        ptx::mbar_wait(WB(i, PROJ_FULL), nj & 1);
        ATTN_TRACE(i, 41);
        ptx::tc_fence_after();
        // ---- projection epilogue: q = rs * acc + c_q (folded LN1), same for k, v
        // (fp32 pairs: FFMA2 does two lanes' worth per issue slot)
        const uint64_t rs2 = f2::make(rs, rs);
        uint64_t dot2 = f2::make(0.f, 0.f);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t qa[32], ka[32];
          ptx::tmem_ld_32x32b_x32(tW + half * 32, qa);
          ptx::tmem_ld_32x32b_x32(tW + 64 + half * 32, ka);
          ptx::tmem_ld_wait();
          uint32_t qb[16];
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 bq = __ldg(reinterpret_cast<const float4*>(cq + half * 32 + e));
            const float4 bk = __ldg(reinterpret_cast<const float4*>(ck + half * 32 + e));
            const uint64_t q01 = f2::fma(rs2, f2::make(__uint_as_float(qa[e]), __uint_as_float(qa[e + 1])), f2::make(bq.x, bq.y));
            const uint64_t q23 = f2::fma(rs2, f2::make(__uint_as_float(qa[e + 2]), __uint_as_float(qa[e + 3])), f2::make(bq.z, bq.w));
            const uint64_t k01 = f2::fma(rs2, f2::make(__uint_as_float(ka[e]), __uint_as_float(ka[e + 1])), f2::make(bk.x, bk.y));
            const uint64_t k23 = f2::fma(rs2, f2::make(__uint_as_float(ka[e + 2]), __uint_as_float(ka[e + 3])), f2::make(bk.z, bk.w));
            dot2 = f2::fma(q01, k01, dot2);
            dot2 = f2::fma(q23, k23, dot2);
            float q0, q1, q2, q3;
            f2::split(q01, q0, q1);
            f2::split(q23, q2, q3);
            qb[e / 2] = pack_bf16x2(q0, q1);
            qb[e / 2 + 1] = pack_bf16x2(q2, q3);
          }
          ptx::tmem_st_32x32b_x16(tQ + half * 16, qb);
        }
        float dot;
        {
          float d0, d1;
          f2::split(dot2, d0, d1);
          dot = d0 + d1;
        }
        // Q is in TMEM: the S MMAs may start (they overwrite q | k, columns [0, 128);
        // v, read below, lives in [128, 192), which only this warpgroup's P
        // overwrites).  Without history there is no S / P: the next projection
        // (all of [0, 192)) is what follows Q_READY, so v must be read first.
        ptx::tmem_st_wait();
        if (un.nk > 0) {
          ptx::tc_fence_before();
          ptx::mbar_arrive(WB(i, Q_READY));
        }
        ATTN_TRACE(i, 42);
        // V_self rows -> the staging tile (bf16, SW128 row layout); the previous
        // job's output store must have finished reading the staging first
        if (store_pending) {
          if (row == 0) ptx::tma_store_wait_read<0>();
          asm volatile("bar.sync %0, 128;" ::"r"(1 + i) : "memory");
          store_pending = false;
        }
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t va[32];
          ptx::tmem_ld_32x32b_x32(tW + 128 + half * 32, va);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            const int e = c8 * 8;
            const float4 b0 = __ldg(reinterpret_cast<const float4*>(cv + half * 32 + e));
            const float4 b1 = __ldg(reinterpret_cast<const float4*>(cv + half * 32 + e + 4));
            float v[8];
            f2::split(f2::fma(rs2, f2::make(__uint_as_float(va[e]), __uint_as_float(va[e + 1])), f2::make(b0.x, b0.y)), v[0], v[1]);
            f2::split(f2::fma(rs2, f2::make(__uint_as_float(va[e + 2]), __uint_as_float(va[e + 3])), f2::make(b0.z, b0.w)), v[2], v[3]);
            f2::split(f2::fma(rs2, f2::make(__uint_as_float(va[e + 4]), __uint_as_float(va[e + 5])), f2::make(b1.x, b1.y)), v[4], v[5]);
            f2::split(f2::fma(rs2, f2::make(__uint_as_float(va[e + 6]), __uint_as_float(va[e + 7])), f2::make(b1.z, b1.w)), v[6], v[7]);
            uint4 w;
            w.x = pack_bf16x2(v[0], v[1]);
            w.y = pack_bf16x2(v[2], v[3]);
            w.z = pack_bf16x2(v[4], v[5]);
            w.w = pack_bf16x2(v[6], v[7]);
            *reinterpret_cast<uint4*>(stage + ptx::sw128_offset(row, (half * 32 + e) * 2)) = w;
          }
        }
        if (un.nk == 0) {
          ptx::tc_fence_before();
          ptx::mbar_arrive(WB(i, Q_READY));
        }
        // the diagonal of the SUMI mask seeds the state: m = s_self, l = 1 (attention.py:134)
        const float m_self = dot * sl2;
        float m = m_self, l = 1.f;
        for (int c = 0; c < un.nk; ++c, ++cc) {
          const int key_lim = un.hb - c * kKeys;
          const bool full = __all_sync(0xffffffffu, key_lim >= kKeys);
          ptx::mbar_wait(WB(i, S_FULL), cc & 1);
          ATTN_TRACE(i, 43);
          ptx::tc_fence_after();
          uint32_t s[kKeys];
#pragma unroll
          for (int q = 0; q < kKeys / 32; ++q)
            ptx::tmem_ld_32x32b_x32(tS + q * 32, *reinterpret_cast<uint32_t(*)[32]>(s + q * 32));
          ptx::tmem_ld_wait();
          ptx::tc_fence_before();
          ptx::mbar_arrive(WB(i, S_FREE));
          if (!full) {
#pragma unroll
            for (int e = 0; e < kKeys; ++e)
              if (e >= key_lim) s[e] = __float_as_uint(-INFINITY);
          }
          float mx[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) mx[q] = __uint_as_float(s[q]);
#pragma unroll
          for (int e = 8; e < kKeys; ++e) mx[e & 7] = fmaxf(mx[e & 7], __uint_as_float(s[e]));
          const float cmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                   fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
          const float cm = cmax * sl2;
          const bool raise = cm - m > kRescaleThreshold;
          const float m_new = raise ? cm : m;
          const float alpha = raise ? ptx::exp2_approx(m - m_new) : 1.f;
          m = m_new;
          const uint64_t sl2x2 = f2::make(sl2, sl2);
          const uint64_t nm2 = f2::make(-m, -m);
          uint64_t ps2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
          for (int e = 0; e < kKeys; e += 2) {
            const uint64_t x = f2::fma(f2::make(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), sl2x2, nm2);
            uint64_t pr;
            if ((attn::kPolyMask >> ((e >> 1) & 7)) & 1) {
              pr = attn::exp2_poly3_x2(x);
            } else {
              float x0, x1;
              f2::split(x, x0, x1);
              pr = f2::make(ptx::exp2_approx(x0), ptx::exp2_approx(x1));
            }
            ps2[(e >> 1) & 3] = f2::add(ps2[(e >> 1) & 3], pr);
            float p0, p1;
            f2::split(pr, p0, p1);
            s[e / 2] = pack_bf16x2(p0, p1);
          }
          float psum;
          {
            float a0, a1;
            f2::split(f2::add(f2::add(ps2[0], ps2[1]), f2::add(ps2[2], ps2[3])), a0, a1);
            psum = a0 + a1;
          }
          l = l * alpha + psum;
          if (c > 0) {
            ptx::mbar_wait(WB(i, O_FULL), (cc - 1) & 1);  // PV_{c-1} done: P and O may change
            ptx::tc_fence_after();
            if (__any_sync(0xffffffffu, alpha != 1.f)) {
              uint32_t ov[DH];
#pragma unroll
              for (int q = 0; q < DH / 32; ++q)
                ptx::tmem_ld_32x32b_x32(tO + q * 32, *reinterpret_cast<uint32_t(*)[32]>(ov + q * 32));
              ptx::tmem_ld_wait();
              const uint64_t al2 = f2::make(alpha, alpha);
#pragma unroll
              for (int e = 0; e < DH; e += 2) {
                float o0, o1;
                f2::split(f2::mul(f2::make(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1])), al2), o0, o1);
                ov[e] = __float_as_uint(o0);
                ov[e + 1] = __float_as_uint(o1);
              }
#pragma unroll
              for (int q = 0; q < DH / 16; ++q)
                ptx::tmem_st_32x32b_x16(tO + q * 16, *reinterpret_cast<uint32_t(*)[16]>(ov + q * 16));
            }
          }
#pragma unroll
          for (int q = 0; q < kKeys / 32; ++q)
            ptx::tmem_st_32x32b_x16(tP + q * 16, *reinterpret_cast<uint32_t(*)[16]>(s + q * 16));
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
          ptx::mbar_arrive(WB(i, P_FULL));
          ATTN_TRACE(i, 44);
        }
        // out = (O + exp2(s_self - m) v_self) / l; H = 0 gives out = v_self
        float o[DH];
        if (un.nk > 0) {
          ptx::mbar_wait(WB(i, O_FULL), (cc - 1) & 1);
          ATTN_TRACE(i, 45);
          ptx::tc_fence_after();
          uint32_t ov[DH];
#pragma unroll
          for (int q = 0; q < DH / 32; ++q)
            ptx::tmem_ld_32x32b_x32(tO + q * 32, *reinterpret_cast<uint32_t(*)[32]>(ov + q * 32));
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < DH; ++e) o[e] = __uint_as_float(ov[e]);
          ptx::tc_fence_before();
        } else {
#pragma unroll
          for (int e = 0; e < DH; ++e) o[e] = 0.f;
        }
        const float w_self = ptx::exp2_approx(m_self - m);
#pragma unroll
        for (int c8 = 0; c8 < DH / 8; ++c8) {
          const uint4 vv = *reinterpret_cast<const uint4*>(stage + ptx::sw128_offset(row, c8 * 16));
          const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vv);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 v = __bfloat1622float2(v2[e]);
            float& oa = o[c8 * 8 + 2 * e];
            float& ob = o[c8 * 8 + 2 * e + 1];
            f2::split(f2::fma(f2::make(w_self, w_self), f2::make(v.x, v.y), f2::make(oa, ob)), oa, ob);
          }
        }
        {
          // fold 1 / l in here, so the stores below only pack
          const float inv = 1.f / l;
          const uint64_t inv2 = f2::make(inv, inv);
#pragma unroll
          for (int e = 0; e < DH; e += 2) f2::split(f2::mul(f2::make(o[e], o[e + 1]), inv2), o[e], o[e + 1]);
        }
        const int q_row0 = cand_row0 + un.r * a.c_bkt + t * kRows;
        if (a.store_tma) {
#pragma unroll
          for (int c8 = 0; c8 < DH / 8; ++c8) {
            uint4 w;
            w.x = pack_bf16x2(o[c8 * 8 + 0], o[c8 * 8 + 1]);
            w.y = pack_bf16x2(o[c8 * 8 + 2], o[c8 * 8 + 3]);
            w.z = pack_bf16x2(o[c8 * 8 + 4], o[c8 * 8 + 5]);
            w.w = pack_bf16x2(o[c8 * 8 + 6], o[c8 * 8 + 7]);
            *reinterpret_cast<uint4*>(stage + ptx::sw128_offset(row, c8 * 16)) = w;
          }
          ptx::fence_proxy_async_smem();
          asm volatile("bar.sync %0, 128;" ::"r"(1 + i) : "memory");
          if (row == 0) {
            ptx::tma_store_3d(&tm_out, stage, un.h * DH, q_row0, un.g);
            ptx::tma_store_commit();
          }
          store_pending = true;
        } else {
          if (row_ok) {
            __nv_bfloat16* dst = a.out + un.g * a.out_gstride + static_cast<long long>(q_row0 + row) * a.out_ld +
                                 un.h * DH;
#pragma unroll
            for (int c8 = 0; c8 < DH / 8; ++c8) {
              uint4 w;
              w.x = pack_bf16x2(o[c8 * 8 + 0], o[c8 * 8 + 1]);
              w.y = pack_bf16x2(o[c8 * 8 + 2], o[c8 * 8 + 3]);
              w.z = pack_bf16x2(o[c8 * 8 + 4], o[c8 * 8 + 5]);
              w.w = pack_bf16x2(o[c8 * 8 + 6], o[c8 * 8 + 7]);
              reinterpret_cast<uint4*>(dst)[c8] = w;
            }
          }
          // every row read its V_self before any row's next-job epilogue rewrites the staging
          asm volatile("bar.sync %0, 128;" ::"r"(1 + i) : "memory");
        }
        ATTN_TRACE(i, 46);
        ++nj;
      }
    }
    if (row == 0) ptx::tma_store_wait<0>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem);
  }
}

}  // namespace flame
