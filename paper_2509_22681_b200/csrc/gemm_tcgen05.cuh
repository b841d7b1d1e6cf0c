// Persistent, warp-specialised tcgen05 GEMM for the FLAME projections and FFN.
//
//   D[g][m][n] = epi( sum_k A[g][m][k] * W[g][n][k] )      (bf16 in, fp32 accumulate)
//
// A rows are token rows (history / candidate rows of one Climber block), W is
// the block's weight stored transposed ([out, in], K-major) so both operands
// are K-major and stream through TMA with a 128-byte swizzle.  One CTA per SM
// loops over 128 x BN output tiles; roles:
//   warp 0      : TMA producer (A + W tiles into a kStages-deep smem ring)
//   warp 1      : MMA issuer (one thread issues tcgen05.mma, commits to mbarriers)
//   warp 2      : TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..11 : epilogue — two warps per TMEM lane quadrant, each taking every
//                 other 32-column chunk: tcgen05.ld -> bias / tanh-GELU / fp32
//                 residual in registers -> swizzled smem box -> TMA bulk store
// The epilogue of tile i overlaps the MMAs of tile i+1 through the second
// accumulator buffer.  The K loop order is fixed per row, so a row's result is
// independent of which tile / batch position it lands in (batch invariance:
// chunked == unchunked, duplicate candidates give identical scores).
#pragma once
#include "ptx.cuh"
#include "common.cuh"

namespace flame {

struct GemmEpilogue {
  void* out;              // bf16 or fp32 [G][M][ldo]
  long long out_ld;       // elements
  long long out_gstride;  // elements per group
  int out_col0;           // column offset inside the output row
  const float* bias;      // [G][N] (fp32), may be null
  long long bias_gstride;
  const float* resid;     // [G][M][ld] fp32 residual, may be null
  const __nv_bfloat16* resid_b;  // same, bf16 (EPI_RESID_BF16)
  long long resid_ld;
  long long resid_gstride;
  const float* rowscale;  // [G][M] per-row factor (folded LayerNorm rstd), may be null
  long long rowscale_gstride;
  const float* dot_w;     // [N][4] fp32: row-dot epilogue weights (expert W2, tasks padded to 4)
  int dot_n;              // outputs per row of the row-dot epilogue (num_tasks <= 4)
  // EPI_STATS (producer of a folded LayerNorm): bf16 copy of the output + per-row
  // partial (sum, sum of squares) over this tile's columns
  __nv_bfloat16* out2;    // [G][M][out2_ld]
  long long out2_ld, out2_gstride;
  float* stats;           // [G][M][2 * n_tiles][2]
  long long stats_gstride;
  // EPI_LNSTATS (consumer): LN(x) W = rstd (x W' - mean u) + c, mean / rstd from the
  // producer's partials (stats_parts per row, fixed-order sum over d_true columns)
  const float* lnstats;   // [G][M][stats_parts][2]
  long long lnstats_gstride;
  int stats_parts;
  int d_true;
  const float* colsum;    // [G][N] u = gamma . W (column sums of the folded weight)
  long long colsum_gstride;
  int M, N;               // logical bounds of this problem
};

// Epilogue stages, applied in this order: ROWSCALE (acc *= rowscale[row]),
// BIAS, GELU, RESID, then either a store (bf16 / fp32) or ROWDOT: per row the
// partial dot of the tile's columns with dot_w, written to
// out[row][n_tile * 2 + half][t] (fp32) and reduced by a fixed-order combine.
enum : int {
  EPI_BIAS = 1,
  EPI_GELU = 2,
  EPI_RESID = 4,
  EPI_OUT_F32 = 8,
  EPI_ROWSCALE = 16,
  EPI_ROWDOT = 32,
  EPI_STATS = 64,
  EPI_LNSTATS = 128,
  EPI_RESID_BF16 = 256,
};

namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle row
constexpr int kSmemBudget = 227 * 1024;

// Per-variant configuration: heavy epilogues (GELU, folded LayerNorm) get 12
// epilogue warps (3 per TMEM lane quadrant) so they keep up with the MMAs; the
// smem ring gets whatever the staging boxes leave (up to 6 stages).
template <int BN, int EPI>
struct Cfg {
  static constexpr bool kHeavy = (EPI & (EPI_GELU | EPI_LNSTATS | EPI_STATS)) != 0;
  static constexpr int kEpiWarps = kHeavy ? 12 : 8;
  static constexpr int kThreads = 128 + 32 * kEpiWarps;
  // STATS with an fp32 primary output also emits a bf16 copy (second TMA store)
  static constexpr bool kDual = (EPI & EPI_STATS) != 0 && (EPI & EPI_OUT_F32) != 0;
  static constexpr int kBoxBytes = 32 * 32 * 4 + (kDual ? 32 * 32 * 2 : 0);
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kFixed = kEpiWarps * kBoxBytes + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int kStagesFit = (kSmemBudget - kFixed) / kStageBytes;
  static constexpr int kStages = kStagesFit > 6 ? 6 : kStagesFit;
  static_assert(kStages >= 2, "GEMM smem ring too shallow");
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + kFixed;
};

}  // namespace gemm

template <int BN, int EPI>
__global__ void __launch_bounds__(gemm::Cfg<BN, EPI>::kThreads, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2,
                      int num_k_blocks, int m_tiles, int n_tiles, int groups, int a_shared, GemmEpilogue ep) {
  using C = gemm::Cfg<BN, EPI>;
  constexpr int kEpiWarps = C::kEpiWarps;
  constexpr int kEpiPerQuad = kEpiWarps / 4;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t pad = ((raw_addr + 1023) & ~1023u) - raw_addr;
  uint8_t* smem = smem_raw + pad;
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * C::kABytes;
  uint8_t* smem_box = smem + kStages * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_box + kEpiWarps * C::kBoxBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tmem_full = bars + 2 * kStages;
  uint64_t* tmem_empty = bars + 2 * kStages + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    ptx::tma_prefetch_desc(&tmO);
    if (C::kDual) ptx::tma_prefetch_desc(&tmO2);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tmem_full[s], 1);
      ptx::mbar_init(&tmem_empty[s], kEpiWarps);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_base_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  const int total_tiles = groups * m_tiles * n_tiles;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // whole warp walks the schedule (operands stay warp-uniform); one lane issues
    const bool leader = ptx::elect_one();
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int n_blk = tile % n_tiles;
      const int m_blk = (tile / n_tiles) % m_tiles;
      const int g = tile / (n_tiles * m_tiles);
      const int ga = a_shared ? 0 : g;
      for (int kb = 0; kb < num_k_blocks; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (leader) {
          ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          ptx::tma_load_3d(smem_a + stage * C::kABytes, &tmA, &full[stage], kb * gemm::BK,
                           m_blk * gemm::BM, ga);
          ptx::tma_load_3d(smem_b + stage * C::kBBytes, &tmB, &full[stage], kb * gemm::BK,
                           n_blk * BN, g);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer
    const bool leader = ptx::elect_one();
    constexpr uint32_t idesc = ptx::make_idesc_bf16(gemm::BM, BN, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      ptx::mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < num_k_blocks; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t a_addr = ptx::smem_u32(smem_a + stage * C::kABytes);
        const uint32_t b_addr = ptx::smem_u32(smem_b + stage * C::kBBytes);
        if (leader) {
#pragma unroll
          for (int k = 0; k < gemm::BK / 16; ++k) {
            const uint64_t ad = ptx::make_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = ptx::make_desc_sw128(b_addr + k * 32, 16, 1024);
            ptx::mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          ptx::mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (leader) ptx::mma_commit(&tmem_full[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    // ----------------------------------------------------------- epilogue
    constexpr bool kF32 = (EPI & EPI_OUT_F32) != 0;
    const int ew = warp - 4;
    const int wq = warp & 3;    // TMEM lane quadrant this warp may access
    const int half = ew >> 2;   // which interleaved share of the 32-column chunks
    uint8_t* box = smem_box + ew * C::kBoxBytes;
    uint8_t* box2 = box + 32 * 32 * 4;  // bf16 side-output box (kDual)
    const bool epi_leader = ptx::elect_one();  // same lane issues stores and waits (bulk groups are per thread)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int n_blk = tile % n_tiles;
      const int m_blk = (tile / n_tiles) % m_tiles;
      const int g = tile / (n_tiles * m_tiles);
      ptx::mbar_wait(&tmem_full[acc], acc_phase);
      ptx::tc_fence_after();
      const int row0 = m_blk * gemm::BM + wq * 32;
      // rows past M are clipped by the TMA store; clamp their residual reads
      const int row = min(row0 + lane, ep.M - 1);
      const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(wq * 32) << 16);
      float rs = (EPI & EPI_ROWSCALE) ? ep.rowscale[g * ep.rowscale_gstride + row] : 1.f;
      float ln_mean = 0.f;
      if constexpr ((EPI & EPI_LNSTATS) != 0) {
        // combine the producer's per-tile (sum, sumsq) partials in fixed order
        const float2* pst = reinterpret_cast<const float2*>(ep.lnstats + g * ep.lnstats_gstride) +
                            static_cast<long long>(row) * ep.stats_parts;
        float s1 = 0.f, s2 = 0.f;
        for (int k = 0; k < ep.stats_parts; ++k) {
          const float2 p = pst[k];
          s1 += p.x;
          s2 += p.y;
        }
        ln_mean = s1 / ep.d_true;
        rs = rsqrtf(fmaxf(s2 / ep.d_true - ln_mean * ln_mean, 0.f) + 1e-5f);
      }
      float st_sum = 0.f, st_sq = 0.f;
      float dot[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
      for (int c = half; c < BN / 32; c += kEpiPerQuad) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
        ptx::tmem_ld_wait();
        const int col0 = n_blk * BN + c * 32;
        if (col0 >= ep.N) continue;  // warp-uniform
        float v[32];
        if constexpr ((EPI & EPI_LNSTATS) != 0) {
          const float* u = ep.colsum + g * ep.colsum_gstride + col0;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 uu = __ldg(reinterpret_cast<const float4*>(u + j));
            v[j + 0] = (__uint_as_float(r[j + 0]) - ln_mean * uu.x) * rs;
            v[j + 1] = (__uint_as_float(r[j + 1]) - ln_mean * uu.y) * rs;
            v[j + 2] = (__uint_as_float(r[j + 2]) - ln_mean * uu.z) * rs;
            v[j + 3] = (__uint_as_float(r[j + 3]) - ln_mean * uu.w) * rs;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * rs;
        }
        epilogue_math<EPI, 32, true>(v, ep, g, row, col0);
        if constexpr ((EPI & EPI_STATS) != 0) {
          // padded columns are exactly 0 and add nothing to the sums
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            st_sum += v[j];
            st_sq = fmaf(v[j], v[j], st_sq);
          }
        }
        if constexpr ((EPI & EPI_ROWDOT) != 0) {
          // partial dot with dot_w over this chunk (fixed order; cols >= N have dot_w rows
          // zero-padded by the caller)
          // dot_w is [N][4] (tasks zero-padded to 4): one broadcast float4 load per column
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(ep.dot_w) + (col0 + j));
            dot[0] = fmaf(v[j], w.x, dot[0]);
            dot[1] = fmaf(v[j], w.y, dot[1]);
            dot[2] = fmaf(v[j], w.z, dot[2]);
            dot[3] = fmaf(v[j], w.w, dot[3]);
          }
        } else {
          if (epi_leader) ptx::tma_store_wait_read<0>();  // staging boxes free again
          __syncwarp();
          stage_row32<kF32>(box, lane, v);
          if constexpr (C::kDual) stage_row32<false>(box2, lane, v);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (epi_leader) {
            ptx::tma_store_3d(&tmO, box, ep.out_col0 + col0, row0, g);
            if constexpr (C::kDual) ptx::tma_store_3d(&tmO2, box2, col0, row0, g);
            ptx::tma_store_commit();
          }
        }
      }
      if constexpr ((EPI & EPI_STATS) != 0) {
        if (row0 + lane < ep.M) {
          float2* dst = reinterpret_cast<float2*>(ep.stats + g * ep.stats_gstride) +
                        static_cast<long long>(row0 + lane) * (kEpiPerQuad * n_tiles) + n_blk * kEpiPerQuad + half;
          *dst = make_float2(st_sum, st_sq);
        }
      }
      if constexpr ((EPI & EPI_ROWDOT) != 0) {
        if (row0 + lane < ep.M) {
          float* dst = reinterpret_cast<float*>(ep.out) +
                       (static_cast<long long>(row0 + lane) * (kEpiPerQuad * n_tiles) + n_blk * kEpiPerQuad + half) * ep.dot_n;
          for (int t = 0; t < ep.dot_n; ++t) dst[t] = dot[t];
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tmem_empty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (epi_leader) ptx::tma_store_wait<0>();
    __syncwarp();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

}  // namespace flame
