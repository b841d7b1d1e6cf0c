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
// accumulator buffer.
// Launched as CTA pairs (2-CTA clusters, cta_group::2): the pair computes a
// 256 x BN tile with M = 256 MMAs issued by the even CTA.  Each CTA loads its
// own 128 A rows and HALF of the W tile into its own smem; the tensor core reads
// both CTAs' operands, and each CTA's TMEM receives its own 128 rows.  So the
// L2->SM operand traffic per CTA is (BM + BN/2) rows per k-block instead of
// (BM + BN) (the GEMMs here are L2-bandwidth-bound at 128 x 256 tiles; ncu shows
// TMA multicast does not reduce L2 traffic at cluster size 2, the pair MMA does).
// Every TMA of the pair completes on the even CTA's full barrier; MMA commits
// multicast to both CTAs' empty / tmem_full barriers; both CTAs' epilogue warps
// release an accumulator on the even CTA's tmem_empty barrier.  The K loop
// order is fixed per row, so a row's result is independent of which tile /
// batch position it lands in (batch invariance: chunked == unchunked,
// duplicate candidates give identical scores).
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
  // EPI_GATED (FFN W2 of the last layer + gated fusion): per group g the tile's
  // X2 = acc + b2 + X1 is folded into sum_g sigmoid(X2 * gate_w[g] + gate_b[g]) * X2
  // (kept in TMEM across the groups, which one CTA walks in order); only the sum
  // reaches HBM, as the fp32 operand of the tf32 expert GEMM ([M][N])
  const float* gate_w;    // [G][N]
  const float* gate_b;    // [G][N]
  // balanced gated schedule (BN = 256, sum in registers): a cluster may end inside
  // a chain of groups and hand its running sum to the next cluster, which finishes
  // that chain last.  Scratch per (cluster, CTA, epilogue warp): the sum rows
  // (32 lanes x kMyChunks x 32 fp32) and a flag (0 / 1, reset by the consumer).
  // Null: whole chains per cluster.
  float* gpart;
  int* gflag;
  // device-side active row count (DSO executors): rows >= *m_active * rows_per_slot
  // are unused slots and their tiles are skipped (null: all M rows)
  const int* m_active;
  int rows_per_slot;
  int M, N;               // logical bounds of this problem
  int g_inner;            // tile order: 1 = group index fastest (operand / residual shared by all groups)
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
  EPI_GATED = 512,
  EPI_TF32 = 2048,  // operands are fp32, multiplied as tf32 (kind::tf32): 32 K-elements per 128-byte row
};

// Debug-only event trace of CTA 0 (flame_debug_gemm_trace): slot 0 = MMA issuer,
// slot 1 = epilogue warp 0, slot 2 = epilogue warp 4, slot 3 = producer;
// entry = clock64 << 8 | code.  One writer per slot, no atomics.
__device__ unsigned long long* g_gemm_trace = nullptr;
#ifdef FLAME_DEBUG_TRACE
#define GEMM_TRACE(slot, code)                                                                  \
  do {                                                                                          \
    if (g_gemm_trace != nullptr && blockIdx.x == 0 && lane == 0) {                              \
      if (gtrace_k < 4096) g_gemm_trace[(slot) * 4096 + gtrace_k] = (clock64() << 8) | (code);  \
      ++gtrace_k;                                                                               \
    }                                                                                           \
  } while (0)
#else
// Production builds keep a compiler memory barrier at the trace sites of the MMA
// issuer (slot 0: after the accumulator wait, at the first k-block, after the
// commit) and of the producer (slot 3: after each stage's empty wait).  Measured:
// without it ptxas schedules the BN = 256 gated-fusion W2 into 0.51 ms at cfg3,
// with it 0.445 ms (the debug-trace build, whose trace sites act as the same
// barriers, had shown the gap; profiles/r02h/sched_fence_ab).  FLAME_PROBE_MASK
// (bit 0 MMA issuer, 1-2 epilogue, 3 producer) overrides it for A/B builds.
#ifndef FLAME_PROBE_MASK
#define FLAME_PROBE_MASK 9
#endif
#define GEMM_TRACE(slot, code)                                        \
  do {                                                                \
    (void)gtrace_k;                                                   \
    if ((FLAME_PROBE_MASK >> (slot)) & 1) asm volatile("" ::: "memory"); \
  } while (0)
#endif

namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle row
constexpr int kSmemBudget = 227 * 1024;

// Per-variant configuration.  The epilogue does its arithmetic on fp32 pairs
// (fma.rn.f32x2: twice the FMA-pipe throughput of scalar FFMA) and prefetches
// the next TMEM chunk while processing the current one, so two warps per TMEM
// lane quadrant keep up with the MMAs (FLAME_GEMM_HEAVY_WARPS=12 restores three
// for the GELU / LayerNorm variants).  Per-column vectors (bias, folded-LN
// column sums u) of bf16-output variants are staged once per tile into a
// per-warp smem slice and read back as broadcasts.  The smem ring gets whatever
// the staging boxes leave (up to 6 stages).
#ifndef FLAME_GEMM_OUT_BOXES
#define FLAME_GEMM_OUT_BOXES 0
#endif
#ifndef FLAME_GEMM_HEAVY_WARPS
#define FLAME_GEMM_HEAVY_WARPS 8
#endif
// epilogue warps of a variant: FLAME_GEMM_HEAVY_WARPS for the bf16 GELU epilogues,
// 8 otherwise (host code sizes the row-partial buffers with the same rule)
__host__ __device__ constexpr int gemm_epi_warps(int epi) {
  return ((epi & EPI_GELU) != 0 && (epi & EPI_OUT_F32) == 0) ? FLAME_GEMM_HEAVY_WARPS : 8;
}
template <int BN, int EPI, int kCG>
struct Cfg {
  static constexpr bool kHeavy = (EPI & (EPI_GELU | EPI_LNSTATS | EPI_STATS)) != 0;
  static constexpr int kEpiWarps = gemm_epi_warps(EPI);
  static constexpr int kEpiPerQuad = kEpiWarps / 4;
  static constexpr int kThreads = 128 + 32 * kEpiWarps;
  static constexpr bool kF32 = (EPI & EPI_OUT_F32) != 0;
  static constexpr bool kRowDot = (EPI & EPI_ROWDOT) != 0;
  static constexpr bool kGated = (EPI & EPI_GATED) != 0;
  static_assert(!kGated || ((BN == 128 || BN == 256) && !kF32 && (EPI & EPI_RESID_BF16) != 0),
                "gated-fusion epilogue: BN = 128 / 256, bf16 output, bf16 residual");
  // gated fusion at BN = 256: both TMEM halves hold accumulators, so the running
  // sum over groups lives in the epilogue threads' registers (kMyChunks x 32 fp32
  // per thread), paid for by setmaxnreg (kRegsEpi for the epilogue warpgroups,
  // kRegsCtl for the producer / MMA warpgroup; together the launch allocation)
  static constexpr bool kRegSum = kGated && BN == 256;
  static constexpr int kRegsEpi = 232, kRegsCtl = 40;
  // STATS with an fp32 primary output, and the gated sum (hi + lo halves), also
  // stage a second bf16 box
  static constexpr bool kDual = (EPI & EPI_STATS) != 0 && kF32;
  // staging slots per epilogue warp ([out box | bf16 side box]); with two, a
  // chunk's staging does not wait for the previous chunk's TMA store to read smem.
  // Measured at cfg3: pays for the GELU (FFN W1) epilogue (0.533 -> 0.497 ms),
  // costs the others a smem ring stage (QKV 0.347 -> 0.394 ms), so by default
  // (FLAME_GEMM_OUT_BOXES = 0) only the bf16 GELU variants get two.
  static constexpr int kOutBoxes =
      FLAME_GEMM_OUT_BOXES != 0 ? (FLAME_GEMM_OUT_BOXES == 2 && !kF32 ? 2 : 1)
                                : ((EPI & EPI_GELU) != 0 && !kF32 && !kRowDot ? 2 : 1);
  // (the gated-fusion sum leaves as fp32: the tf32 expert GEMM reads it)
  static constexpr int kOutBoxBytes = kRowDot ? 0 : 32 * 32 * ((kF32 || kGated) ? 4 : 2);
  static constexpr int kSlotBytes = kOutBoxBytes + (kDual ? 32 * 32 * 2 : 0);
  static constexpr int kBoxBytes = kOutBoxes * kSlotBytes;
  // chunks of 32 columns per warp and the per-warp column-vector slices
  static constexpr int kChunks = BN / 32;
  static constexpr int kMyChunks = (kChunks + kEpiPerQuad - 1) / kEpiPerQuad;
  static constexpr bool kBiasSmem = (EPI & EPI_BIAS) != 0 && !kF32;
  static constexpr bool kUSmem = (EPI & EPI_LNSTATS) != 0;
  static constexpr int kCvecs = (kBiasSmem ? 1 : 0) + (kUSmem ? 1 : 0) + (kGated ? 2 : 0);
  static constexpr int kCvecBytes = kCvecs * kMyChunks * 32 * 4;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = (BN / kCG) * BK * 2;  // this CTA's share of the W tile
  static constexpr int kStageBytes = kABytes + kBBytes;
  // residuals are TMA-loaded as 32x32 boxes (fp32: SW128, bf16: SW64; row-per-lane
  // global loads would cost one L1 wavefront per 16 bytes and expose their full
  // latency in every chunk), two boxes in flight per warp
  static constexpr bool kResidTma = (EPI & EPI_RESID) != 0;
  static constexpr int kResidBox = 32 * 32 * ((EPI & EPI_RESID_BF16) != 0 ? 2 : 4);
  static constexpr int kResidBytes = kResidTma ? 2 * kResidBox : 0;
  static constexpr int kFixed = kEpiWarps * (kBoxBytes + kCvecBytes + kResidBytes) + 1024 /*align*/ + 512 /*barriers*/;
  static constexpr int kStagesFit = (kSmemBudget - kFixed) / kStageBytes;
#ifndef FLAME_GEMM_MAX_STAGES
#define FLAME_GEMM_MAX_STAGES 6
#endif
  static constexpr int kStages = kStagesFit > FLAME_GEMM_MAX_STAGES ? FLAME_GEMM_MAX_STAGES : kStagesFit;
  static_assert(kStages >= 2, "GEMM smem ring too shallow");
  // two accumulators (+ the gated running sum at columns [2 BN, 3 BN))
  // accumulator ring: as many BN-column buffers as TMEM holds (BN = 128: four), so
  // the MMAs can run several tiles ahead of a latency-bound epilogue
  static constexpr int kAcc = kGated ? 2 : 512 / BN;
  static constexpr int kTmemCols = kGated ? 512 : kAcc * BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + kFixed;
};

}  // namespace gemm

template <int BN, int EPI, int kCG>
__global__ void __launch_bounds__(gemm::Cfg<BN, EPI, kCG>::kThreads, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2,
                      const __grid_constant__ CUtensorMap tmR, int num_k_blocks, int m_tiles_max, int n_tiles, int groups, int a_shared, GemmEpilogue ep) {
  using C = gemm::Cfg<BN, EPI, kCG>;
  constexpr int kEpiWarps = C::kEpiWarps;
  constexpr bool kTF32 = (EPI & EPI_TF32) != 0;
  constexpr int kBKe = kTF32 ? 32 : gemm::BK;  // K elements per 128-byte smem row
  constexpr int kEpiPerQuad = kEpiWarps / 4;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t pad = ((raw_addr + 1023) & ~1023u) - raw_addr;
  uint8_t* smem = smem_raw + pad;
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * C::kABytes;
  uint8_t* smem_box = smem + kStages * C::kStageBytes;
  uint8_t* smem_cvec = smem_box + kEpiWarps * C::kBoxBytes;
  uint8_t* smem_resid = smem_cvec + kEpiWarps * C::kCvecBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_resid + kEpiWarps * C::kResidBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tmem_full = bars + 2 * kStages;               // [kAcc]
  uint64_t* tmem_empty = tmem_full + C::kAcc;             // [kAcc]
  uint64_t* resid_full = tmem_empty + C::kAcc;            // [kEpiWarps][2]
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(resid_full + 2 * kEpiWarps);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  // CTA pair (kCG = 2): the two CTAs of a cluster own vertically adjacent 128-row
  // halves of a 256-row tile; the even CTA issues cta_group::2 MMAs for both
  constexpr int ncl = kCG;
  const int crank = kCG == 2 ? static_cast<int>(ptx::cluster_ctarank()) : 0;
  int m_tiles = m_tiles_max;
  if (ep.m_active != nullptr) {
    const int rows = __ldg(ep.m_active) * ep.rows_per_slot;
    m_tiles = max(1, min(m_tiles_max, (rows + gemm::BM - 1) / gemm::BM));
  }
  const int m_pairs = (m_tiles + ncl - 1) / ncl;
  const int cid = blockIdx.x / ncl;
  const int nclusters = gridDim.x / ncl;
  const int total_tiles = groups * m_pairs * n_tiles;
  // Balanced gated schedule: the chains of G group tiles laid end to end and cut
  // into nclusters equal ranges.  A range may end inside a chain (its TAIL piece:
  // groups [0, e % G) of chain e / G, worked FIRST, its running sum handed over
  // through ep.gpart) and begin inside one (its HEAD piece: groups [b % G, G) of
  // chain b / G, worked LAST, continuing the previous cluster's sum); whole chains
  // in between.  The fp32 sum still runs over the groups in order.  Chains are
  // numbered n-block-major, so clusters k and k + S / n_tiles work the same rows
  // (the shared A tiles) at the same time and those re-reads hit L2.
  bool bal = false;
  int bt_nt = 0, bt_st = 0, bt_sa = 0, bt_nf = 0, bt_nh = 0, bt_sh = 0, bt_gh = 0;
  if constexpr (C::kRegSum) {
    const long long T = static_cast<long long>(groups) * m_pairs * n_tiles;
    if (ep.gpart != nullptr && T / nclusters >= 2 * groups) {
      bal = true;
      const int b = static_cast<int>(cid * T / nclusters), e = static_cast<int>((cid + 1) * T / nclusters);
      bt_nt = e % groups;
      bt_st = e / groups;
      bt_sa = (b + groups - 1) / groups;
      bt_nf = (e / groups - bt_sa) * groups;
      bt_gh = b % groups;
      bt_nh = bt_gh != 0 ? groups - bt_gh : 0;
      bt_sh = b / groups;
    }
  }
  // tile -> (group, m pair, n block).  Group-fastest order when every group reads
  // the same A rows or residual tile: the G consecutive tiles hit it in L2.
  auto decode = [&](int t, int& g, int& mp, int& nb) {
    if (C::kRegSum && bal) {
      g = t % groups;
      nb = (t / groups) / m_pairs;
      mp = (t / groups) % m_pairs;
    } else if (C::kGated || ep.g_inner) {
      g = t % groups;
      nb = (t / groups) % n_tiles;
      mp = t / (groups * n_tiles);
    } else {
      nb = t % n_tiles;
      mp = (t / n_tiles) % m_pairs;
      g = t / (n_tiles * m_pairs);
    }
  };
  // the it-th tile of this cluster (>= total_tiles when done).  Gated fusion: a
  // cluster owns whole (m pair, n block) super tiles and walks their groups in order
  auto tile_at = [&](int it) -> int {
    if constexpr (C::kGated) {
      if (bal) {
        if (it < bt_nt) return bt_st * groups + it;
        const int j = it - bt_nt;
        if (j < bt_nf) return bt_sa * groups + j;
        return j - bt_nf < bt_nh ? bt_sh * groups + bt_gh + (j - bt_nf) : total_tiles;
      }
      const int st = cid + (it / groups) * nclusters;
      return st < m_pairs * n_tiles ? st * groups + it % groups : total_tiles;
    } else {
      return cid + it * nclusters;
    }
  };

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    ptx::tma_prefetch_desc(&tmO);
    if (C::kDual) ptx::tma_prefetch_desc(&tmO2);
    if (C::kResidTma) ptx::tma_prefetch_desc(&tmR);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::kAcc; ++s) {
      ptx::mbar_init(&tmem_full[s], 1);
      ptx::mbar_init(&tmem_empty[s], kEpiWarps * kCG);  // both CTAs' epilogue warps
    }
    if (C::kResidTma)
      for (int s = 0; s < 2 * kEpiWarps; ++s) ptx::mbar_init(&resid_full[s], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg<C::kTmemCols, kCG>(tmem_base_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  if constexpr (kCG > 1) ptx::cluster_sync();  // peer barriers / TMEM ready before any pair MMA
  // PDL: the prologue above overlapped the previous kernel's tail; its outputs
  // (A operand, residual, row statistics) are read only after this
  ptx::griddep_wait();
  ptx::griddep_launch();
#ifdef FLAME_DEBUG_TRACE
  // per-CTA start / end (globaltimer ns) after the 4 x 4096 per-event slots
  if (g_gemm_trace != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemm_trace[4 * 4096 + 2 * blockIdx.x] = t;
  }
#endif
  static_assert(!C::kRegSum || (C::kThreads == 384 && 128 * C::kRegsCtl + 256 * C::kRegsEpi <= 384 * 168),
                "setmaxnreg budget above the launch allocation");

  // warpgroup 0: producer (warp 0), MMA issuer (warp 1 of the even CTA), TMEM
  // allocator (warp 2); warpgroups 1-2: epilogue.  setmaxnreg is executed per
  // warpgroup, before the warps split into roles
  if (warp < 4) {
  if constexpr (C::kRegSum) ptx::setmaxnreg_dec<C::kRegsCtl>();
  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // whole warp walks the schedule (operands stay warp-uniform); one lane issues
    const bool leader = ptx::elect_one();
    int stage = 0;
    uint32_t phase = 0;
    unsigned gtrace_k = 0;
    for (int it = 0, tile = tile_at(0); tile < total_tiles; tile = tile_at(++it)) {
      int g, mp, n_blk;
      decode(tile, g, mp, n_blk);
      // the odd tail CTA of a cluster recomputes the last tile; its stores fall past M
      const int m_blk = min(mp * ncl + crank, m_tiles - 1);
      const int ga = a_shared ? 0 : g;
      for (int kb = 0; kb < num_k_blocks; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        GEMM_TRACE(3, 7);
#ifdef FLAME_DBG_GEMM_NO_TMA
        if (leader) ptx::mbar_arrive(&full[stage]);
        if (false) {
#else
        if (leader) {
#endif
          if constexpr (kCG == 1) {
            ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
            ptx::tma_load_3d(smem_a + stage * C::kABytes, &tmA, &full[stage], kb * kBKe,
                             m_blk * gemm::BM, ga);
            ptx::tma_load_3d(smem_b + stage * C::kBBytes, &tmB, &full[stage], kb * kBKe,
                             n_blk * BN, g);
          } else {
            // this CTA's A rows and its half of the W tile, both completing on the
            // even CTA's full barrier (which expects the pair's bytes)
            if (crank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
            const uint32_t fb = ptx::mapa_shared(ptx::smem_u32(&full[stage]), 0);
            ptx::tma_load_3d_cg2(smem_a + stage * C::kABytes, &tmA, fb, kb * kBKe, m_blk * gemm::BM, ga);
            ptx::tma_load_3d_cg2(smem_b + stage * C::kBBytes, &tmB, fb, kb * kBKe,
                                 n_blk * BN + crank * (BN / 2), g);
          }
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
    if constexpr (kCG > 1) {
      // drain: every stage released by the pair's MMAs, so no multicast arrival
      // is still in flight towards this CTA when it exits
      for (int i = 0; i < kStages; ++i) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && crank == 0) {
    // --------------------------------------------------------- MMA issuer
    const bool leader = ptx::elect_one();
    constexpr uint32_t idesc = kTF32 ? ptx::make_idesc_tf32(gemm::BM * kCG, BN)
                                     : ptx::make_idesc_bf16(gemm::BM * kCG, BN, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    unsigned gtrace_k = 0;
    for (int it = 0, tile = tile_at(0); tile < total_tiles; tile = tile_at(++it)) {
      ptx::mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
      GEMM_TRACE(0, 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < num_k_blocks; ++kb) {
#ifdef FLAME_DEBUG_TRACE_KB
        GEMM_TRACE(0, 11);
#endif
        ptx::mbar_wait(&full[stage], phase);
#ifdef FLAME_DEBUG_TRACE_KB
        GEMM_TRACE(0, 10);
#else
        if (kb == 0) GEMM_TRACE(0, 2);
#endif
        ptx::tc_fence_after();
        const uint32_t a_addr = ptx::smem_u32(smem_a + stage * C::kABytes);
        const uint32_t b_addr = ptx::smem_u32(smem_b + stage * C::kBBytes);
        if (leader) {
#pragma unroll
          for (int k = 0; k < gemm::BK / 16; ++k) {
            const uint64_t ad = ptx::make_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = ptx::make_desc_sw128(b_addr + k * 32, 16, 1024);
            // four 32-byte K steps per 128-byte row: K = 16 bf16 or 8 tf32 each
            if constexpr (kTF32) {
              if constexpr (kCG == 1) ptx::mma_tf32_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
              else ptx::mma_tf32_ss_cg2(d_tmem, ad, bd, idesc, (kb | k) != 0);
            } else {
              if constexpr (kCG == 1) ptx::mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
              else ptx::mma_bf16_ss_cg2(d_tmem, ad, bd, idesc, (kb | k) != 0);
            }
          }
          if constexpr (kCG == 1) ptx::mma_commit(&empty[stage]);
          else ptx::mma_commit_cg2_mc(&empty[stage], 0x3);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (leader) {
        if constexpr (kCG == 1) ptx::mma_commit(&tmem_full[acc]);
        else ptx::mma_commit_cg2_mc(&tmem_full[acc], 0x3);
      }
      __syncwarp();
      GEMM_TRACE(0, 3);
      if (++acc == C::kAcc) { acc = 0; acc_phase ^= 1; }
    }
  }
  } else {
    if constexpr (C::kRegSum) ptx::setmaxnreg_inc<C::kRegsEpi>();
    // ----------------------------------------------------------- epilogue
    constexpr bool kF32 = C::kF32;
    constexpr int kChunks = C::kChunks;
    const int ew = warp - 4;
    const int wq = warp & 3;    // TMEM lane quadrant this warp may access
    const int half = ew >> 2;   // which interleaved share of the 32-column chunks
    uint8_t* box = smem_box + ew * C::kBoxBytes;
    int box_i = 0;                           // alternating staging box (bf16 outputs)
    const bool epi_leader = ptx::elect_one();  // same lane issues stores and waits (bulk groups are per thread)
    // fp32 residual stream: this warp's valid chunks of all its tiles, in order;
    // position p lives in buffer p & 1 and is loaded while position p - 2 is consumed
    uint8_t* rbuf = smem_resid + ew * C::kResidBytes;
    uint64_t* rfull = resid_full + 2 * ew;
    auto nk_of_nb = [&](int nb) {  // this warp's valid chunks of an n block
      int n = 0;
#pragma unroll
      for (int k = 0; k < C::kMyChunks; ++k)
        n += (half + k * kEpiPerQuad < kChunks && nb * BN + (half + k * kEpiPerQuad) * 32 < ep.N) ? 1 : 0;
      return n;
    };
    int ld_it = 0, ld_t = tile_at(0), ld_k = 0, ld_buf = 0, rd_buf = 0;
    uint32_t rd_phase = 0;  // bit b: parity of buffer b's next completion
    // ld_t decoded once per tile (the divisions are not redone per residual box)
    int ld_g = 0, ld_mb = 0, ld_nb = 0, ld_nk = 0;
    auto ld_decode = [&]() {
      if (ld_t >= total_tiles) return;
      int mp;
      decode(ld_t, ld_g, mp, ld_nb);
      ld_mb = mp * ncl + crank;
      ld_nk = nk_of_nb(ld_nb);
    };
    auto ld_advance = [&](bool step) {
      if (step) ++ld_k;
      while (ld_t < total_tiles && ld_k >= ld_nk) {
        ld_t = tile_at(++ld_it);
        ld_k = 0;
        ld_decode();
      }
    };
    auto ld_issue = [&]() {
      if (ld_t >= total_tiles) return;
      if (epi_leader) {
        const int c0 = ld_nb * BN + (half + ld_k * kEpiPerQuad) * 32;
        const int r0 = min(ld_mb * gemm::BM + wq * 32, ep.M - 1);
        ptx::mbar_arrive_expect_tx(&rfull[ld_buf], C::kResidBox);
        ptx::tma_load_3d(rbuf + ld_buf * C::kResidBox, &tmR, &rfull[ld_buf], c0, r0, ep.resid_gstride ? ld_g : 0);
      }
      ld_buf ^= 1;
      ld_advance(true);
    };
    if constexpr (C::kResidTma) {
      ld_decode();
      ld_advance(false);
      ld_issue();
      ld_issue();
    }
    float* cv_bias = reinterpret_cast<float*>(smem_cvec + ew * C::kCvecBytes);
    float* cv_u = cv_bias + (C::kBiasSmem ? C::kMyChunks * 32 : 0);
    float* cv_gw = cv_u + (C::kUSmem ? C::kMyChunks * 32 : 0);
    float* cv_gb = cv_gw + (C::kGated ? C::kMyChunks * 32 : 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    unsigned gtrace_k = 0;
    const int tslot = ew == 0 ? 1 : (ew == 4 ? 2 : -1);
#define EPI_TRACE(code) do { if (tslot > 0) GEMM_TRACE(tslot, code); } while (0)
    // per-row epilogue operands of a tile, prefetched one tile ahead
    constexpr int kMaxPre = (EPI & EPI_LNSTATS) != 0 ? 4 : 0;
    struct RowOps {
      float rs;
      float2 p[kMaxPre > 0 ? kMaxPre : 1];
    };
    auto load_row_ops = [&](int t) {
      RowOps o;
      o.rs = 1.f;
#pragma unroll
      for (int k = 0; k < (kMaxPre > 0 ? kMaxPre : 1); ++k) o.p[k] = make_float2(0.f, 0.f);
      if (t >= total_tiles) return o;
      int gg, mpp, nbb;
      decode(t, gg, mpp, nbb);
      const int r = min((mpp * ncl + crank) * gemm::BM + wq * 32 + lane, ep.M - 1);
      if constexpr ((EPI & EPI_ROWSCALE) != 0) o.rs = __ldg(ep.rowscale + gg * ep.rowscale_gstride + r);
      if constexpr (kMaxPre > 0) {
        if (ep.stats_parts <= kMaxPre) {
          const float2* pst = reinterpret_cast<const float2*>(ep.lnstats + gg * ep.lnstats_gstride) +
                              static_cast<long long>(r) * ep.stats_parts;
#pragma unroll
          for (int k = 0; k < kMaxPre; ++k)
            if (k < ep.stats_parts) o.p[k] = __ldg(pst + k);
        }
      }
      return o;
    };
    RowOps row_ops = load_row_ops(tile_at(0));
    // kRegSum: this thread's row of the running gated sum, chunk k at gsum[k]
    float gsum[C::kRegSum ? C::kMyChunks : 1][32];
    for (int it = 0, tile = tile_at(0); tile < total_tiles; tile = tile_at(++it)) {
      int g, mp, n_blk;
      decode(tile, g, mp, n_blk);
      const int m_blk = mp * ncl + crank;  // may be m_tiles (tail): rows >= M
      if constexpr (C::kCvecs > 0) {
        // this warp's slice of the per-column vectors, fetched while the MMAs run
        __syncwarp();
#pragma unroll
        for (int k = 0; k < C::kMyChunks; ++k) {
          const int col = n_blk * BN + (half + k * kEpiPerQuad) * 32 + lane;
          const bool ok = half + k * kEpiPerQuad < kChunks && col < ep.N;
          if constexpr (C::kBiasSmem) cv_bias[k * 32 + lane] = ok ? __ldg(ep.bias + g * ep.bias_gstride + col) : 0.f;
          if constexpr (C::kUSmem) cv_u[k * 32 + lane] = ok ? __ldg(ep.colsum + g * ep.colsum_gstride + col) : 0.f;
          if constexpr (C::kGated) {
            cv_gw[k * 32 + lane] = ok ? __ldg(ep.gate_w + g * ep.N + col) : 0.f;
            cv_gb[k * 32 + lane] = ok ? __ldg(ep.gate_b + g * ep.N + col) : 0.f;
          }
        }
        __syncwarp();
      }
      const int row0 = m_blk * gemm::BM + wq * 32;
      // rows past M are clipped by the TMA store; clamp their residual reads
      const int row = min(row0 + lane, ep.M - 1);
      const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(wq * 32) << 16);
      // gated fusion: running sum over groups at TMEM columns [2 BN, 3 BN)
      const uint32_t t_gsum = tmem_base + 2 * BN + (static_cast<uint32_t>(wq * 32) << 16);
      const bool g_first = g == 0, g_last = g == groups - 1;
      // per-row operands (rowscale, folded-LN2 partials) were loaded one tile ahead;
      // queue the next tile's now, so their global-load latency is never exposed
      const RowOps cur_ops = row_ops;
      row_ops = load_row_ops(tile_at(it + 1));
      float rs = 1.f;
      float ln_mean = 0.f;
      if constexpr ((EPI & EPI_ROWSCALE) != 0) rs = cur_ops.rs;
      if constexpr ((EPI & EPI_LNSTATS) != 0) {
        // combine the producer's per-tile (sum, sumsq) partials in fixed order
        float s1 = 0.f, s2 = 0.f;
        if (ep.stats_parts <= kMaxPre) {
#pragma unroll
          for (int k = 0; k < kMaxPre; ++k) {
            if (k < ep.stats_parts) {
              s1 += cur_ops.p[k].x;
              s2 += cur_ops.p[k].y;
            }
          }
        } else {
          const float2* pst = reinterpret_cast<const float2*>(ep.lnstats + g * ep.lnstats_gstride) +
                              static_cast<long long>(row) * ep.stats_parts;
          for (int k = 0; k < ep.stats_parts; ++k) {
            const float2 p = pst[k];
            s1 += p.x;
            s2 += p.y;
          }
        }
        ln_mean = s1 / ep.d_true;
        rs = rsqrtf(fmaxf(s2 / ep.d_true - ln_mean * ln_mean, 0.f) + 1e-5f);
      }
      ptx::mbar_wait(&tmem_full[acc], acc_phase);
      EPI_TRACE(4);
      ptx::tc_fence_after();
      // LN(x) W + b = rs * acc + (b - rs * mean * u)
      const uint64_t rs2 = f2::make(rs, rs);
      const uint64_t nm2 = f2::make(-rs * ln_mean, -rs * ln_mean);
      const uint64_t zero2 = f2::make(0.f, 0.f);
      uint64_t st_s = zero2, st_q = zero2;  // STATS: (sum, sumsq) over this warp's columns, in pairs
      uint64_t dot01 = zero2, dot23 = zero2;  // ROWDOT: tasks 0-1 and 2-3

      auto chunk = [&](const int k, const uint32_t (&r)[32]) {
        const int c = half + k * kEpiPerQuad;
        const int col0 = n_blk * BN + c * 32;
        if (col0 >= ep.N) return;  // warp-uniform
        const bool full = col0 + 32 <= ep.N;
        if constexpr (C::kResidTma) {
          ptx::mbar_wait(&rfull[rd_buf], (rd_phase >> rd_buf) & 1);
          rd_phase ^= 1u << rd_buf;
        }
        float v[32];
        uint32_t gs[32];  // gated running sum of this chunk (groups < g)
        if constexpr (C::kGated && !C::kRegSum) {
          if (!g_first) {
            ptx::tmem_ld_32x32b_x32(t_gsum + c * 32, gs);
            ptx::tmem_ld_wait();
          }
        }
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          uint64_t p0 = f2::make(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
          uint64_t p1 = f2::make(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
          uint64_t b0 = zero2, b1 = zero2;
          if constexpr (C::kBiasSmem) {
            const float4 bb = *reinterpret_cast<const float4*>(cv_bias + k * 32 + j);
            b0 = f2::make(bb.x, bb.y);
            b1 = f2::make(bb.z, bb.w);
          } else if constexpr ((EPI & EPI_BIAS) != 0) {
            const float* bp = ep.bias + g * ep.bias_gstride + col0 + j;
            float4 bb;
            if (full) {
              bb = __ldg(reinterpret_cast<const float4*>(bp));
            } else {
              bb.x = col0 + j + 0 < ep.N ? bp[0] : 0.f;
              bb.y = col0 + j + 1 < ep.N ? bp[1] : 0.f;
              bb.z = col0 + j + 2 < ep.N ? bp[2] : 0.f;
              bb.w = col0 + j + 3 < ep.N ? bp[3] : 0.f;
            }
            b0 = f2::make(bb.x, bb.y);
            b1 = f2::make(bb.z, bb.w);
          }
          if constexpr ((EPI & EPI_LNSTATS) != 0) {
            const float4 uu = *reinterpret_cast<const float4*>(cv_u + k * 32 + j);
            p0 = f2::fma(rs2, p0, f2::fma(nm2, f2::make(uu.x, uu.y), b0));
            p1 = f2::fma(rs2, p1, f2::fma(nm2, f2::make(uu.z, uu.w), b1));
          } else if constexpr ((EPI & EPI_ROWSCALE) != 0 && (EPI & EPI_BIAS) != 0) {
            p0 = f2::fma(p0, rs2, b0);
            p1 = f2::fma(p1, rs2, b1);
          } else if constexpr ((EPI & EPI_ROWSCALE) != 0) {
            p0 = f2::mul(p0, rs2);
            p1 = f2::mul(p1, rs2);
          } else if constexpr ((EPI & EPI_BIAS) != 0) {
            p0 = f2::add(p0, b0);
            p1 = f2::add(p1, b1);
          }
          if constexpr ((EPI & EPI_GELU) != 0) {
            p0 = f2::gelu2x(p0);  // 2 GELU: consumers hold W / 2
            p1 = f2::gelu2x(p1);
          }
          if constexpr ((EPI & EPI_RESID) != 0) {
            float4 rr;
            if constexpr (C::kResidTma && (EPI & EPI_RESID_BF16) != 0) {
              // SW64 32 x 32 bf16 box: 16-byte chunk q of row r at q ^ ((r >> 1) & 3)
              const uint2 u = *reinterpret_cast<const uint2*>(
                  rbuf + rd_buf * C::kResidBox + lane * 64 + ((((j >> 3) ^ ((lane >> 1) & 3))) << 4) + (j & 4) * 2);
              const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
              const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
              rr = make_float4(lo.x, lo.y, hi.x, hi.y);
            } else if constexpr ((EPI & EPI_RESID_BF16) != 0) {
              const __nv_bfloat16* rp =
                  ep.resid_b + g * ep.resid_gstride + static_cast<long long>(row) * ep.resid_ld + col0 + j;
              if (full) {
                const uint2 u = *reinterpret_cast<const uint2*>(rp);
                const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
                const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
                rr = make_float4(lo.x, lo.y, hi.x, hi.y);
              } else {
                rr.x = col0 + j + 0 < ep.N ? __bfloat162float(rp[0]) : 0.f;
                rr.y = col0 + j + 1 < ep.N ? __bfloat162float(rp[1]) : 0.f;
                rr.z = col0 + j + 2 < ep.N ? __bfloat162float(rp[2]) : 0.f;
                rr.w = col0 + j + 3 < ep.N ? __bfloat162float(rp[3]) : 0.f;
              }
            } else if constexpr (C::kResidTma) {
              // swizzled (SW128) 32 x 32 fp32 box: 16-byte chunk q of row r at q ^ (r & 7)
              rr = *reinterpret_cast<const float4*>(rbuf + rd_buf * C::kResidBox + lane * 128 + (((j >> 2) ^ (lane & 7)) << 4));
            } else {
              const float* rp = ep.resid + g * ep.resid_gstride + static_cast<long long>(row) * ep.resid_ld + col0 + j;
              if (full) {
                rr = *reinterpret_cast<const float4*>(rp);
              } else {
                rr.x = col0 + j + 0 < ep.N ? rp[0] : 0.f;
                rr.y = col0 + j + 1 < ep.N ? rp[1] : 0.f;
                rr.z = col0 + j + 2 < ep.N ? rp[2] : 0.f;
                rr.w = col0 + j + 3 < ep.N ? rp[3] : 0.f;
              }
            }
            p0 = f2::add(p0, f2::make(rr.x, rr.y));
            p1 = f2::add(p1, f2::make(rr.z, rr.w));
          }
          if constexpr (C::kGated) {
            // forward.py:153-156: fused += sigmoid(h * w_g + c_g) * h, in block order
            const float4 gw = *reinterpret_cast<const float4*>(cv_gw + k * 32 + j);
            const float4 gb = *reinterpret_cast<const float4*>(cv_gb + k * 32 + j);
            const uint64_t z0 = f2::fma(p0, f2::make(gw.x, gw.y), f2::make(gb.x, gb.y));
            const uint64_t z1 = f2::fma(p1, f2::make(gw.z, gw.w), f2::make(gb.z, gb.w));
            float a0, a1, a2, a3;
            f2::split(z0, a0, a1);
            f2::split(z1, a2, a3);
            p0 = f2::mul(p0, f2::make(sigmoid_fast(a0), sigmoid_fast(a1)));
            p1 = f2::mul(p1, f2::make(sigmoid_fast(a2), sigmoid_fast(a3)));
            if (!g_first) {
              if constexpr (C::kRegSum) {
                p0 = f2::add(f2::make(gsum[k][j], gsum[k][j + 1]), p0);
                p1 = f2::add(f2::make(gsum[k][j + 2], gsum[k][j + 3]), p1);
              } else {
                p0 = f2::add(f2::make(__uint_as_float(gs[j]), __uint_as_float(gs[j + 1])), p0);
                p1 = f2::add(f2::make(__uint_as_float(gs[j + 2]), __uint_as_float(gs[j + 3])), p1);
              }
            }
          }
          if constexpr ((EPI & EPI_STATS) != 0) {
            // padded columns are exactly 0 and add nothing to the sums
            st_s = f2::add(st_s, f2::add(p0, p1));
            st_q = f2::fma(p0, p0, st_q);
            st_q = f2::fma(p1, p1, st_q);
          }
          f2::split(p0, v[j], v[j + 1]);
          f2::split(p1, v[j + 2], v[j + 3]);
        }
        if constexpr (C::kRowDot) {
          // partial dot with dot_w ([N][4], tasks zero-padded; cols >= N zero rows), fixed order
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(ep.dot_w) + (col0 + j));
            const uint64_t vv = f2::make(v[j], v[j]);
            dot01 = f2::fma(vv, f2::make(w.x, w.y), dot01);
            dot23 = f2::fma(vv, f2::make(w.z, w.w), dot23);
          }
        } else if (C::kRegSum && !g_last) {
#pragma unroll
          for (int j = 0; j < 32; ++j) gsum[C::kRegSum ? k : 0][j] = v[j];  // carried in registers
        } else if (C::kGated && !g_last) {
          // carry the running sum to the next group's tile (same thread, same lanes)
#pragma unroll
          for (int j = 0; j < 32; ++j) gs[j] = __float_as_uint(v[j]);
          ptx::tmem_st_32x32b_x16(t_gsum + c * 32, *reinterpret_cast<const uint32_t(*)[16]>(gs));
          ptx::tmem_st_32x32b_x16(t_gsum + c * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(gs + 16));
          ptx::tmem_st_wait();
        } else {
          if (epi_leader) ptx::tma_store_wait_read<C::kOutBoxes - 1>();  // this staging box free again
          __syncwarp();
          uint8_t* ob = box + box_i * C::kSlotBytes;
          uint8_t* box2 = ob + C::kOutBoxBytes;  // bf16 side-output box (kDual)
          if constexpr (C::kOutBoxes > 1) box_i ^= 1;
          if constexpr (C::kGated) {
            stage_row32<true>(ob, lane, v);  // the fp32 gated sum (tf32 expert operand)
          } else {
            stage_row32<kF32>(ob, lane, v);
            if constexpr (C::kDual) stage_row32<false>(box2, lane, v);
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (epi_leader) {
            if (row0 < ep.M) {
              if constexpr (C::kGated) {
                ptx::tma_store_3d(&tmO, ob, col0, row0, 0);  // one [M][N] fp32 output for all groups
              } else {
                ptx::tma_store_3d(&tmO, ob, ep.out_col0 + col0, row0, g);
                if constexpr (C::kDual) ptx::tma_store_3d(&tmO2, box2, col0, row0, g);
              }
            }
            ptx::tma_store_commit();  // one group per chunk keeps the box rotation exact
          }
        }
        EPI_TRACE(5);
        if constexpr (C::kResidTma) {
          // the residual box was read before a proxy fence (the store path's, or
          // this one): refill it with the next box of the stream
          if (C::kGated && !g_last) {
            ptx::fence_proxy_async_smem();
            __syncwarp();
          }
          ld_issue();
          rd_buf ^= 1;
        }
      };

      // balanced schedule hand-over slots of this warp (see bal above)
      const bool from_part = C::kRegSum && bal && bt_nh > 0 && it == bt_nt + bt_nf;
      const bool to_part = C::kRegSum && bal && bt_nt > 0 && it == bt_nt - 1;
      if constexpr (C::kRegSum) {
        if (from_part) {
          // the previous cluster's running sum over groups [0, g) of this chain; it
          // made it as its first work, so the wait is normally already satisfied
          const long long slot = ((static_cast<long long>(cid - 1) * ncl + crank) * kEpiWarps + ew);
          int* fl = ep.gflag + slot;
          if (lane == 0) {
            long long spins = 0;
            while (ptx::ld_acquire_gpu(fl) == 0) {
              __nanosleep(64);
              if (++spins > (1LL << 26)) __trap();  // a lost hand-over must fail, not hang
            }
            *fl = 0;  // single consumer: ready for the next launch
          }
          __syncwarp();
          const float4* src = reinterpret_cast<const float4*>(ep.gpart + slot * (32 * C::kMyChunks * 32)) +
                              lane * (C::kMyChunks * 8);
#pragma unroll
          for (int k = 0; k < C::kMyChunks; ++k)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 t4 = __ldcg(src + k * 8 + q);
              gsum[k][4 * q] = t4.x; gsum[k][4 * q + 1] = t4.y; gsum[k][4 * q + 2] = t4.z; gsum[k][4 * q + 3] = t4.w;
            }
        }
      }
      if constexpr (C::kRegSum) {
        // fully unrolled, so gsum is indexed statically (registers, not local
        // memory); the 16k-cycle K = 2048 mainloop hides the unpipelined loads
#pragma unroll
        for (int k = 0; k < C::kMyChunks; ++k) {
          if (half + k * kEpiPerQuad < kChunks) {
            uint32_t rr[32];
            ptx::tmem_ld_32x32b_x32(t_row + (half + k * kEpiPerQuad) * 32, rr);
            ptx::tmem_ld_wait();
            chunk(k, rr);
          }
        }
        if (to_part) {
          // hand the sum over groups [0, g] to the next cluster (its head piece)
          const long long slot = ((static_cast<long long>(cid) * ncl + crank) * kEpiWarps + ew);
          float4* dst = reinterpret_cast<float4*>(ep.gpart + slot * (32 * C::kMyChunks * 32)) + lane * (C::kMyChunks * 8);
#pragma unroll
          for (int k = 0; k < C::kMyChunks; ++k)
#pragma unroll
            for (int q = 0; q < 8; ++q)
              __stcg(dst + k * 8 + q, make_float4(gsum[k][4 * q], gsum[k][4 * q + 1], gsum[k][4 * q + 2], gsum[k][4 * q + 3]));
          __threadfence();
          __syncwarp();
          if (lane == 0) ptx::st_release_gpu(ep.gflag + slot, 1);
        }
      } else {
      // TMEM chunks ping-pong between two register sets: the load of chunk k+1
      // is in flight while chunk k is processed
      uint32_t ra[32], rb[32];
      ptx::tmem_ld_32x32b_x32(t_row + half * 32, ra);
#pragma unroll 1
      for (int k = 0; k < C::kMyChunks; k += 2) {
        ptx::tmem_ld_wait();
        const bool has1 = k + 1 < C::kMyChunks && half + (k + 1) * kEpiPerQuad < kChunks;
        if (has1) ptx::tmem_ld_32x32b_x32(t_row + (half + (k + 1) * kEpiPerQuad) * 32, rb);
        chunk(k, ra);
        if (!has1) break;
        ptx::tmem_ld_wait();
        const bool has2 = k + 2 < C::kMyChunks && half + (k + 2) * kEpiPerQuad < kChunks;
        if (has2) ptx::tmem_ld_32x32b_x32(t_row + (half + (k + 2) * kEpiPerQuad) * 32, ra);
        chunk(k + 1, rb);
        if (!has2) break;
      }
      }
      if constexpr ((EPI & EPI_STATS) != 0) {
        if (row0 + lane < ep.M) {
          float a0, a1, q0, q1;
          f2::split(st_s, a0, a1);
          f2::split(st_q, q0, q1);
          float2* dst = reinterpret_cast<float2*>(ep.stats + g * ep.stats_gstride) +
                        static_cast<long long>(row0 + lane) * (kEpiPerQuad * n_tiles) + n_blk * kEpiPerQuad + half;
          *dst = make_float2(a0 + a1, q0 + q1);
        }
      }
      if constexpr (C::kRowDot) {
        if (row0 + lane < ep.M) {
          float d[4];
          f2::split(dot01, d[0], d[1]);
          f2::split(dot23, d[2], d[3]);
          float* dst = reinterpret_cast<float*>(ep.out) +
                       (static_cast<long long>(row0 + lane) * (kEpiPerQuad * n_tiles) + n_blk * kEpiPerQuad + half) * ep.dot_n;
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (t < ep.dot_n) dst[t] = d[t];
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kCG == 1) ptx::mbar_arrive(&tmem_empty[acc]);
        else ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tmem_empty[acc]), 0));
      }
      EPI_TRACE(6);
      if (++acc == C::kAcc) { acc = 0; acc_phase ^= 1; }
    }
    if (epi_leader) ptx::tma_store_wait<0>();
    __syncwarp();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kCG > 1) ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg<C::kTmemCols, kCG>(tmem_base);
  }
#ifdef FLAME_DEBUG_TRACE
  if (g_gemm_trace != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemm_trace[4 * 4096 + 2 * blockIdx.x + 1] = t;
  }
#endif
}

}  // namespace flame
