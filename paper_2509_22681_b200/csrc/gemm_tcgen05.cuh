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
  long long resid_ld;
  long long resid_gstride;
  int M, N;               // logical bounds of this problem
};

enum : int {
  EPI_BIAS = 1,
  EPI_GELU = 2,
  EPI_RESID = 4,
  EPI_OUT_F32 = 8,
};

namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle row
constexpr int kEpiWarps = 8;
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr int kBoxBytes = 32 * 32 * 4;  // one 32x32 staging box per epilogue warp (fp32 worst case)

template <int BN>
struct Cfg {
  static constexpr int kStages = BN >= 256 ? 4 : 6;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmemBytes =
      kStages * kStageBytes + kEpiWarps * kBoxBytes + 1024 /*align*/ + 256 /*barriers*/;
};

}  // namespace gemm

template <int BN, int EPI>
__global__ void __launch_bounds__(gemm::kThreads, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, int num_k_blocks, int m_tiles, int n_tiles, int groups, int a_shared,
                      GemmEpilogue ep) {
  using C = gemm::Cfg<BN>;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t pad = ((raw_addr + 1023) & ~1023u) - raw_addr;
  uint8_t* smem = smem_raw + pad;
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * C::kABytes;
  uint8_t* smem_box = smem + kStages * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_box + gemm::kEpiWarps * gemm::kBoxBytes);
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
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tmem_full[s], 1);
      ptx::mbar_init(&tmem_empty[s], gemm::kEpiWarps);
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
    const int half = ew >> 2;   // which interleaved half of the 32-column chunks
    uint8_t* box = smem_box + ew * gemm::kBoxBytes;
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
#pragma unroll 1
      for (int c = half; c < BN / 32; c += 2) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
        ptx::tmem_ld_wait();
        const int col0 = n_blk * BN + c * 32;
        if (col0 >= ep.N) continue;  // warp-uniform
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        epilogue_math<EPI, 32, true>(v, ep, g, row, col0);
        if (epi_leader) ptx::tma_store_wait_read<0>();  // staging box free again
        __syncwarp();
        stage_row32<kF32>(box, lane, v);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (epi_leader) {
          ptx::tma_store_3d(&tmO, box, ep.out_col0 + col0, row0, g);
          ptx::tma_store_commit();
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
