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
//
// Softmax (1 thread = 1 query row).  The candidate's own key (the diagonal of
// the SUMI mask) seeds the state: m = s_self, l = 1.  History chunks update a
// reference max m that is only raised when a chunk max exceeds it by more than
// 2^8 (then the TMEM accumulator O is rescaled by the warp); otherwise
// p = exp2(s - m) stays within [0, 2^8] and O keeps accumulating in TMEM across
// chunks (PV with accumulate = 1).  At the end
//   out = (O + exp2(s_self - m) * v_self) / l,
// which equals attention_sumi_candidates' softmax over [history | self]
// (attention.py:131-146); H = 0 gives out = v_self.
//
// TMEM columns of warpgroup i: S [i*256, +128), P [+128, +64), O [+192, +64).
//   S = Q K^T      tcgen05.mma SS, M=128 N=128 K=64
//   P -> TMEM      tcgen05.st of the bf16 probabilities (never touches smem)
//   O += P V       tcgen05.mma TS (A = P from TMEM, B = V MN-major smem), N=64
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
  int store_tma;             // 1: 128-row output tiles never cross a request (bkt % 128 == 0)
  const int* active;         // [1] requests in use (null: all R); units of unused slots are skipped
};

// Debug-only event trace of CTA 0 (set through flame_debug_attn_trace): slot 0/1 =
// warpgroup rows 0, slot 2/3 = their control threads; entry = clock64 << 8 | code.
__device__ unsigned long long* g_attn_trace = nullptr;
__device__ unsigned int g_attn_trace_n[4];
// Each slot has exactly one writer thread, which keeps its own counter
// (trace_k, declared in each role) — no atomics on the traced path.
#ifdef FLAME_DEBUG_TRACE
#define ATTN_TRACE(slot, code)                                                            \
  do {                                                                                    \
    if (g_attn_trace != nullptr && blockIdx.x == 0 && ((slot) >= 2 ? (threadIdx.x & 31) == 0 : (threadIdx.x & 127) == 0)) { \
      if (trace_k < 4096) g_attn_trace[(slot) * 4096 + trace_k] = (clock64() << 8) | (code);  \
      ++trace_k;                                                                          \
    }                                                                                     \
  } while (0)
#else
// FLAME_ATTN_PROBE_MASK (dev A/B): a compiler memory barrier at the trace sites of
// the slots in the mask (bits 0-1 softmax warpgroups, 2 MMA issuer, 3 producer)
#ifndef FLAME_ATTN_PROBE_MASK
#define FLAME_ATTN_PROBE_MASK 0
#endif
#define ATTN_TRACE(slot, code)                                             \
  do {                                                                     \
    (void)trace_k;                                                         \
    if ((FLAME_ATTN_PROBE_MASK >> (slot)) & 1) asm volatile("" ::: "memory"); \
  } while (0)
#endif

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
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef FLAME_ATTN_POLY_MASK
#define FLAME_ATTN_POLY_MASK 0x24  // pairs 2 and 5 of every 8 (1/4 of the exponentials)
#endif
constexpr unsigned kPolyMask = FLAME_ATTN_POLY_MASK;

// exp2 of an fp32 pair on the FMA pipe (ptx::exp2_poly3, vectorised)
__device__ __forceinline__ uint64_t exp2_poly3_x2(uint64_t x) {
  float a, b;
  f2::split(x, a, b);
  x = f2::make(fmaxf(a, -126.0f), fmaxf(b, -126.0f));
  const uint64_t M = f2::make(12582912.0f, 12582912.0f);
  const uint64_t m1 = f2::make(-1.0f, -1.0f);
  const uint64_t t = f2::add(x, M);      // round(x) in the low mantissa bits
  const uint64_t r = f2::fma(M, m1, t);  // round(x), exact
  const uint64_t f = f2::fma(r, m1, x);  // x - round(x) in [-0.5, 0.5], exact
  uint64_t p = f2::fma(f2::make(0.05286737531423569f, 0.05286737531423569f), f,
                       f2::make(0.24215202033519745f, 0.24215202033519745f));
  p = f2::fma(p, f, f2::make(0.6935867667198181f, 0.6935867667198181f));
  p = f2::fma(p, f, f2::make(0.9999627470970154f, 0.9999627470970154f));
  float p0, p1, t0, t1;
  f2::split(p, p0, p1);
  f2::split(t, t0, t1);
  return f2::make(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
                  __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}
}  // namespace attn

template <bool kHist>
__global__ void __launch_bounds__(attn::kThreads, 1) sumi_attention_tcgen05(
    const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_out, AttnArgs a) {
  using namespace attn;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kWGBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * 14);

  const int warp = threadIdx.x / 32;
  const int G = a.num_blocks;
  const int R_eff = a.active != nullptr ? min(a.R, __ldg(a.active)) : a.R;
  const int n_units = R_eff * G * a.nh;
  const int bkt = kHist ? a.hb_bkt : a.c_bkt;
  const int n_tiles = (bkt + kRows - 1) / kRows;

  // barriers of warpgroup i (14 slots each):
  // 0 q_full (tx)  1 qs_free (128 WG + 1 control)  2,3 k_full  4,5 v_full
  // 6,7 kv_free (commit)  8 s_full (commit)  9 p_full (128)  10 o_full (commit)
  // 11 vself_full (tx: the candidates' own V rows for the job's end; for history
  //    rows a plain arrive that frees the output staging)  12 staging_ready (128)
  // 13 s_free (128): the WG has S_c in registers, so S_{c+1} may overwrite the
  //    S columns while the softmax of chunk c is still running
  auto B = [&](int i, int k) { return bars + i * 14 + k; };
  if (threadIdx.x == 256) {
    ptx::tma_prefetch_desc(&tm_qkv);
    for (int i = 0; i < 2; ++i) {
      for (int k = 0; k < 14; ++k) ptx::mbar_init(B(i, k), 1);
      ptx::mbar_init(B(i, 1), 129);
      ptx::mbar_init(B(i, 9), 128);
      ptx::mbar_init(B(i, 12), 128);
      ptx::mbar_init(B(i, 13), 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 8) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::griddep_wait();  // PDL: previous kernel's outputs visible from here on
  ptx::griddep_launch();

  // warpgroup i owns whole units: its k-th job is tile k % n_tiles of the CTA's
  // unit number i + 2 * (k / n_tiles), i.e. u = blockIdx.x + that * gridDim.x; a
  // unit's K/V is therefore loaded once per warpgroup and reused by all its tiles
  struct Job {
    bool valid;
    int u, r, g, h, t, hb, nk_all, nk, q_valid;
    int hist_row0, q_row0;
  };
  auto job_at = [&](int wg, int jk) {
    Job j{};
    j.u = blockIdx.x + (wg + 2 * (jk / n_tiles)) * gridDim.x;
    j.valid = j.u < n_units;
    if (!j.valid) return j;
    j.t = jk % n_tiles;
    j.h = j.u % a.nh;
    j.g = (j.u / a.nh) % G;
    j.r = j.u / (a.nh * G);
    j.hb = __ldg(a.hist_len + j.r) / G;
    j.nk_all = (j.hb + kKeys - 1) / kKeys;
    j.nk = kHist ? min(j.nk_all, j.t + 1) : j.nk_all;
    j.q_valid = kHist ? j.hb : __ldg(a.cand_len + j.r);
    j.hist_row0 = j.r * a.hb_bkt;
    j.q_row0 = (kHist ? j.hist_row0 : a.R * a.hb_bkt + j.r * a.c_bkt) + j.t * kRows;
    return j;
  };

  if (warp >= 8) {
    // ---------------------------------------------- control warp of WG i
    // The whole warp runs the schedule (waits, bookkeeping) so every operand
    // stays warp-uniform; one elected lane issues TMA / MMA / commits.
    const int i = warp - 8;
    const bool leader = ptx::elect_one();
    unsigned trace_k = 0;
    uint8_t* base = smem + i * kWGBytes;
    uint8_t *sQ = base, *sKs = base + kTile, *sVs = base + 2 * kTile;
    uint8_t *sK = base + 3 * kTile, *sV = base + 5 * kTile;
    const uint32_t tS = tmem + i * 256, tP = tS + 128, tO = tS + 192;
    constexpr uint32_t idesc_s = ptx::make_idesc_bf16(kRows, kKeys, 0, 0);
    constexpr uint32_t idesc_o = ptx::make_idesc_bf16(kRows, DH, 0, 1);
    uint32_t k_loads[2] = {0, 0}, v_loads[2] = {0, 0}, v_frees[2] = {0, 0};
    int res_unit = -1;    // unit whose K/V is resident in the slots (hb <= 256)
    int res_loaded = 0;   // chunks of res_unit already loaded
    auto load_qs = [&](const Job& j) {
      if (leader) {
        // Q and the candidates' own K (s_self); their own V arrives separately
        ptx::mbar_arrive_expect_tx(B(i, 0), (kHist ? 1 : 2) * kTile);
        const int h = j.h;
        ptx::tma_load_3d(sQ, &tm_qkv, B(i, 0), h * DH, j.q_row0, j.g);
        if (!kHist) ptx::tma_load_3d(sKs, &tm_qkv, B(i, 0), a.DA + h * DH, j.q_row0, j.g);
      }
      __syncwarp();
    };
    // V slot: reusable once the PV that read it completed (kv_free commit)
    auto load_v = [&](const Job& j, int chunk, int slot) {
      if (v_loads[slot] > v_frees[slot]) {  // slot still read by an earlier PV
        ptx::mbar_wait(B(i, 6 + slot), v_frees[slot] & 1);
        ++v_frees[slot];
      }
      const int row = j.hist_row0 + chunk * kKeys;
      if (leader) {
        ptx::mbar_arrive_expect_tx(B(i, 4 + slot), kTile);
        ptx::tma_load_3d(sV + slot * kTile, &tm_qkv, B(i, 4 + slot), 2 * a.DA + j.h * DH, row, j.g);
      }
      __syncwarp();
      ++v_loads[slot];
    };
    // K slot: the caller guarantees the S MMA that read it completed
    auto load_k = [&](const Job& j, int chunk, int slot) {
      const int row = j.hist_row0 + chunk * kKeys;
      if (leader) {
        ptx::mbar_arrive_expect_tx(B(i, 2 + slot), kTile);
        ptx::tma_load_3d(sK + slot * kTile, &tm_qkv, B(i, 2 + slot), a.DA + j.h * DH, row, j.g);
      }
      __syncwarp();
      ++k_loads[slot];
    };
    // both: the V wait (PV done) also orders the K reload after every earlier S on the slot
    auto load_kv = [&](const Job& j, int chunk, int slot) {
      load_v(j, chunk, slot);
      load_k(j, chunk, slot);
    };
    // K/V needed at the start of a job
    auto prepare_kv = [&](const Job& j) {
      if (j.nk_all <= 2) {
        if (res_unit != j.u) res_loaded = 0;
        for (int c = res_loaded; c < j.nk_all; ++c) load_kv(j, c, c);
        res_unit = j.u;
        res_loaded = j.nk_all;
      } else {
        res_unit = -1;
        for (int c = 0; c < 2 && c < j.nk; ++c) load_kv(j, c, c);
      }
    };
    Job cur = job_at(i, 0);
    if (cur.valid) {
      load_qs(cur);
      prepare_kv(cur);
    }
    auto load_vself = [&](const Job& jb) {  // the candidates' own V rows (needed at job end)
      if (leader) {
        if (kHist) {
          ptx::mbar_arrive(B(i, 11));  // history rows: just "staging free"
        } else {
          ptx::mbar_arrive_expect_tx(B(i, 11), kTile);
          ptx::tma_load_3d(sVs, &tm_qkv, B(i, 11), 2 * a.DA + jb.h * DH, jb.q_row0, jb.g);
        }
      }
      __syncwarp();
    };
    auto issue_s = [&](const Job& jb, int c) {  // S = Q K_c^T into the WG's S columns
      const int slot = jb.nk_all <= 2 ? c : (c & 1);
      ptx::mbar_wait(B(i, 2 + slot), (k_loads[slot] - 1) & 1);
      ptx::tc_fence_after();
      const uint32_t aQ = ptx::smem_u32(sQ), aK = ptx::smem_u32(sK + slot * kTile);
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          ptx::mma_bf16_ss(tS, ptx::make_desc_sw128(aQ + kk * 32, 16, 1024),
                           ptx::make_desc_sw128(aK + kk * 32, 16, 1024), idesc_s, kk != 0);
        ptx::mma_commit(B(i, 8));
        if (c == jb.nk - 1) ptx::mma_commit(B(i, 1));  // last read of Q for this job
      }
      __syncwarp();
      ATTN_TRACE(2 + i, 13);
    };
    if (cur.valid) load_vself(cur);
    uint32_t n = 0, cc = 0;  // jobs / chunks processed by this warpgroup
    bool s0_done = false;     // S_0 of `cur` was issued at the end of the previous job
    for (int jk = 0; cur.valid; ++jk, ++n) {
      const Job nxt = job_at(i, jk + 1);
      ATTN_TRACE(2 + i, 11);
      {
        // warm L2 two jobs ahead (the smem slots are all in use): that job's Q /
        // K_self / V_self tiles and, for a new unit, its history K / V chunks
        const Job far = job_at(i, jk + 2);
        if (leader && far.valid) {
          ptx::tma_prefetch_3d(&tm_qkv, far.h * DH, far.q_row0, far.g);
          if (!kHist) {
            ptx::tma_prefetch_3d(&tm_qkv, a.DA + far.h * DH, far.q_row0, far.g);
            ptx::tma_prefetch_3d(&tm_qkv, 2 * a.DA + far.h * DH, far.q_row0, far.g);
          }
          if (far.u != nxt.u)
            for (int c = 0; c < far.nk_all; ++c) {
              ptx::tma_prefetch_3d(&tm_qkv, a.DA + far.h * DH, far.hist_row0 + c * kKeys, far.g);
              ptx::tma_prefetch_3d(&tm_qkv, 2 * a.DA + far.h * DH, far.hist_row0 + c * kKeys, far.g);
            }
        }
        __syncwarp();
      }
      const bool resident = cur.nk_all <= 2;
      // Q / K_self of `nxt` may load once the last S of `cur` completed and the WG
      // read its q / k_self rows (qs_free phase n)
      auto prefetch_next_q = [&]() {
        if (!nxt.valid) return;
        ptx::mbar_wait(B(i, 1), n & 1);
        load_qs(nxt);
      };
      if (!s0_done && cur.nk > 0) {
        ptx::mbar_wait(B(i, 0), n & 1);  // Q (+ K_self) landed
        ATTN_TRACE(2 + i, 12);
        issue_s(cur, 0);
        if (cur.nk == 1) prefetch_next_q();
      } else if (s0_done && cur.nk == 1) {
        prefetch_next_q();
      }
      s0_done = false;
      for (int c = 0; c < cur.nk; ++c, ++cc) {
        const int slot = resident ? c : (c & 1);
        // S_{c+1} as soon as the WG holds S_c in registers: it runs under the
        // softmax of chunk c (PV_c is only needed before P_{c+1} is stored)
        ptx::mbar_wait(B(i, 13), cc & 1);
        if (c + 1 < cur.nk) {
          issue_s(cur, c + 1);
          if (c + 1 == cur.nk - 1) prefetch_next_q();
        }
        if (!resident) {
          // streamed chunks, K and V on their own schedules: K_{c+2} takes K_c's slot
          // (S_c completed: the WG read it), V_{c+1} takes V_{c-1}'s (PV_{c-1} was
          // issued an iteration ago), each a full chunk ahead of its MMA
          if (c + 2 < cur.nk) load_k(cur, c + 2, c & 1);
          if (c >= 1 && c + 1 < cur.nk) load_v(cur, c + 1, (c + 1) & 1);
        }
        ptx::mbar_wait(B(i, 9), cc & 1);  // WG stored P_c (and rescaled O)
        ATTN_TRACE(2 + i, 14);
        ptx::mbar_wait(B(i, 4 + slot), (v_loads[slot] - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t aV = ptx::smem_u32(sV + slot * kTile);
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < kKeys / 16; ++kk)
            ptx::mma_bf16_ts(tO, tP + kk * 8, ptx::make_desc_sw128(aV + kk * 16 * 128, kRows * 128, 1024),
                             idesc_o, (c | kk) != 0);
          ptx::mma_commit(B(i, 10));
        }
        __syncwarp();
        ATTN_TRACE(2 + i, 15);
        if (!resident) {
          if (leader) ptx::mma_commit(B(i, 6 + slot));  // V_c's slot is free once PV_c completes
          __syncwarp();
        } else if (!(nxt.valid && nxt.u == cur.u)) {
          // last job of this unit: recycle slot c as soon as PV_c is issued and,
          // when the next unit is resident too, start loading its chunk c into it
          if (leader) ptx::mma_commit(B(i, 6 + slot));
          __syncwarp();
          if (nxt.valid && nxt.nk_all <= 2 && c < nxt.nk_all) {
            if (res_unit != nxt.u) { res_unit = nxt.u; res_loaded = 0; }
            load_kv(nxt, c, c);
            res_loaded = c + 1;
          }
          if (c == cur.nk - 1) {
            // chunks this (causal) tile never used: their TMA must land before reuse
            for (int s = cur.nk; s < cur.nk_all; ++s) {
              ptx::mbar_wait(B(i, 2 + s), (k_loads[s] - 1) & 1);
              ptx::mbar_wait(B(i, 4 + s), (v_loads[s] - 1) & 1);
              if (leader) ptx::mma_commit(B(i, 6 + s));
              __syncwarp();
            }
          }
        }
      }
      if (cur.nk == 0) {
        if (leader) ptx::mbar_arrive(B(i, 1));
        __syncwarp();
        prefetch_next_q();
      }
      if (nxt.valid) {
        prepare_kv(nxt);
        // head start: the next job's first S runs while this job's output drains
        if (nxt.nk > 0) {
          ptx::mbar_wait(B(i, 0), (n + 1) & 1);
          issue_s(nxt, 0);
          s0_done = true;
        }
      }
      // this job's output: the WG staged its rows (or wrote them directly); store the
      // tile, then reuse the staging buffer for the next job's V_self
      ptx::mbar_wait(B(i, 12), n & 1);
      if (a.store_tma) {
        if (leader) {
          ptx::tma_store_3d(&tm_out, sVs, cur.h * DH, cur.q_row0, cur.g);
          ptx::tma_store_commit();
          ptx::tma_store_wait_read<0>();
        }
        __syncwarp();
      }
      if (nxt.valid) load_vself(nxt);
      cur = nxt;
    }
    if (leader) ptx::tma_store_wait<0>();
    __syncwarp();
  } else if (warp < 8) {
    // ------------------------------------------------- softmax / epilogue rows
    const int i = warp >> 2;
    const int row = threadIdx.x & 127;  // query row within the tile == TMEM lane
    unsigned trace_k = 0;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + i * 256 + lane_base, tP = tS + 128, tO = tS + 192;
    const uint8_t* base = smem + i * kWGBytes;
    const uint8_t *sQ = base, *sKs = base + kTile, *sVs = base + 2 * kTile;
    uint8_t* stage = smem + i * kWGBytes + 2 * kTile;  // = the V_self tile; reused as output staging
    uint32_t n = 0, cc = 0;
    Job nj = job_at(i, 0);
    for (int jk = 0;; ++jk, ++n) {
      const Job j = nj;
      ATTN_TRACE(i, 1);
      if (!j.valid) break;
      nj = job_at(i, jk + 1);  // metadata loads overlap this job
      const int qi = j.t * kRows + row;
      const bool row_ok = qi < j.q_valid;
      const float sl2 = a.scale_log2[j.g];
      float m_self, m, l;
      ptx::mbar_wait(B(i, 0), n & 1);
      ATTN_TRACE(i, 2);
      // the diagonal of the SUMI mask: s_self = q . k_self (attention.py:134) seeds
      // m = s_self, l = 1; its value term is added at the end.  History rows start
      // empty (m = -inf, l = 0).
      if (!kHist) {
        float dot = 0.f;
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) {
          const uint32_t off = ptx::sw128_offset(row, c * 16);
          const uint4 qv = *reinterpret_cast<const uint4*>(sQ + off);
          const uint4 kv = *reinterpret_cast<const uint4*>(sKs + off);
          const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&qv);
          const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 qf = __bfloat1622float2(q2[e]);
            const float2 kf = __bfloat1622float2(k2[e]);
            dot = fmaf(qf.x, kf.x, dot);
            dot = fmaf(qf.y, kf.y, dot);
          }
        }
        m_self = dot * sl2;
        m = m_self;
        l = 1.f;
      } else {
        m_self = -INFINITY;
        m = -INFINITY;
        l = 0.f;
      }
      ptx::mbar_arrive(B(i, 1));  // q / k_self rows read
      for (int c = 0; c < j.nk; ++c, ++cc) {
        const int key0 = c * kKeys;
        int key_lim = j.hb - key0;  // keys with local index < key_lim are valid
        if (kHist) key_lim = min(key_lim, qi - key0 + 1);
        const bool full = __all_sync(0xffffffffu, key_lim >= kKeys);
        ptx::mbar_wait(B(i, 8), cc & 1);
        ATTN_TRACE(i, 3);
        ptx::tc_fence_after();
        // the whole 128-key row of S in registers: 4 loads, one wait
        uint32_t s[kKeys];
#pragma unroll
        for (int k = 0; k < kKeys / 32; ++k)
          ptx::tmem_ld_32x32b_x32(tS + k * 32, *reinterpret_cast<uint32_t(*)[32]>(s + k * 32));
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(B(i, 13));  // S columns free for S_{c+1}
        if (!full) {
#pragma unroll
          for (int e = 0; e < kKeys; ++e)
            if (e >= key_lim) s[e] = __float_as_uint(-INFINITY);
        }
        // tree reductions (8 independent chains): only two warps share a scheduler,
        // so a serial max / sum chain would be latency-bound
        float mx[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mx[q] = __uint_as_float(s[q]);
#pragma unroll
        for (int e = 8; e < kKeys; ++e) mx[e & 7] = fmaxf(mx[e & 7], __uint_as_float(s[e]));
        const float cmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        // raise the reference max only when the chunk max exceeds it by > 2^8
        const float cm = cmax * sl2;
        const bool raise = (m == -INFINITY) ? (cm != -INFINITY) : (cm - m > kRescaleThreshold);
        const float m_new = raise ? cm : m;
        const float alpha = (raise && m != -INFINITY) ? ptx::exp2_approx(m - m_new) : 1.f;
        m = m_new;
        const float m_use = (m == -INFINITY) ? 0.f : m;
        // p = exp2(s*scale - m) on fp32 pairs (FFMA2 / FADD2), packed to bf16 pairs in
        // place (s[e/2] is dead).  kPolyMask selects the pairs (of every 8) whose exp2
        // runs as a polynomial on the FMA pipe instead of the MUFU: once the loop is
        // vectorised the MUFU, not the issue slots, is the limit.  Masked keys are
        // -inf and give 0 (poly: 2^-126, below bf16 resolution of any sum).
        const uint64_t sl2x2 = f2::make(sl2, sl2);
        const uint64_t nm2 = f2::make(-m_use, -m_use);
        uint64_t ps2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int e = 0; e < kKeys; e += 2) {
          const uint64_t x = f2::fma(f2::make(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), sl2x2, nm2);
          uint64_t p;
          if ((kPolyMask >> ((e >> 1) & 7)) & 1) {
            p = exp2_poly3_x2(x);
          } else {
            float x0, x1;
            f2::split(x, x0, x1);
            p = f2::make(ptx::exp2_approx(x0), ptx::exp2_approx(x1));
          }
          ps2[(e >> 1) & 3] = f2::add(ps2[(e >> 1) & 3], p);
          float p0, p1;
          f2::split(p, p0, p1);
          s[e / 2] = pack_bf16x2(p0, p1);
        }
        float psum;
        {
          float a0, a1, b0, b1;
          f2::split(f2::add(f2::add(ps2[0], ps2[1]), f2::add(ps2[2], ps2[3])), a0, a1);
          psum = a0 + a1;
          (void)b0; (void)b1;
        }
        l = l * alpha + psum;
        if (c > 0) {
          // PV(c-1) must be done before P is overwritten and O rescaled
          ptx::mbar_wait(B(i, 10), (cc - 1) & 1);
          ptx::tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
            uint32_t ov[DH];
#pragma unroll
            for (int k = 0; k < DH / 32; ++k)
              ptx::tmem_ld_32x32b_x32(tO + k * 32, *reinterpret_cast<uint32_t(*)[32]>(ov + k * 32));
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
            for (int k = 0; k < DH / 16; ++k)
              ptx::tmem_st_32x32b_x16(tO + k * 16, *reinterpret_cast<uint32_t(*)[16]>(ov + k * 16));
          }
        }
#pragma unroll
        for (int k = 0; k < kKeys / 32; ++k)
          ptx::tmem_st_32x32b_x16(tP + k * 16, *reinterpret_cast<uint32_t(*)[16]>(s + k * 16));
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(B(i, 9));
        ATTN_TRACE(i, 4);
      }
      // out = (O + exp2(s_self - m) v_self) / l
      float o[DH];
      if (j.nk > 0) {
        ptx::mbar_wait(B(i, 10), (cc - 1) & 1);
        ptx::tc_fence_after();
        uint32_t ov[DH];
#pragma unroll
        for (int k = 0; k < DH / 32; ++k)
          ptx::tmem_ld_32x32b_x32(tO + k * 32, *reinterpret_cast<uint32_t(*)[32]>(ov + k * 32));
        ptx::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < DH; ++e) o[e] = __uint_as_float(ov[e]);
        ptx::tc_fence_before();
      } else {
#pragma unroll
        for (int e = 0; e < DH; ++e) o[e] = 0.f;
      }
      ATTN_TRACE(i, 5);
      ptx::mbar_wait(B(i, 11), n & 1);  // V_self rows of this job (history: staging free)
      if (!kHist) {
        const float w_self = ptx::exp2_approx(m_self - (m == -INFINITY ? 0.f : m));
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) {
          const uint4 vv = *reinterpret_cast<const uint4*>(stage + ptx::sw128_offset(row, c * 16));
          const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vv);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 v = __bfloat1622float2(v2[e]);
            float& oa = o[c * 8 + 2 * e];
            float& ob = o[c * 8 + 2 * e + 1];
            f2::split(f2::fma(f2::make(w_self, w_self), f2::make(v.x, v.y), f2::make(oa, ob)), oa, ob);
          }
        }
      }
      {
        // 1 / l folded in here (fp32 pairs), so the stores below only pack
        const float inv = 1.f / l;
        const uint64_t inv2 = f2::make(inv, inv);
#pragma unroll
        for (int e = 0; e < DH; e += 2) f2::split(f2::mul(f2::make(o[e], o[e + 1]), inv2), o[e], o[e + 1]);
      }
      if (a.store_tma) {
        // stage the bf16 rows over the V_self tile (each thread rewrites exactly the
        // row it just read); the control warp TMA-stores the 128 x 64 tile
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) {
          uint4 w;
          w.x = pack_bf16x2(o[c * 8 + 0], o[c * 8 + 1]);
          w.y = pack_bf16x2(o[c * 8 + 2], o[c * 8 + 3]);
          w.z = pack_bf16x2(o[c * 8 + 4], o[c * 8 + 5]);
          w.w = pack_bf16x2(o[c * 8 + 6], o[c * 8 + 7]);
          *reinterpret_cast<uint4*>(stage + ptx::sw128_offset(row, c * 16)) = w;
        }
        ptx::fence_proxy_async_smem();
      } else if (row_ok) {
        __nv_bfloat16* dst = a.out + j.g * a.out_gstride + static_cast<long long>(j.q_row0 + row) * a.out_ld + j.h * DH;
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) {
          uint4 w;
          w.x = pack_bf16x2(o[c * 8 + 0], o[c * 8 + 1]);
          w.y = pack_bf16x2(o[c * 8 + 2], o[c * 8 + 3]);
          w.z = pack_bf16x2(o[c * 8 + 4], o[c * 8 + 5]);
          w.w = pack_bf16x2(o[c * 8 + 6], o[c * 8 + 7]);
          reinterpret_cast<uint4*>(dst)[c] = w;
        }
      }
      ptx::mbar_arrive(B(i, 12));  // staging written / V_self rows consumed
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
