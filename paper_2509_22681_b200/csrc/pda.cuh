// Proximal Data Accelerator: device-side feature assembly.
//
// Reference: Service.resolve_embeddings (service.py:97-108):
//     unique, inverse = np.unique(item_ids, return_inverse=True)
//     table[row] = embedding(unique[row])  (unknown / empty -> zeros)
//     return table[inverse]
// called once for the history ids and once for the candidate ids of a request.
//
// pda_dedup   : one CTA per id list.  Stable radix sort of (id, position) pairs,
//               adjacent-difference flags, block scan -> the ascending unique ids
//               and the int64 inverse map (bit-exact with np.unique), the sorted
//               positions, each unique id's run start, and the gather work list
//               (runs cut into pieces of <= kRunPiece positions).
// pda_gather  : grid-wide.  One warp per work piece reads the id's embedding row
//               (float4 / 8-byte vector loads) and writes it to the piece's
//               positions — history rows straight into the block-major row space
//               the projection GEMMs read (Climber split, forward.py:50-62),
//               candidate rows into the shared candidate row space.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include <type_traits>
#include <cub/block/block_radix_sort.cuh>

namespace flame {

constexpr int kRunPiece = 32;  // positions one gather warp writes per work item
constexpr int kPdaMaxList = 8192;  // ids per list SEGMENT handled by one CTA (cfg5: 8184 = one segment)

struct PdaLists {
  const long long* hist_ids;  // [R][H_bkt]
  const long long* cand_ids;  // [R][C_bkt]
  const int* hist_len;        // [R]
  const int* cand_len;        // [R]
  int R, H_bkt, C_bkt;
  // outputs, per list SEGMENT L = list * nseg + s (list = r for history, R + r for
  // candidates; segment s holds list positions [s * cap, (s + 1) * cap)); a list
  // longer than kPdaMaxList ids is deduplicated segment by segment (its rows are
  // still exact: a duplicate across segments is only gathered twice), so the
  // np.unique maps below are per segment, and exactly np.unique's when nseg == 1
  long long* unique;   // [2R * nseg][cap]
  long long* inverse;  // [2R * nseg][cap] (segment-local positions)
  int* n_unique;       // [2R * nseg]
  int* spos;           // [2R * nseg][cap] segment-local positions in sorted order
  int* ustart;         // [2R * nseg][cap] run start (index into spos) of each unique id
  int2* work;          // [2R * nseg][wcap] gather work items (unique index, first sorted position):
                       // each unique id's run split into pieces of <= kRunPiece positions
  int* n_work;         // [2R * nseg]
  int wcap;            // cap + cap / kRunPiece + 1
  int cap;             // ids per segment: min(max(H_bkt, C_bkt), kPdaMaxList)
  int nseg;            // segments per list
  const int* active;   // [1] requests in use (null: all R); lists of unused slots are skipped
};

// Sort phase: cub::BlockRadixSort of (id, position) pairs, kThreads x kItems =
// the list capacity.  Radix sort is stable, so equal ids keep ascending positions
// (the (id, position) order np.unique's inverse needs).  When every id of the list
// is non-negative only the bits up to the largest id are sorted (item ids < 2^17
// at 100k items: 5 passes instead of 16).
template <int kThreads, int kItems>
__global__ void __launch_bounds__(kThreads) pda_dedup(PdaLists a) {
  ptx::griddep_launch();  // let pda_gather's CTAs launch as this grid drains
  using Sort = cub::BlockRadixSort<unsigned long long, kThreads, kItems, int>;
  constexpr int P = kThreads * kItems;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int seg_list = blockIdx.x;  // output slot of this (list, segment)
  const int list = seg_list / a.nseg, seg = seg_list % a.nseg;
  const bool is_hist = list < a.R;
  const int r = is_hist ? list : list - a.R;
  if (a.active != nullptr && r >= __ldg(a.active)) {
    if (threadIdx.x == 0) {
      a.n_unique[seg_list] = 0;
      a.n_work[seg_list] = 0;
    }
    return;
  }
  const int n_list = is_hist ? a.hist_len[r] : a.cand_len[r];
  const int n = max(0, min(a.cap, n_list - seg * a.cap));  // ids of this segment
  const long long* ids = (is_hist ? a.hist_ids + static_cast<long long>(r) * a.H_bkt
                                  : a.cand_ids + static_cast<long long>(r) * a.C_bkt) +
                         static_cast<long long>(seg) * a.cap;
  __shared__ unsigned long long s_max;
  __shared__ int warp_tot[32];
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  long long raw[kItems];
  bool neg = false;
  unsigned long long mx = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int i = threadIdx.x * kItems + k;
    raw[k] = i < n ? ids[i] : 0;
    neg |= raw[k] < 0;
    mx = raw[k] > static_cast<long long>(mx) ? static_cast<unsigned long long>(raw[k]) : mx;
  }
  const bool any_neg = __syncthreads_or(neg);
  if (!any_neg && mx) atomicMax(&s_max, mx);
  __syncthreads();
  const int end_bit = any_neg ? 64 : (s_max == 0 ? 1 : 64 - __clzll(s_max));
  const unsigned long long pad = end_bit == 64 ? ~0ull : ((1ull << end_bit) - 1);
  unsigned long long keys[kItems];
  int vals[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int i = threadIdx.x * kItems + k;
    const unsigned long long u = static_cast<unsigned long long>(raw[k]);
    keys[k] = i < n ? (any_neg ? u ^ 0x8000000000000000ull : u) : pad;
    vals[k] = i;
  }
  Sort(*reinterpret_cast<typename Sort::TempStorage*>(smem_raw)).Sort(keys, vals, 0, end_bit);
  __syncthreads();  // the key / pos arrays alias the sort's temp storage
  long long* key = reinterpret_cast<long long*>(smem_raw);
  int* pos = reinterpret_cast<int*>(key + P);
  int* rank = pos + P;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int i = threadIdx.x * kItems + k;  // blocked arrangement: sorted order
    key[i] = vals[k] < n ? static_cast<long long>(any_neg ? keys[k] ^ 0x8000000000000000ull : keys[k])
                         : INT64_MAX;
    pos[i] = vals[k];
  }
  __syncthreads();
  // flags + inclusive scan (each thread owns a contiguous segment)
  const int per = (P + blockDim.x - 1) / blockDim.x;
  const int s0 = threadIdx.x * per;
  int local = 0;
  for (int i = s0; i < min(s0 + per, P); ++i) {
    const int f = (i < n && (i == 0 || key[i] != key[i - 1])) ? 1 : 0;
    local += f;
    rank[i] = local;
  }
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int v = lane < (blockDim.x / 32) ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    warp_tot[lane] = v;  // inclusive prefix over warps
  }
  __syncthreads();
  const int offset = (incl - local) + (w > 0 ? warp_tot[w - 1] : 0);
  long long* uq = a.unique + static_cast<long long>(seg_list) * a.cap;
  long long* inv = a.inverse + static_cast<long long>(seg_list) * a.cap;
  int* sp = a.spos + static_cast<long long>(seg_list) * a.cap;
  int* us = a.ustart + static_cast<long long>(seg_list) * a.cap;
  int first_rk[kItems];  // unique index of this thread's run starts (-1: not a start)
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int i = s0 + k;
    first_rk[k] = -1;
    if (i < n) {
      const int rk = rank[i] + offset - 1;  // unique index of sorted element i
      if (i == 0 || key[i] != key[i - 1]) {
        uq[rk] = key[i];
        us[rk] = i;
        first_rk[k] = rk;
      }
      inv[pos[i]] = rk;
      sp[i] = pos[i];
    }
  }
  if (threadIdx.x == blockDim.x - 1) a.n_unique[seg_list] = offset + local;

  // gather work list: a Zipf-hot id's run (hundreds of positions) would otherwise
  // be written by one warp while the rest of the grid idles; cut every run into
  // pieces of <= kRunPiece positions (run starts staged in smem over `rank`)
  __syncthreads();
  const int nu = warp_tot[blockDim.x / 32 - 1];
  int* rs = rank;  // rs[rk] = first sorted position of unique rk (rank[] is consumed)
#pragma unroll
  for (int k = 0; k < kItems; ++k)
    if (first_rk[k] >= 0) rs[first_rk[k]] = s0 + k;
  __syncthreads();
  // pieces per unique (kItems consecutive uniques per thread), block scan, emit
  int pcs[kItems];
  int plocal = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int rk = threadIdx.x * kItems + k;
    int c = 0;
    if (rk < nu) {
      const int len = (rk + 1 < nu ? rs[rk + 1] : n) - rs[rk];
      c = (len + kRunPiece - 1) / kRunPiece;
    }
    pcs[k] = c;
    plocal += c;
  }
  int pincl = plocal;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, pincl, o);
    if (lane >= o) pincl += t;
  }
  __syncthreads();  // warp_tot reused
  if (lane == 31) warp_tot[w] = pincl;
  __syncthreads();
  if (w == 0) {
    int v = lane < (blockDim.x / 32) ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    warp_tot[lane] = v;
  }
  __syncthreads();
  int woff = (pincl - plocal) + (w > 0 ? warp_tot[w - 1] : 0);
  int2* wk = a.work + static_cast<long long>(seg_list) * a.wcap;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int rk = threadIdx.x * kItems + k;
    for (int c = 0; c < pcs[k]; ++c) wk[woff + c] = make_int2(rk, rs[rk] + c * kRunPiece);
    woff += pcs[k];
  }
  if (threadIdx.x == blockDim.x - 1) a.n_work[seg_list] = woff;
}

template <typename TTab>
__device__ __forceinline__ float4 load_row4(const TTab* row, int c);
template <>
__device__ __forceinline__ float4 load_row4<float>(const float* row, int c) {
  return __ldg(reinterpret_cast<const float4*>(row + c));
}
template <>
__device__ __forceinline__ float4 load_row4<__nv_bfloat16>(const __nv_bfloat16* row, int c) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(row + c));
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

struct PdaGatherArgs {
  PdaLists l;
  const void* table;  // [num_items][D] (bf16 or fp32), unknown ids -> zero rows
  long long num_items;
  int D, d_true;
  int G;       // Climber blocks (history split)
  int hb_bkt;  // history rows per request-block in the row space
  AssembleOut o;  // fp32 rows (optional) + centered bf16 rows + rstd (folded LN1)
};

template <int kChunks>
__device__ __forceinline__ void assemble_row_st(const AssembleOut& o, bool hist, long long row,
                                                const float4 (&v)[kChunks], int lane, int D, int d_true,
                                                RowStats st) {
  float* f = hist ? o.Eh : o.Ec;
  if (f != nullptr) {
    float* dst = f + row * D;
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      const int c = (k * 32 + lane) * 4;
      if (c < D) *reinterpret_cast<float4*>(dst + c) = v[k];
    }
  }
  __nv_bfloat16* y = hist ? o.Ehc : o.Ecc;
  if (y != nullptr) {
    store_centered<kChunks>(y + row * D, v, st.mean, lane, D, d_true);
    if (lane == 0) (hist ? o.rs_h : o.rs_c)[row] = st.rstd;
  }
}

// One warp per unique id of a list (grid.x covers the list capacity twice: warps
// past the unique count zero the list's padding rows).  The warp reads the id's
// table row once, computes its LayerNorm statistics once, then fetches the run's
// destination positions 32 at a time (one coalesced load) and writes the row to
// each.  kChunks = D / 128 float4 per lane keeps registers low enough for 8
// resident CTAs per SM: the kernel is memory-latency bound.
template <typename TTab, int kChunks>
__global__ void __launch_bounds__(256) pda_gather(PdaGatherArgs a) {
  ptx::griddep_wait();  // PDL: pda_dedup's unique lists / work list
  ptx::griddep_launch();
  const int seg_list = blockIdx.y;  // (list, segment) of pda_dedup
  const int list = seg_list / a.l.nseg, seg = seg_list % a.l.nseg;
  const bool is_hist = list < a.l.R;
  const int r = is_hist ? list : list - a.l.R;
  if (a.l.active != nullptr && r >= __ldg(a.l.active)) return;  // unused slot: its rows are never read
  const int n = is_hist ? a.l.hist_len[r] : a.l.cand_len[r];
  const int n_seg = max(0, min(a.l.cap, n - seg * a.l.cap));  // positions of this segment
  const int p0 = seg * a.l.cap;                               // first list position of the segment
  const int nu = a.l.n_unique[seg_list];
  const int nw = a.l.n_work[seg_list];
  const int lane = threadIdx.x % 32;
  const int hb = is_hist ? n / a.G : 0;
  // the list's padding rows are zeroed by its first segment's warps
  const int pad_rows = seg != 0 ? 0 : (is_hist ? a.G * (a.hb_bkt - hb) : (a.l.C_bkt - n));
  const int work = nw + pad_rows;
  const int stride = gridDim.x * (blockDim.x / 32);
  for (int u = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; u < work; u += stride) {
  auto row_of = [&](int q) -> long long {  // destination row of segment position q
    const int p = p0 + q;
    if (is_hist) {
      const int g = p / hb, i = p % hb;
      return static_cast<long long>(g) * a.l.R * a.hb_bkt + static_cast<long long>(r) * a.hb_bkt + i;
    }
    return static_cast<long long>(r) * a.l.C_bkt + p;
  };
  if (u < nw) {
    // one piece (<= kRunPiece positions) of one unique id's run
    const long long* uq = a.l.unique + static_cast<long long>(seg_list) * a.l.cap;
    const int* sp = a.l.spos + static_cast<long long>(seg_list) * a.l.cap;
    const int* us = a.l.ustart + static_cast<long long>(seg_list) * a.l.cap;
    const int2 wi = a.l.work[static_cast<long long>(seg_list) * a.l.wcap + u];
    const long long id = uq[wi.x];
    const int b = wi.y;
    const int e = min(b + kRunPiece, (wi.x + 1 < nu) ? us[wi.x + 1] : n_seg);
    const bool known = id >= 0 && id < a.num_items;
    const TTab* table = reinterpret_cast<const TTab*>(a.table) + (known ? id : 0) * a.D;
    float4 v[kChunks];
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      const int c = (k * 32 + lane) * 4;
      v[k] = (known && c < a.D) ? load_row4<TTab>(table, c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int pos = b + lane < e ? sp[b + lane] : 0;  // the piece's positions, in flight with the row
    const RowStats st = warp_row_stats<kChunks>(v, lane, a.D, a.d_true);
    for (int j = 0; j < e - b; ++j)
      assemble_row_st<kChunks>(a.o, is_hist, row_of(__shfl_sync(0xffffffffu, pos, j)), v, lane, a.D, a.d_true,
                               st);
    continue;
  }
  // zero the padding rows of this list's region (rows past the actual length)
  const int k = u - nw;
  float4 z[kChunks];
#pragma unroll
  for (int q = 0; q < kChunks; ++q) z[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  long long row;
  if (is_hist) {
    const int per = a.hb_bkt - hb;
    const int g = k / per, i = hb + k % per;
    row = static_cast<long long>(g) * a.l.R * a.hb_bkt + static_cast<long long>(r) * a.hb_bkt + i;
  } else {
    row = static_cast<long long>(r) * a.l.C_bkt + n + k;
  }
  assemble_row_st<kChunks>(a.o, is_hist, row, z, lane, a.D, a.d_true, RowStats{0.f, 0.f});
  }
}

// Incremental refresh of the device item table (changed store rows,
// e.g. a key whose version was bumped): one warp per updated row, fp32 source
// rows [n][d] scattered to table[id] (converted to the table dtype, padding
// columns zeroed).  Ids outside the table are ignored (they stay zero rows).
template <typename TTab>
__global__ void table_scatter_rows(TTab* __restrict__ table, long long num_items, int D, int d,
                                   const long long* __restrict__ ids, const float* __restrict__ rows, int n) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (w >= n) return;
  const long long id = ids[w];
  if (id < 0 || id >= num_items) return;
  for (int c = lane; c < D; c += 32) {
    const float v = c < d ? rows[static_cast<long long>(w) * d + c] : 0.f;
    if constexpr (std::is_same<TTab, float>::value) table[id * D + c] = v;
    else table[id * D + c] = __float2bfloat16_rn(v);
  }
}

// Store feature values straight into the table: the reference's wire format
// (store.py:66-78 encode_feature_value / decode_embedding) is d little-endian
// float64 followed by filler up to bytes_per_value; a value shorter than d * 8
// bytes (e.g. empty) decodes to a zero row.  One warp per value.
template <typename TTab>
__global__ void table_decode_values(TTab* __restrict__ table, long long num_items, int D, int d,
                                    const long long* __restrict__ ids, const uint8_t* __restrict__ values,
                                    long long value_stride, const int* __restrict__ value_len, int n) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (w >= n) return;
  const long long id = ids[w];
  if (id < 0 || id >= num_items) return;
  const bool ok = value_len[w] >= d * 8;
  const uint8_t* v = values + static_cast<long long>(w) * value_stride;
  for (int c = lane; c < D; c += 32) {
    double x = 0.0;
    if (ok && c < d) {
      unsigned long long bits = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) bits |= static_cast<unsigned long long>(v[c * 8 + b]) << (8 * b);  // little endian
      x = __longlong_as_double(static_cast<long long>(bits));
    }
    if constexpr (std::is_same<TTab, float>::value) table[id * D + c] = static_cast<float>(x);
    else table[id * D + c] = __float2bfloat16_rn(static_cast<float>(x));
  }
}

}  // namespace flame
