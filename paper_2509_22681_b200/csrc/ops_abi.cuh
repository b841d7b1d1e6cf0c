// Operator-level entry points of the C ABI (include/flame_b200.h, "operators"):
// the reference's model/__init__.py operators (attention.py, forward.py) over
// host fp64 arrays, each computed on the device.
//
// The SUMI attention, block and expert operators run the SAME kernels as the
// forward pass (Pipe::attention / Pipe::run / Pipe::experts on a one-request
// executor), so an operator-level parity test exercises the product kernels.
// The small helpers (gelu, sigmoid, layer_norm, masked softmax rows, masked
// attention over an arbitrary permission matrix) are plain fp64 SIMT kernels:
// the reference computes them in fp64 and they are not on the scoring path.
//
// Included at the end of flame.cu (one translation unit: it uses Pipe,
// FlameCtx and FlameExec from there).
#pragma once

namespace {

constexpr double kLnEps = 1e-5;  // reference forward.py:28 LN_EPS

// Device buffers freed on scope exit (operators are synchronous).
struct OpBufs {
  std::vector<void*> p;
  ~OpBufs() {
    for (void* q : p) cudaFree(q);
  }
  template <typename T>
  T* get(size_t count) {
    void* q = nullptr;
    if (cudaMalloc(&q, (count > 0 ? count : 1) * sizeof(T)) != cudaSuccess) return nullptr;
    p.push_back(q);
    return static_cast<T*>(q);
  }
};

// ------------------------------------------------------------- fp64 helpers
__device__ __forceinline__ double gelu_f64(double x) {
  // forward.py:33-35, tanh form
  const double k = 0.7978845608028654;  // sqrt(2/pi)
  return 0.5 * x * (1.0 + tanh(k * (x + 0.044715 * x * x * x)));
}

__global__ void op_unary_f64(int op, const double* __restrict__ x, double* __restrict__ y, long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = x[i];
  y[i] = op == 0 ? gelu_f64(v) : 1.0 / (1.0 + exp(-v));
}

// One block per row: layer_norm (forward.py:43-47) or masked_softmax_rows
// (attention.py:28-36; -inf entries stay excluded, a row of only -inf gives NaN
// as in the reference).  Fixed-order reductions through shared memory.
__device__ double block_sum(double v, double* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (t < o) red[t] += red[t + o];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

__device__ double block_max(double v, double* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (t < o) red[t] = fmax(red[t], red[t + o]);
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

__global__ void op_rows_f64(int op, const double* __restrict__ x, const double* __restrict__ scale,
                            const double* __restrict__ shift, double* __restrict__ y, int width) {
  __shared__ double red[256];
  const double* xr = x + static_cast<long long>(blockIdx.x) * width;
  double* yr = y + static_cast<long long>(blockIdx.x) * width;
  if (op == 2) {  // layer_norm
    double s = 0.0;
    for (int k = threadIdx.x; k < width; k += blockDim.x) s += xr[k];
    const double mean = block_sum(s, red) / width;
    double q = 0.0;
    for (int k = threadIdx.x; k < width; k += blockDim.x) {
      const double dv = xr[k] - mean;
      q += dv * dv;
    }
    const double var = block_sum(q, red) / width;
    const double den = sqrt(var + kLnEps);
    for (int k = threadIdx.x; k < width; k += blockDim.x) yr[k] = (xr[k] - mean) / den * scale[k] + shift[k];
  } else {  // masked softmax
    double m = -INFINITY;
    for (int k = threadIdx.x; k < width; k += blockDim.x) m = fmax(m, xr[k]);
    m = block_max(m, red);
    double s = 0.0;
    for (int k = threadIdx.x; k < width; k += blockDim.x) s += exp(xr[k] - m);
    const double z = block_sum(s, red);
    for (int k = threadIdx.x; k < width; k += blockDim.x) yr[k] = exp(xr[k] - m) / z;
  }
}

// Scores of masked attention over an arbitrary permission matrix
// (attention.py:55-67): S[i][j] = scale * q_i . k_j where allowed, else -inf.
__global__ void op_masked_scores_f64(const double* __restrict__ q, const double* __restrict__ k,
                                     const unsigned char* __restrict__ allowed, double* __restrict__ S, int T,
                                     int dh, double scale) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(T) * T) return;
  const int i = static_cast<int>(idx / T), j = static_cast<int>(idx % T);
  if (!allowed[idx]) {
    S[idx] = -INFINITY;
    return;
  }
  double acc = 0.0;
  for (int c = 0; c < dh; ++c) acc += q[static_cast<long long>(i) * dh + c] * k[static_cast<long long>(j) * dh + c];
  S[idx] = acc * scale;
}

// out[i][c] = sum_j P[i][j] v[j][c] over the row-normalised scores; one block per row.
__global__ void op_weighted_values_f64(const double* __restrict__ P, const double* __restrict__ v,
                                       double* __restrict__ out, int T, int dh) {
  const double* pr = P + static_cast<long long>(blockIdx.x) * T;
  for (int c = threadIdx.x; c < dh; c += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < T; ++j) acc += pr[j] * v[static_cast<long long>(j) * dh + c];
    out[static_cast<long long>(blockIdx.x) * dh + c] = acc;
  }
}

template <typename Act>
Act to_act(double v);
template <>
float to_act<float>(double v) { return static_cast<float>(v); }
template <>
__nv_bfloat16 to_act<__nv_bfloat16>(double v) { return __float2bfloat16_rn(static_cast<float>(v)); }

inline double from_act(float v) { return v; }
inline double from_act(__nv_bfloat16 v) { return static_cast<double>(__bfloat162float(v)); }

// SUMI attention over one request through the forward pass's kernels:
// Pipe::attention on a one-request, one-block executor whose QKV rows hold the
// caller's q / k / v (head h in lanes [h*HS, h*HS+dh) of each third, HS = 64 or 128).
template <typename Act>
int op_attention(int device, int nh, int T, int dh, int h, int cand_only, double temperature, const double* q,
                 const double* k, const double* v, double* out) {
  const int C = T - h;
  FlameCtx c;
  c.precision = std::is_same<Act, __nv_bfloat16>::value ? FLAME_BF16 : FLAME_FP32;
  c.device = device;
  cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device);
  c.HS = dh <= 64 ? 64 : 128;
  c.nh = nh; c.dh = dh; c.G = 1; c.DA = nh * c.HS; c.d = nh * dh; c.D = pad_to(c.d, 64);
  c.act_bytes = sizeof(Act);
  OpBufs b;
  const double sc = 1.0 / (temperature * std::sqrt(static_cast<double>(dh)));
  const float scale = static_cast<float>(sc);
  const float scale_log2 = static_cast<float>(sc * 1.4426950408889634);
  c.scale = b.get<float>(1);
  c.scale_log2 = b.get<float>(1);
  FlameExec e;
  e.ctx = &c;
  e.R = 1; e.hb_bkt = h; e.c_bkt = C; e.H_bkt = h;
  e.Rh = h; e.Rc = C; e.rows = T;
  const size_t DA = c.DA, rows = T;
  e.QKV = b.get<Act>(rows * 3 * DA);
  e.AO = b.get<Act>(rows * DA);
  int* meta = b.get<int>(4);
  if (!c.scale || !c.scale_log2 || !e.QKV || !e.AO || !meta) return fail(2, "operator workspace allocation failed");
  e.io.hist_len = meta; e.io.cand_len = meta + 1; e.io.out_offset = meta + 2;
  // QKV rows: history rows [0, h), candidate rows [h, T); unused lanes are zero
  std::vector<Act> hq(rows * 3 * DA, to_act<Act>(0.0));
  for (int hd = 0; hd < nh; ++hd)
    for (int t = 0; t < T; ++t) {
      Act* row = hq.data() + static_cast<size_t>(t) * 3 * DA + static_cast<size_t>(hd) * c.HS;
      const bool has_q = !cand_only || t >= h;
      const long long qt = cand_only ? t - h : t;
      const long long qrows = cand_only ? C : T;
      for (int l = 0; l < dh; ++l) {
        if (has_q) row[l] = to_act<Act>(q[(static_cast<long long>(hd) * qrows + qt) * dh + l]);
        row[DA + l] = to_act<Act>(k[(static_cast<long long>(hd) * T + t) * dh + l]);
        row[2 * DA + l] = to_act<Act>(v[(static_cast<long long>(hd) * T + t) * dh + l]);
      }
    }
  const int hmeta[4] = {h, C, 0, 1};
  cudaStream_t s = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{s};
  CUDA_TRY(cudaMemcpyAsync(e.QKV, hq.data(), hq.size() * sizeof(Act), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(meta, hmeta, sizeof(hmeta), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(c.scale, &scale, sizeof(float), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(c.scale_log2, &scale_log2, sizeof(float), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemsetAsync(e.AO, 0, rows * DA * sizeof(Act), s));
  Pipe<Act> p{&e, &c, s};
  if (!cand_only && h > 0)
    if (int rc = p.attention(true)) return rc;
  if (C > 0)
    if (int rc = p.attention(false)) return rc;
  std::vector<Act> ho(rows * DA);
  CUDA_TRY(cudaMemcpyAsync(ho.data(), e.AO, ho.size() * sizeof(Act), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  const int t0 = cand_only ? h : 0;
  const long long orows = T - t0;
  for (int hd = 0; hd < nh; ++hd)
    for (int t = t0; t < T; ++t)
      for (int l = 0; l < dh; ++l)
        out[(static_cast<long long>(hd) * orows + (t - t0)) * dh + l] =
            from_act(ho[static_cast<size_t>(t) * DA + static_cast<size_t>(hd) * c.HS + l]);
  return 0;
}

template <typename Act>
int op_block_states(FlameCtx* c, const double* history, long long H, const double* cand, long long C, double* out) {
  const int G = c->G, d = c->d, D = c->D;
  const int hb = static_cast<int>(H / G);
  OpBufs b;
  float* dh = b.get<float>(static_cast<size_t>(H) * d);
  float* dc = b.get<float>(static_cast<size_t>(C) * d);
  int* meta = b.get<int>(4);
  float* scores = b.get<float>(static_cast<size_t>(C) * c->tasks);
  if (!dh || !dc || !meta || !scores) return fail(2, "operator workspace allocation failed");
  FlameIO io{};
  io.hist_emb = dh; io.cand_emb = dc;
  io.hist_len = meta; io.cand_len = meta + 1; io.out_offset = meta + 2; io.scores = scores;
  FlameExec* e = nullptr;
  if (int rc = flame_exec_create(c, 1, hb, static_cast<int>(C), &io, &e)) return rc;
  struct ExecGuard {
    FlameExec* e;
    ~ExecGuard() { delete e; }
  } eg{e};
  std::vector<float> hh(static_cast<size_t>(H) * d), hc(static_cast<size_t>(C) * d);
  for (size_t i = 0; i < hh.size(); ++i) hh[i] = static_cast<float>(history[i]);
  for (size_t i = 0; i < hc.size(); ++i) hc[i] = static_cast<float>(cand[i]);
  const int hmeta[4] = {static_cast<int>(H), static_cast<int>(C), 0, 1};
  cudaStream_t s = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{s};
  CUDA_TRY(cudaMemcpyAsync(dh, hh.data(), hh.size() * 4, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(dc, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(meta, hmeta, sizeof(hmeta), cudaMemcpyHostToDevice, s));
  Pipe<Act> p{e, c, s};
  p.block_states = true;
  if (int rc = p.run(FLAME_INPUT_EMBEDDINGS)) return rc;
  // candidate rows of every block: [G][rows][D] starting at row Rh = hb
  std::vector<float> ho(static_cast<size_t>(G) * C * d);
  for (int g = 0; g < G; ++g)
    CUDA_TRY(cudaMemcpy2DAsync(ho.data() + static_cast<size_t>(g) * C * d, static_cast<size_t>(d) * 4,
                               p.final_x + static_cast<size_t>(g) * e->rows * D + static_cast<size_t>(hb) * D,
                               static_cast<size_t>(D) * 4, static_cast<size_t>(d) * 4, static_cast<size_t>(C),
                               cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  for (size_t i = 0; i < ho.size(); ++i) out[i] = ho[i];
  return 0;
}

template <typename Act>
int op_expert_heads(FlameCtx* c, const double* fused, long long C, double* out) {
  const int d = c->d, D = c->D;
  OpBufs b;
  int* meta = b.get<int>(4);
  float* scores = b.get<float>(static_cast<size_t>(C) * c->tasks);
  if (!meta || !scores) return fail(2, "operator workspace allocation failed");
  FlameIO io{};
  io.hist_len = meta; io.cand_len = meta + 1; io.out_offset = meta + 2; io.scores = scores;
  FlameExec* e = nullptr;
  if (int rc = flame_exec_create(c, 1, 0, static_cast<int>(C), &io, &e)) return rc;
  struct ExecGuard {
    FlameExec* e;
    ~ExecGuard() { delete e; }
  } eg{e};
  std::vector<float> hf(static_cast<size_t>(C) * D, 0.f);
  for (long long r = 0; r < C; ++r)
    for (int k = 0; k < d; ++k) hf[static_cast<size_t>(r) * D + k] = static_cast<float>(fused[r * d + k]);
  const int hmeta[4] = {0, static_cast<int>(C), 0, 1};
  cudaStream_t s = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{s};
  CUDA_TRY(cudaMemcpyAsync(e->Fz, hf.data(), hf.size() * 4, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(meta, hmeta, sizeof(hmeta), cudaMemcpyHostToDevice, s));
  Pipe<Act> p{e, c, s};
  if (int rc = p.experts()) return rc;
  std::vector<float> ho(static_cast<size_t>(C) * c->tasks);
  CUDA_TRY(cudaMemcpyAsync(ho.data(), scores, ho.size() * 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  for (size_t i = 0; i < ho.size(); ++i) out[i] = ho[i];
  return 0;
}

}  // namespace

extern "C" {

int flame_op_attention_sumi(int precision, int device, int num_heads, int seq_len, int head_dim, int hist_len,
                            int candidates_only, double temperature, const double* q, const double* k,
                            const double* v, double* out) {
  if (precision != FLAME_BF16 && precision != FLAME_FP32) return fail(1, "bad precision");
  if (num_heads < 1 || seq_len < 0 || head_dim < 1) return fail(1, "bad attention shape");
  if (head_dim > 128) return fail(1, "head_dim above 128 is not supported by the SUMI attention kernels");
  if (hist_len < 0 || hist_len > seq_len)
    return fail(1, "hist_len " + std::to_string(hist_len) + " out of range for sequence length " +
                       std::to_string(seq_len));
  if (!(temperature > 0)) return fail(1, "temperature must be positive");
  if (seq_len == 0 || (candidates_only && seq_len == hist_len)) return 0;
  if (!q || !k || !v || !out) return fail(1, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  return precision == FLAME_BF16
             ? op_attention<__nv_bfloat16>(device, num_heads, seq_len, head_dim, hist_len, candidates_only,
                                           temperature, q, k, v, out)
             : op_attention<float>(device, num_heads, seq_len, head_dim, hist_len, candidates_only, temperature,
                                   q, k, v, out);
}

int flame_op_attention_masked(int device, int seq_len, int head_dim, double temperature, const double* q,
                              const double* k, const double* v, const unsigned char* allowed, double* out) {
  if (seq_len < 0 || head_dim < 1) return fail(1, "bad attention shape");
  if (!(temperature > 0)) return fail(1, "temperature must be positive");
  if (seq_len == 0) return 0;
  if (!q || !k || !v || !allowed || !out) return fail(1, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  const size_t T = seq_len, n = T * head_dim;
  OpBufs b;
  double *dq = b.get<double>(n), *dk = b.get<double>(n), *dv = b.get<double>(n), *dS = b.get<double>(T * T),
         *dP = b.get<double>(T * T), *dout = b.get<double>(n);
  unsigned char* dm = b.get<unsigned char>(T * T);
  if (!dq || !dk || !dv || !dS || !dP || !dout || !dm) return fail(2, "operator workspace allocation failed");
  CUDA_TRY(cudaMemcpy(dq, q, n * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dk, k, n * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dv, v, n * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dm, allowed, T * T, cudaMemcpyHostToDevice));
  const double scale = 1.0 / (temperature * std::sqrt(static_cast<double>(head_dim)));
  op_masked_scores_f64<<<static_cast<unsigned>((T * T + 255) / 256), 256>>>(dq, dk, dm, dS, seq_len, head_dim,
                                                                             scale);
  CUDA_TRY(cudaGetLastError());
  op_rows_f64<<<seq_len, 256>>>(3, dS, nullptr, nullptr, dP, seq_len);
  CUDA_TRY(cudaGetLastError());
  op_weighted_values_f64<<<seq_len, 64>>>(dP, dv, dout, seq_len, head_dim);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out, dout, n * 8, cudaMemcpyDeviceToHost));
  return 0;
}

int flame_op_rows(int op, int device, long long rows, int width, const double* x, const double* scale,
                  const double* shift, double* out) {
  if (op < FLAME_OP_GELU || op > FLAME_OP_SOFTMAX) return fail(1, "bad row operator");
  if (rows < 0 || width < 0) return fail(1, "bad row operator shape");
  if (op == FLAME_OP_LAYER_NORM && (!scale || !shift)) return fail(1, "layer_norm needs scale and shift");
  const long long n = rows * width;
  if (n == 0) return 0;
  if (!x || !out) return fail(1, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  OpBufs b;
  double *dx = b.get<double>(n), *dy = b.get<double>(n);
  double *ds = nullptr, *dt = nullptr;
  if (!dx || !dy) return fail(2, "operator workspace allocation failed");
  CUDA_TRY(cudaMemcpy(dx, x, n * 8, cudaMemcpyHostToDevice));
  if (op == FLAME_OP_LAYER_NORM) {
    ds = b.get<double>(width);
    dt = b.get<double>(width);
    if (!ds || !dt) return fail(2, "operator workspace allocation failed");
    CUDA_TRY(cudaMemcpy(ds, scale, width * 8LL, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dt, shift, width * 8LL, cudaMemcpyHostToDevice));
  }
  if (op == FLAME_OP_GELU || op == FLAME_OP_SIGMOID) {
    op_unary_f64<<<static_cast<unsigned>((n + 255) / 256), 256>>>(op == FLAME_OP_GELU ? 0 : 1, dx, dy, n);
  } else {
    if (rows > 0x7fffffffLL) return fail(1, "too many rows");
    op_rows_f64<<<static_cast<unsigned>(rows), 256>>>(op == FLAME_OP_LAYER_NORM ? 2 : 3, dx, ds, dt, dy, width);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out, dy, n * 8, cudaMemcpyDeviceToHost));
  return 0;
}

int flame_op_gated_fusion(int device, int num_blocks, long long rows, int width, const double* block_outputs,
                          const double* gate_w, const double* gate_b, double* out) {
  if (num_blocks < 1 || rows < 0 || width < 1) return fail(1, "bad gated fusion shape");
  if (rows == 0) return 0;
  if (!block_outputs || !gate_w || !gate_b || !out) return fail(1, "null argument");
  if (rows > 0x7fffffffLL) return fail(1, "too many rows");
  CUDA_TRY(cudaSetDevice(device));
  const int D = pad_to(width, 64), G = num_blocks;
  // the forward pass's kernel (rowops.cuh gated_fusion_rows): fp32, rows padded to D
  std::vector<float> hx(static_cast<size_t>(G) * rows * D, 0.f), hw(static_cast<size_t>(G) * D, 0.f),
      hb(static_cast<size_t>(G) * D, 0.f);
  for (int g = 0; g < G; ++g) {
    for (long long r = 0; r < rows; ++r)
      for (int k = 0; k < width; ++k)
        hx[(static_cast<size_t>(g) * rows + r) * D + k] = static_cast<float>(block_outputs[(g * rows + r) * width + k]);
    for (int k = 0; k < width; ++k) {
      hw[static_cast<size_t>(g) * D + k] = static_cast<float>(gate_w[static_cast<size_t>(g) * width + k]);
      hb[static_cast<size_t>(g) * D + k] = static_cast<float>(gate_b[static_cast<size_t>(g) * width + k]);
    }
  }
  OpBufs b;
  float *dx = b.get<float>(hx.size()), *dw = b.get<float>(hw.size()), *db = b.get<float>(hb.size()),
        *dy = b.get<float>(static_cast<size_t>(rows) * D);
  if (!dx || !dw || !db || !dy) return fail(2, "operator workspace allocation failed");
  CUDA_TRY(cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dw, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(db, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
  const long long n = rows * (D / 4);
  gated_fusion_rows<float><<<static_cast<unsigned>((n + 255) / 256), 256>>>(dx, D, rows * D, G, dw, db, dy, D,
                                                                            static_cast<int>(rows), D);
  CUDA_TRY(cudaGetLastError());
  std::vector<float> hy(static_cast<size_t>(rows) * D);
  CUDA_TRY(cudaMemcpy(hy.data(), dy, hy.size() * 4, cudaMemcpyDeviceToHost));
  for (long long r = 0; r < rows; ++r)
    for (int k = 0; k < width; ++k) out[r * width + k] = hy[static_cast<size_t>(r) * D + k];
  return 0;
}

int flame_op_block_states(FlameCtx* c, const double* history, long long hist_len, const double* candidates,
                          long long cand_count, double* out) {
  if (!c) return fail(1, "null context");
  if (hist_len < 0 || cand_count < 1) return fail(1, "candidates must be non-empty");
  if (hist_len % c->G != 0) return fail(1, "history length is not divisible by num_blocks");
  if (hist_len > c->cfg.max_history_len) return fail(1, "history length exceeds max_history_len");
  if ((hist_len > 0 && !history) || !candidates || !out) return fail(1, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  return c->precision == FLAME_BF16 ? op_block_states<__nv_bfloat16>(c, history, hist_len, candidates, cand_count, out)
                                    : op_block_states<float>(c, history, hist_len, candidates, cand_count, out);
}

int flame_op_expert_heads(FlameCtx* c, const double* fused, long long rows, double* out) {
  if (!c) return fail(1, "null context");
  if (rows < 0) return fail(1, "bad row count");
  if (rows == 0) return 0;
  if (!fused || !out) return fail(1, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  constexpr long long kChunk = 8192;  // rows per one-request executor (its list capacity bound)
  for (long long r0 = 0; r0 < rows; r0 += kChunk) {
    const long long n = rows - r0 < kChunk ? rows - r0 : kChunk;
    const double* f = fused + r0 * c->d;
    double* o = out + r0 * c->tasks;
    if (int rc = c->precision == FLAME_BF16 ? op_expert_heads<__nv_bfloat16>(c, f, n, o)
                                            : op_expert_heads<float>(c, f, n, o))
      return rc;
  }
  return 0;
}

}  // extern "C"
