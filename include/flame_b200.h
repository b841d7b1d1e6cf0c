/*
 * flame_b200.h — C ABI of the B200-native FLAME SUMI-ranker hot path.
 *
 * This is the drop-in boundary under the reference's Python operator API.
 * Each entry point replaces one piece of the reference hot path
 * (paths relative to the reference's pkg/src/flameserve/):
 *
 *   flame_create / flame_create_flmp
 *       replace  model/params.py:77-109  init_params / :154-207 load_params as
 *       the weight source of model_forward: the caller passes the fp64 arrays
 *       in iter_param_arrays order (model/params.py:112-128) or a whole FLMP
 *       file image; the library repacks them into padded, transposed (K-major)
 *       bf16 or fp32 device tensors.
 *   flame_set_table
 *       replaces the per-id feature lookup behind Service.resolve_embeddings
 *       (service.py:97-108, store.py:59-78) with a device-resident embedding
 *       table (row = item id; unknown ids decode to zero rows).
 *   flame_exec_create
 *       replaces orchestrator.py:104-133 Executor: a fixed-shape compute slot
 *       with buffers allocated once (zero steady-state allocations) bound to a
 *       run closure.  Shape = (R requests, hb_bkt history rows per
 *       request-block, c_bkt candidate rows per request).
 *   flame_exec_run / flame_exec_capture / flame_exec_replay
 *       replace Executor.bound_run -> model/forward.py:186-204 model_forward
 *       (mode FLAME_INPUT_EMBEDDINGS) and Service.resolve_embeddings +
 *       model_forward (mode FLAME_INPUT_IDS); FLAME_INPUT_GATHER_ONLY runs only
 *       the PDA feature assembly (np.unique maps + rows).  capture/replay
 *       record the same launches once into a CUDA graph and replay it.
 *
 * Conventions: 0 = ok, 1 = bad argument (Python maps to ValueError),
 * 2 = CUDA error (RuntimeError).  flame_last_error() describes the last
 * failure of the calling thread.  All work is stream-ordered on the stream
 * passed in (a cudaStream_t, or NULL for the legacy default stream).  The
 * context owns weights and workspace; the caller owns every I/O buffer bound
 * in FlameIO.  One context per device; threads may share a context as long as
 * each drives its own executor.
 */
#ifndef FLAME_B200_H
#define FLAME_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct FlameCtx FlameCtx;
typedef struct FlameExec FlameExec;

/* Mirrors model/config.py:9-19 ModelConfig field for field. */
typedef struct FlameModelDesc {
  int hidden_dim;
  int head_dim;
  int num_blocks;
  int layers_per_block;
  int ffn_dim;
  int num_tasks;
  int max_history_len;
  int max_candidates;
  unsigned long long seed;
} FlameModelDesc;

enum FlamePrecision { FLAME_BF16 = 0, FLAME_FP32 = 1 };
enum FlameInputMode { FLAME_INPUT_EMBEDDINGS = 0, FLAME_INPUT_IDS = 1, FLAME_INPUT_GATHER_ONLY = 2 };
enum FlameTableDtype { FLAME_TABLE_BF16 = 0, FLAME_TABLE_FP32 = 1 };

/* Caller-owned device buffers bound to an executor.  Unused ones may be NULL
 * (e.g. the id buffers when only embeddings are scored). Shapes use the
 * executor's R / H_bkt = num_blocks*hb_bkt / C_bkt = c_bkt. */
typedef struct FlameIO {
  const float* hist_emb;      /* [R][H_bkt][hidden_dim] fp32 */
  const float* cand_emb;      /* [R][C_bkt][hidden_dim] fp32 */
  const long long* hist_ids;  /* [R][H_bkt] int64 */
  const long long* cand_ids;  /* [R][C_bkt] int64 */
  const int* hist_len;        /* [R] actual history length H_r (multiple of num_blocks) */
  const int* cand_len;        /* [R] actual candidate count C_r (1..C_bkt) */
  const int* out_offset;      /* [R] first output row of request r */
  float* scores;              /* [sum C_r][num_tasks] fp32 */
  long long* unique_ids;      /* [2R][cap] per list: np.unique values (lists: R history, then R candidate) */
  long long* inverse;         /* [2R][cap] per list: np.unique inverse */
  int* n_unique;              /* [2R] */
  const int* active;          /* [1] slots 0..active-1 are in use this run (NULL: all R).  Read on the
                                 device, so one captured graph serves any batch size <= R: the
                                 kernels skip the rows, units and lists of the unused slots */
} FlameIO;

int flame_create(const FlameModelDesc* cfg, const double* weights_fp64, long long n_values,
                 int precision, int device, FlameCtx** out);
int flame_create_flmp(const void* flmp_bytes, long long n_bytes, int precision, int device,
                      FlameCtx** out);
int flame_destroy(FlameCtx* ctx);
int flame_set_table(FlameCtx* ctx, const float* host_table, long long num_items, int table_dtype);
/* Incremental refresh of the device item table: rows [n][hidden_dim] fp32 written
 * to table[ids[i]] on `stream` (synchronised before return).  Replaces the
 * reference's per-key cache refresh after SimulatedRemoteStore.mutate
 * (store.py:104-108, cache.py:170-357) for the device-resident table. */
int flame_update_table(FlameCtx* ctx, const long long* host_ids, const float* host_rows, long long n,
                       void* stream);
/* Same, from raw store feature values in the reference wire format (store.py:66-78:
 * hidden_dim little-endian float64 + filler): value i occupies value_len[i] bytes at
 * host_values + i * value_stride; values shorter than hidden_dim * 8 bytes decode to
 * zero rows (decode_embedding).  The decode runs on the device. */
int flame_update_table_values(FlameCtx* ctx, const long long* host_ids, const void* host_values,
                              long long value_stride, const int* host_value_len, long long n, void* stream);

/* Host staging helper: n variable-length records stored back to back in `flat`
 * (record i = lens[i] elements of elem_bytes bytes) are copied into fixed-stride
 * slots, record i at dst + i * dst_stride_bytes.  Fills an executor's pinned id /
 * row mirrors with one call per batch instead of one copy per request (the
 * reference copies each request into its executor's preallocated buffers,
 * orchestrator.py:209-213).  Returns 1 if a record exceeds its slot. */
int flame_pack_padded(void* dst, long long dst_stride_bytes, const void* flat, const long long* lens, long long n,
                      long long elem_bytes);

/* Capacity of one id list in the unique/inverse buffers: max(H_bkt, C_bkt). */
int flame_exec_list_capacity(int num_blocks, int hb_bkt, int c_bkt);
int flame_exec_create(FlameCtx* ctx, int R, int hb_bkt, int c_bkt, const FlameIO* io,
                      FlameExec** out);
int flame_exec_destroy(FlameExec* ex);
int flame_exec_run(FlameExec* ex, int input_mode, void* stream);
/* Pinned host mirrors of an executor's inputs and scores, registered once, so
 * that one flame_exec_submit per batch does the whole round trip (the
 * reference's Executor.bound_run, orchestrator.py:127-131, from the caller's
 * arrays to its scores).  Unused pointers (e.g. ids in embedding-only use) may
 * be NULL.  h_meta / d_meta: the [4][R] int32 block whose rows are the FlameIO
 * hist_len, cand_len, out_offset pointers and whose [3][0] is `active`. */
typedef struct FlameStaging {
  const void* h_meta;
  void* d_meta;
  const long long* h_hist_ids;  /* [R][H_bkt] */
  const long long* h_cand_ids;  /* [R][C_bkt] */
  const float* h_hist_emb;      /* [R][H_bkt][hidden_dim] */
  const float* h_cand_emb;      /* [R][C_bkt][hidden_dim] */
  float* h_scores;              /* [R*C_bkt][num_tasks] */
} FlameStaging;
int flame_exec_set_staging(FlameExec* ex, const FlameStaging* staging);
/* Stream-ordered on `stream`: copy the first n_req slots of the inputs of
 * input_mode and the metadata block to the device, run the pass (the CUDA graph,
 * captured on first use per input mode), copy n_score_rows score rows back, and
 * record the executor's completion event.  Returns without waiting. */
int flame_exec_submit(FlameExec* ex, int input_mode, int n_req, long long n_score_rows, void* stream);
/* Wait for (1) / poll (returns 1 done, 0 pending) the last flame_exec_submit. */
int flame_exec_wait(FlameExec* ex);
int flame_exec_query(FlameExec* ex);
int flame_exec_capture(FlameExec* ex, int input_mode, void* stream);
int flame_exec_replay(FlameExec* ex, void* stream);
/* Eager run with a CUDA event recorded on `stream` before every launch.
 * Fills, per launch i < max_launches: ms[i] (device duration), names[64*i]
 * (NUL-terminated kernel role), flops[i] / bytes[i] (algorithmic FLOPs and
 * bytes of that launch).  Returns the number of launches (>= 0) or
 * -status on failure.  Any output pointer may be NULL. */
int flame_exec_profile(FlameExec* ex, int input_mode, void* stream, int max_launches, float* ms,
                       char* names, double* flops, double* bytes);
/* Number of kernel launches one run issues (for the bench's gpu_launches). */
int flame_exec_launch_count(FlameExec* ex, int input_mode);
/* Device pointer of an internal workspace tensor, for parity debugging:
 * "Eh", "Ec" (assembled fp32 rows), "qkv", "attn", "fused". */
void* flame_exec_workspace(FlameExec* ex, const char* name);

/* Synchronous device-to-host copy (test / debugging helper). */
int flame_copy_to_host(void* dst_host, const void* src_device, long long bytes);

/* ---------------------------------------------------------------- operators
 * The reference's operator-level API (model/__init__.py:4-31) over host fp64
 * arrays, computed on the device (synchronous; results written to `out`).
 *
 * flame_op_attention_sumi replaces model/attention.py:118-146
 *   attention_sumi_candidates (candidates_only = 1: q is (num_heads, C, head_dim)
 *   with C = seq_len - hist_len, out likewise) and :149-178 attention_sumi
 *   (candidates_only = 0: q and out are (num_heads, seq_len, head_dim)); k / v are
 *   (num_heads, seq_len, head_dim).  Runs the forward pass's SUMI attention
 *   kernels (bf16 tcgen05 or fp32 verification); head_dim <= 64.
 * flame_op_attention_masked replaces attention.py:55-67 attention_naive /
 *   :70-115 attention_tiled: one head, (seq_len, head_dim) q / k / v and an
 *   arbitrary seq_len x seq_len permission matrix (1 = allowed), in fp64.
 * flame_op_rows replaces forward.py:33-47 gelu / sigmoid / layer_norm and
 *   attention.py:28-36 masked_softmax_rows, fp64, rows x width row-major
 *   (layer_norm: scale / shift of length width).
 * flame_op_gated_fusion replaces forward.py:143-156 gated_fusion:
 *   block_outputs [num_blocks][rows][width], gate_w / gate_b [num_blocks][width].
 * flame_op_block_states replaces forward.py:75-140 block_forward for every block
 *   of the context at once: out [num_blocks][cand_count][hidden_dim] = each
 *   block's final candidate rows over its contiguous history split.
 * flame_op_expert_heads replaces forward.py:159-166 expert_heads:
 *   fused [rows][hidden_dim] -> out [rows][num_tasks]. */
enum FlameRowOp { FLAME_OP_GELU = 0, FLAME_OP_SIGMOID = 1, FLAME_OP_LAYER_NORM = 2, FLAME_OP_SOFTMAX = 3 };
int flame_op_attention_sumi(int precision, int device, int num_heads, int seq_len, int head_dim, int hist_len,
                            int candidates_only, double temperature, const double* q, const double* k,
                            const double* v, double* out);
int flame_op_attention_masked(int device, int seq_len, int head_dim, double temperature, const double* q,
                              const double* k, const double* v, const unsigned char* allowed, double* out);
int flame_op_rows(int op, int device, long long rows, int width, const double* x, const double* scale,
                  const double* shift, double* out);
int flame_op_gated_fusion(int device, int num_blocks, long long rows, int width, const double* block_outputs,
                          const double* gate_w, const double* gate_b, double* out);
int flame_op_block_states(FlameCtx* ctx, const double* history, long long hist_len, const double* candidates,
                          long long cand_count, double* out);
int flame_op_expert_heads(FlameCtx* ctx, const double* fused, long long rows, double* out);

const char* flame_last_error(void);
int flame_device_sm_count(int device);

#ifdef __cplusplus
}
#endif

#endif /* FLAME_B200_H */
