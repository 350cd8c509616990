/*
 * egt_b200.h -- C-ABI boundary of the B200-native SparseGemv hot path.
 *
 * The reference (arXiv 2605.11582 "egt", a C++20 CPU library) has no FFI; its
 * API is the C++ header surface of egt_core (proj/include/egt/packed.hpp,
 * compress.hpp, model.hpp, decode.hpp).  This header is the thin C layer that
 * the C++ drop-in (paper_2605_11582_b200/csrc/host/, namespace egt_b200)
 * calls, and that any other host language (ctypes, cgo, JNI) can bind.
 * Plain pointers and sizes only; no C++ or torch types cross it.
 *
 * Reference interfaces replaced (paths relative to the reference's proj/):
 *   egt_dev_packed_create     <- PackedSparseMatrix (include/egt/packed.hpp:37-67)
 *                                + check_packed / offset checks
 *                                (src/packed.cpp:145-184), done ONCE at upload
 *   egt_dev_dense_i4_create   <- QuantizedMatrix with an all-kept mask
 *                                (include/egt/compress.hpp:59-71), the
 *                                quant_dense_gemv arm (src/packed.cpp:266-281)
 *   egt_spmv (M = 1)          <- Vector spmv(const PackedSparseMatrix&, const
 *                                Vector&) (include/egt/packed.hpp:83-85,
 *                                src/packed.cpp:211-220)
 *   egt_spmv (M > 1)          <- the M-row X * W^T products of forward_impl
 *                                (src/model.cpp:156-158,186,188,190,195)
 *   egt_dequant               <- UnpackResult unpack(const PackedSparseMatrix&)
 *                                (include/egt/packed.hpp:81, src/packed.cpp:197-209)
 *   egt_spmv_host             <- spmv with host vectors (the drop-in call)
 *   egt_host_*                <- the host encoder (fit_group / quantize_matrix /
 *                                pack / footprint, src/compress.cpp:77-228,
 *                                src/packed.cpp:27-141,222-240), C++ in
 *                                csrc/host, byte-identical to the reference.
 *
 * Error contract (include/egt/common.hpp:37-47, tools/egt_main.cpp:119-139):
 *   EGT_EINVAL    <- std::invalid_argument (bad argument / shape)
 *   EGT_EFORMAT   <- FormatError (malformed packed stream)
 *   EGT_EINTERNAL <- InvariantError and anything else
 *   EGT_ECUDA     <- a CUDA runtime failure (message has the CUDA error)
 * egt_last_error() returns the thread's last message, which keeps the
 * reference's wording ("input length differs from columns", "offsets",
 * "keeps", "dense", ...).
 *
 * Threading: device handles are immutable after create; concurrent egt_spmv
 * calls on one handle are safe.  Split-K workspaces are per stream.
 */
#ifndef EGT_B200_H
#define EGT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EGT_ABI_VERSION 1

#if defined(__GNUC__)
#define EGT_API __attribute__((visibility("default")))
#else
#define EGT_API
#endif

typedef enum egt_status {
  EGT_OK = 0,
  EGT_EINVAL = 1,
  EGT_EFORMAT = 2,
  EGT_EINTERNAL = 3,
  EGT_ECUDA = 4
} egt_status;

/* PackedValueKind (packed.hpp:32-35). */
enum { EGT_KIND_F32 = 0, EGT_KIND_INT4 = 1 };

/* Device storage formats. */
enum {
  EGT_FMT_I4_SP24 = 0,  /* INT4 codes + 2bit-CSR, 2:4 */
  EGT_FMT_I4_SP14 = 1,  /* INT4 codes + 2bit-CSR, 1:4 */
  EGT_FMT_I4_DENSE = 2, /* dense INT4 (quant_dense_gemv arm) */
  EGT_FMT_F16_SP24 = 3, /* sparse-FP16 2bit-CSR, 2:4 */
  EGT_FMT_F16_SP14 = 4  /* sparse-FP16 2bit-CSR, 1:4 */
};

/* Execution paths. */
enum {
  EGT_PATH_TILED = 0,  /* fragment-tiled stream, mma.sp tensor-core gather */
  EGT_PATH_GENERAL = 1 /* reference stream as is, CUDA-core kernel (any group size) */
};

EGT_API int egt_abi_version(void);
EGT_API const char* egt_last_error(void);

/* Flat view of a host PackedSparseMatrix (packed.hpp:37-67). kind selects
 * value_bytes + group tables (INT4) or values (F32; stored as FP16 on device). */
typedef struct egt_packed_view {
  uint8_t n, m;
  uint32_t rows, cols;
  uint8_t kind;
  const uint16_t* index_words; size_t n_index_words;
  const uint8_t* value_bytes;  size_t n_value_bytes;
  const uint32_t* group_sizes; size_t n_group_sizes;
  const uint32_t* group_offsets; size_t n_group_offsets;
  const float* scales;         size_t n_scales;
  const uint8_t* zero_points;  size_t n_zero_points;
  const float* values;         size_t n_values;
} egt_packed_view;

/* Flat view of a QuantizedMatrix with every position retained (dense INT4). */
typedef struct egt_quant_view {
  uint32_t rows, cols;
  const uint32_t* group_sizes;   /* rows */
  const uint32_t* group_offsets; /* rows + 1 */
  const float* scales;           size_t n_scales;
  const uint8_t* zero_points;    /* n_scales */
  const uint8_t* codes;          size_t n_codes; /* rows*cols, one per byte */
} egt_quant_view;

typedef struct egt_dev_packed egt_dev_packed; /* opaque, immutable */

typedef struct egt_dev_packed_info {
  uint32_t rows, cols;
  uint8_t n, m, kind, format, path;
  uint64_t device_bytes;      /* bytes held on the device for this handle */
  uint64_t algorithmic_bytes; /* weight-side bytes one M=1 call must read */
  uint64_t nnz;
} egt_dev_packed_info;

/* Validates (check_packed + in-group offset order, packed.cpp:145-184) and
 * uploads.  stream may be NULL (legacy default stream); the call is
 * synchronous.  Device memory is allocated on the current device.
 * Sparse-FP (EGT_KIND_F32) values are stored as fp16 on the device: values
 * fp16 cannot hold exactly (precision or |v| > 65504) are rejected with
 * EGT_EINVAL unless egt_dev_packed_create_ex is given EGT_UPLOAD_ROUND_FP16,
 * which rounds them to nearest (the reference keeps f32, packed.hpp:33). */
EGT_API egt_status egt_dev_packed_create(const egt_packed_view* view, void* stream, egt_dev_packed** out);
#define EGT_UPLOAD_ROUND_FP16 1u
EGT_API egt_status egt_dev_packed_create_ex(const egt_packed_view* view, uint32_t flags, void* stream,
                                           egt_dev_packed** out);

/* Dense INT4 layer (quant_dense_gemv semantics, packed.cpp:266-281). */
EGT_API egt_status egt_dev_dense_i4_create(const egt_quant_view* view, void* stream, egt_dev_packed** out);

/* Zero-copy row shard [r0, r1).  r0 % 16 == 0 and (r1 % 16 == 0 or r1 == rows)
 * on the tiled path.  The shard keeps the parent's storage alive. */
EGT_API egt_status egt_dev_packed_slice_rows(const egt_dev_packed* h, uint32_t r0, uint32_t r1,
                                     egt_dev_packed** out);

EGT_API egt_status egt_dev_packed_destroy(egt_dev_packed* h);
EGT_API egt_status egt_dev_packed_query(const egt_dev_packed* h, egt_dev_packed_info* info);

/* Y[M x rows] (row stride ldy) = X[M x cols] (row stride ldx) * W^T on the
 * device, stream-ordered and asynchronous.  M == 1 is the SparseGemv. */
EGT_API egt_status egt_spmv(const egt_dev_packed* h, const float* x_dev, float* y_dev, uint32_t M,
                    uint32_t ldx, uint32_t ldy, void* stream);

/* egt_spmv with flags.  EGT_SPMV_INDEPENDENT: x is not written by the
 * kernel issued immediately before this one on the stream, so the product may
 * overlap that kernel entirely (it still completes after it).  Typical use:
 * the Q, K, V (or gate/up) products of one decode step. */
#define EGT_SPMV_INDEPENDENT 1u
/* egt_spmv_fused: apply silu (model.cpp:80-84) to the output instead of the
 * next product applying it to its input (each element once, not per CTA). */
#define EGT_SPMV_OUTPUT_SILU 2u
/* Input transforms of fused products (egt_spmv_fused). */
#define EGT_INPUT_NONE 0u
#define EGT_INPUT_RMSNORM 1u /* x / sqrt(mean(x^2) + eps) over the whole vector */
#define EGT_INPUT_SILU 2u    /* x / (1 + exp(-x)) */
EGT_API egt_status egt_spmv_ex(const egt_dev_packed* h, const float* x_dev, float* y_dev, uint32_t M,
                               uint32_t ldx, uint32_t ldy, uint32_t flags, void* stream);

/* egt_spmv_ex with the forward_impl glue fused (model.cpp:155-190):
 * Y = residual + f(X) * W^T, f = EGT_INPUT_NONE / RMSNORM (per token, eps) /
 * SILU (the EGT_INPUT_* constants below).  residual may be NULL or equal y
 * (row stride ldr).  Tiled path only (else EGT_EINVAL).  With
 * EGT_SPMV_INDEPENDENT neither x nor residual may be written by the
 * immediately preceding kernel on the stream.  l2_next (may be NULL): the
 * matrix the NEXT product will read; its weights are prefetched into L2
 * while this product runs (decode chains, M <= 16). */
EGT_API egt_status egt_spmv_fused(const egt_dev_packed* h, const float* x_dev, float* y_dev, uint32_t M,
                                  uint32_t ldx, uint32_t ldy, const float* residual_dev, uint32_t ldr,
                                  uint32_t input, float eps, uint32_t flags, const egt_dev_packed* l2_next,
                                  void* stream);

/* One launch over n <= 3 matrices of one shape sharing x (the decode step's
 * Q, K, V): ys[i] = f(x) * W_i^T, M = 1, same transform / flags semantics as
 * egt_spmv_fused (no residual).  rows must be a multiple of 16 when n > 1. */
EGT_API egt_status egt_spmv_fused_multi(const egt_dev_packed* const* hs, uint32_t n, const float* x_dev,
                                        float* const* ys_dev, uint32_t input, float eps, uint32_t flags,
                                        void* stream);

/* M tokens through n <= 3 matrices of one shape sharing x (the verify pass's
 * Q, K, V, forward_impl model.cpp:155-158): ys[i] (M x rows, row stride ldy)
 * = f(x) * W_i^T with f = identity or EGT_INPUT_RMSNORM (per token, eps).
 * Many tokens run as ONE tcgen05 launch over the n matrices with one x
 * preparation (the rmsnorm folded into it); otherwise one product per matrix. */
EGT_API egt_status egt_spmm_multi(const egt_dev_packed* const* hs, uint32_t n, const float* x_dev, uint32_t M,
                                  uint32_t ldx, float* const* ys_dev, uint32_t ldy, uint32_t input, float eps,
                                  void* stream);

/* Same as egt_spmv with host buffers: H2D of x, the product, D2H of y, and a
 * stream synchronize.  x_len must equal cols (else EGT_EINVAL with the
 * reference's "spmv: input length differs from columns"). */
EGT_API egt_status egt_spmv_host(const egt_dev_packed* h, const float* x_host, size_t x_len,
                         float* y_host, void* stream);

/* Bit-exact unpack on the device: w_dev[rows x cols] f32 (dropped -> 0) and,
 * if mask_dev != NULL, the keep bitmap (PruneMask bits, LSB-first; the
 * buffer must be 4-byte aligned and hold ceil(rows*cols/32)*4 bytes, of which
 * the first ceil(rows*cols/8) are the bitmap).  Stream-ordered. */
EGT_API egt_status egt_dequant(const egt_dev_packed* h, float* w_dev, uint8_t* mask_dev, void* stream);

/* Enables/disables programmatic dependent launch for egt_spmv launches on
 * this thread (default on).  With PDL a GEMV issues its weight loads before
 * the previous kernel in the stream finishes. */
EGT_API void egt_set_pdl(int enabled);

/* Tuning hook: force the tiled launch plan for subsequent egt_spmv calls on
 * this thread (row tiles per CTA, K splits, consumer warps, stage depth,
 * k-quads per stage; 0 = automatic for that field, rb = 0 restores the
 * automatic planner).  Used by tools/plan_sweep.py. */
/* Tuning hook: with EGT_TILED_TRACE set, every SparseGemv launch stamps
 * globaltimer ns into slot (launch index % 4096) x 8: CTA-0 start, past the
 * PDL wait, x staged, compute done, last CTA exit, ~first CTA start.  Copies
 * n values out (and zeroes the buffer if reset); nonzero if tracing is off. */
EGT_API int egt_tune_read_trace(unsigned long long* host, size_t n, int reset);
EGT_API void egt_tune_force_plan(int rb, int s, int nw, int nst, int ch);

/* Number of kernels the library has launched on this thread (a counter the
 * benchmark reads to report gpu_launches). */
EGT_API uint64_t egt_launch_count(void);

/* ---------------- verify substrate: the multi-token pass -----------------
 * ModelConfig (model.hpp:32-43) and forward (model.hpp:71-72,
 * model.cpp:118-202) over packed layers; prefix-tree verification
 * (verify_parallel, decode.hpp:163-170, decode.cpp:336-421). */
typedef struct egt_model_config {
  uint32_t vocab_size, d_model, n_layers, n_heads, d_ff, max_positions;
} egt_model_config;

typedef struct egt_model egt_model; /* opaque; layer handles must outlive it */

/* embedding: host [vocab x d_model] f32.  layers: n_layers*6 handles in the
 * order wq, wk, wv, wo, ff1, ff2 (linear_layer_names, model.cpp:379-388),
 * any mixed-dispatch format; head: [vocab x d_model]. */
EGT_API egt_status egt_model_create(const egt_model_config* cfg, const float* embedding,
                                    const egt_dev_packed* const* layers, const egt_dev_packed* head,
                                    void* stream, egt_model** out);
EGT_API egt_status egt_model_destroy(egt_model* m);

/* logits_dev[M x vocab] = forward(tokens, mask, positions); host tokens /
 * positions (int32) and visibility bits (bit q*M+k = query q sees key k,
 * LSB-first).  A query row with no visible key gets zero attention output. */
EGT_API egt_status egt_forward(const egt_model* m, const int32_t* tokens, const int32_t* positions,
                               const uint8_t* mask_bits, uint32_t M, float* logits_dev, void* stream);

/* The verify pass's forward with the prefix-tree mask built on the device
 * from the compact encoding flatten_subtree already produces (SURVEY 8(f)
 * row 4; decode.cpp:209-299) instead of an M x M host bitmap: rows
 * [b*padded_len, (b+1)*padded_len) are beam b's committed block (left-padded
 * to committed_len[b] tokens, causal), then one row per flattened node f
 * (DFS order) that sees its beam's committed block, its ancestors (parent[f],
 * -1 for a root, always an earlier node of the same beam) and itself.
 * M = n_beams * padded_len + n_nodes; tokens / positions as egt_forward. */
typedef struct egt_tree_view {
  uint32_t n_beams, padded_len;
  const uint32_t* committed_len; /* [n_beams] */
  uint32_t n_nodes;
  const int32_t* parent;         /* [n_nodes] */
  const uint32_t* beam;          /* [n_nodes] */
} egt_tree_view;
EGT_API egt_status egt_forward_tree(const egt_model* m, const int32_t* tokens, const int32_t* positions,
                                    const egt_tree_view* tree, float* logits_dev, void* stream);

/* KV pool for the KV-cached trie-constrained beam step (
 * the reference recomputes every prefix, decode.cpp:122-190): the keys and
 * values of committed rows, [n_layers][capacity][d_model], a row written once
 * and shared by every beam whose prefix holds it. */
typedef struct egt_kv_pool egt_kv_pool;
EGT_API egt_status egt_kv_pool_create(const egt_model* m, uint32_t capacity, egt_kv_pool** out);
EGT_API egt_status egt_kv_pool_destroy(egt_kv_pool* p);
/* forward over M rows storing each row's keys / values at pool row
 * out_rows[i].  With key lists (key_ptr [M+1], key_rows): row i attends to
 * pool rows key_rows[key_ptr[i] .. key_ptr[i+1]) then itself (its causal
 * prefix, position order) -- no mask.  Without: mask_bits as egt_forward. */
EGT_API egt_status egt_forward_kv(const egt_model* m, egt_kv_pool* pool, const int32_t* tokens,
                                  const int32_t* positions, uint32_t M, const uint8_t* mask_bits,
                                  const uint32_t* out_rows, const uint32_t* key_ptr, const uint32_t* key_rows,
                                  float* logits_dev, void* stream);

/* out[i] = src_dev[rows[i] * ld + cols[i]] (host index lists, host output). */
EGT_API egt_status egt_gather(const float* src_dev, uint64_t ld, const uint32_t* rows,
                              const uint32_t* cols, uint32_t n, float* out, void* stream);

/* PrefixTrie (trie.hpp:72-90) as parent links: node 0 is the root, parents
 * precede children, children are visited in ascending token order. */
typedef struct egt_trie_view {
  uint32_t n_nodes;
  const uint32_t* token;
  const uint32_t* parent; /* parent[0] ignored */
  const int64_t* payload; /* kNoPayload = -1 */
} egt_trie_view;

/* DecodeSession (decode.hpp:43-50): prompt + beams, each beam's generated
 * tokens concatenated in beam order. */
typedef struct egt_session_view {
  const int32_t* prompt;
  uint32_t prompt_len;
  uint32_t n_beams;
  const uint32_t* beam_node;
  const double* beam_log_prob;
  const uint32_t* beam_len;
  const int32_t* beam_tokens;
} egt_session_view;

typedef struct egt_verify_out {
  uint32_t n_selected;    /* <= beam_size */
  double* score;          /* [beam_size] */
  int64_t* payload;       /* [beam_size] */
  uint32_t* beam;         /* [beam_size] */
  uint32_t* len;          /* [beam_size] tokens per selected sequence */
  int32_t* tokens;        /* [beam_size * tokens_stride] */
  uint32_t tokens_stride;
  uint32_t flattened_nodes;
  uint32_t rows;          /* M of the forward pass */
} egt_verify_out;

/* flatten_subtree + build_tree_mask + verify_parallel (decode.cpp:209-421):
 * one masked forward over every remaining node of the beams' subtrees, the
 * trie-restricted log-softmax, B-score recursion, leaf ranking (ties: beam,
 * then flat index) and traceback of the top beam_size. */
EGT_API egt_status egt_verify_parallel(const egt_model* m, const egt_trie_view* trie,
                                       const egt_session_view* session, int beam_size,
                                       egt_verify_out* out, void* stream);

/* decode (decode.cpp:423-483): trie-constrained beam steps (one block-diagonal
 * forward each) until the cost model fires (mode 1), a forced depth is
 * reached (mode 2) or every beam is finished (mode 0, autoregressive); then
 * one parallel verification.  stats = {steps, forward_passes, trigger_step,
 * flattened_nodes}. */
typedef struct egt_decode_options {
  int beam_size;
  int mode; /* 0 autoregressive, 1 ptpv, 2 ptpv forced at depth */
  int forced_depth;
  double t_step, alpha, beta; /* CostModel, seconds */
  uint64_t node_cap;
  int kv_cache; /* 1: constrained steps on a KV pool (egt_forward_kv), one new row per beam per step */
} egt_decode_options;

EGT_API egt_status egt_decode(const egt_model* m, const egt_trie_view* trie, const int32_t* prompt,
                              uint32_t prompt_len, const egt_decode_options* opt, egt_verify_out* out,
                              int32_t stats[4], void* stream);

EGT_API egt_status egt_model_query(const egt_model* m, egt_model_config* cfg);

/* ---------------- KV-cached batch-1 decode loop ---------------------------
 * The reference's decode recomputes the whole prefix each step
 * (decode.cpp:122-190 -> forward, model.cpp:118-202); the decoder runs one
 * token per step against a KV cache -- the same attention arithmetic
 * (model.cpp:161-184) with every linear layer an M = 1 SparseGemv and the
 * rmsnorm / silu / residual glue fused into the products.  Position and
 * token live in device memory, so a step is one CUDA graph replay with no
 * host round trip.  Greedy (argmax, ties -> lowest id) after the prompt.
 * Every layer and the head must be on the tiled path; head dim 16/32/64/128. */
typedef struct egt_decoder egt_decoder;
EGT_API egt_status egt_decoder_create(const egt_model* m, uint32_t max_len, egt_decoder** out);
/* Resets the position to 0 with the prompt's first token; the next
 * prompt_len - 1 steps consume the rest of the prompt. */
EGT_API egt_status egt_decoder_start(egt_decoder* d, const int32_t* prompt, uint32_t prompt_len, void* stream);
/* n_steps graph replays, stream-ordered after `stream` (asynchronous). */
EGT_API egt_status egt_decoder_step(egt_decoder* d, uint32_t n_steps, void* stream);
/* Synchronous read-back: the position t reached (positions [0, t) have been
 * run), tokens_host[0..t] (t = the pending next token; at most n entries),
 * and (optionally) the last step's logits into logits_dev [vocab]. */
EGT_API egt_status egt_decoder_read(const egt_decoder* d, int32_t* tokens_host, uint32_t n, uint32_t* position,
                                    float* logits_dev, void* stream);
EGT_API egt_status egt_decoder_destroy(egt_decoder* d);

/* ---------------- planning around the hot path (host) ----------------
 * plan_sparsity (compress.cpp:298-326): patterns[l] = 2 (2:4) for the
 * ceil(rho_s * L) layers of highest mean(score) / mean(|w|) (ties keep layer
 * order), 1 (1:4) for the rest.  scores / weights: row-major f32. */
EGT_API egt_status egt_host_plan_sparsity(uint32_t n_layers, const uint32_t* rows, const uint32_t* cols,
                                          const float* const* scores, const float* const* weights, double rho_s,
                                          uint8_t* patterns);
/* CostModelEstimator (decode.cpp:84-120): EMA 0.9 of step times, 32-sample
 * least squares of verify time over node count.  egt_measure_cost_model
 * feeds it device-measured (CUDA event) times of this model's forward. */
typedef struct egt_cost_estimator egt_cost_estimator;
EGT_API egt_status egt_cost_estimator_create(double t_step, double alpha, double beta, egt_cost_estimator** out);
EGT_API egt_status egt_cost_estimator_observe_step(egt_cost_estimator* e, double seconds);
EGT_API egt_status egt_cost_estimator_observe_verify(egt_cost_estimator* e, uint64_t nodes, double seconds);
EGT_API egt_status egt_cost_estimator_model(const egt_cost_estimator* e, double out[3]); /* t_step, alpha, beta */
EGT_API egt_status egt_cost_estimator_destroy(egt_cost_estimator* e);
/* Times (CUDA events, reps each, after one warm-up) this model's constrained
 * step forward (n_beams beams of prompt_len + 1 committed rows) and its
 * verify forward over every node count in node_counts (a random tree under
 * n_beams committed blocks), feeding observe_step / observe_verify. */
EGT_API egt_status egt_measure_cost_model(const egt_model* m, uint32_t prompt_len, uint32_t n_beams,
                                          const uint32_t* node_counts, uint32_t n_counts, int reps,
                                          egt_cost_estimator* e, void* stream);
/* estimate_trigger (decode.cpp:192-207) and flatten_subtree + build_tree_mask
 * (decode.cpp:209-299) on host views (no device work). */
EGT_API egt_status egt_host_estimate_trigger(const egt_trie_view* trie, const egt_session_view* session,
                                             double t_step, double alpha, double beta, uint64_t node_cap,
                                             int* trigger, double* saving);
EGT_API egt_status egt_host_tree_mask(const egt_trie_view* trie, const egt_session_view* session, uint32_t cap_nodes,
                                      uint32_t* n_nodes, uint32_t* fn_token, int32_t* fn_parent, uint32_t* fn_depth,
                                      uint32_t* fn_trie, uint32_t* fn_beam, uint32_t cap_rows, uint32_t* n_rows,
                                      int32_t* tokens, int32_t* positions, uint8_t* vis_bits, size_t cap_bits,
                                      uint32_t* padded_len, uint32_t* flat_offset);

/* y = W x for a dense row-major f32 W (device pointers): the mixed
 * dispatch's (dense, !quant) baseline arm, which the reference densifies
 * (materialize_model, compress.cpp:395-414), and bench_spmv's dense-fp. */
EGT_API egt_status egt_gemv_f32(const float* w_dev, const float* x_dev, float* y_dev, uint32_t rows,
                                uint32_t cols, void* stream);

/* bench_spmv (packed.cpp:310-383) on the device: per shape the reference's
 * seeded U(-1,1) W and x (mt19937_64, seed + 0x9e3779b97f4a7c15 (si + 1)),
 * g = min(64, cols), magnitude masks; variants dense-fp, quant-dense,
 * packed-2:4, packed-1:4; one warm-up, then reps products each timed with
 * CUDA events (device ns per product, inputs resident); bytes = the
 * reference's analytic weight-side bytes.  Writes bench_csv's text
 * (packed.cpp:385-393) into csv (cap bytes, NUL-terminated); *len = its
 * length.  EGT_EINVAL with the reference's messages for bad shapes / reps. */
EGT_API egt_status egt_bench_spmv(const uint32_t* rows, const uint32_t* cols, uint32_t n_shapes, int reps,
                                  uint64_t seed, char* csv, size_t cap, size_t* len);

/* ---------------- GPU compression ----------------------
 * The step before the path on the device (re-compressing 7B/70B layers),
 * byte-identical to the host encoder and the reference.  All pointers are
 * device pointers except group_sizes (host, one per row); stream-ordered. */
/* importance_scores (compress.cpp:230-244): |w| x_norms[c] + |w| grad_abs. */
EGT_API egt_status egt_gpu_importance(const float* w_dev, const float* x_norms_dev, const float* grad_abs_dev,
                                      uint32_t rows, uint32_t cols, float* scores_dev, void* stream);
/* prune_nm (compress.cpp:246-278): PruneMask bitmap (ceil(rows*cols/8)
 * bytes) keeping the min(n, #positive) top scores of every group of m = 4
 * columns, ties to the lower column. */
EGT_API egt_status egt_gpu_prune_nm(const float* scores_dev, uint32_t rows, uint32_t cols, int n, int m,
                                    uint8_t* mask_dev, void* stream);
/* Device arrays in the reference's stream layout (may be NULL members except
 * index_words / value_bytes): ceil(nnz/8) u16, ceil(nnz/2) bytes, rows + 1,
 * groups, groups. */
typedef struct egt_gpu_packed_out {
  uint16_t* index_words;
  uint8_t* value_bytes;
  uint32_t* group_offsets;
  float* scales;
  uint8_t* zero_points;
} egt_gpu_packed_out;
/* quantize_matrix(w, group_sizes, mask) + pack(mask, q, n, 4)
 * (compress.cpp:157-197, packed.cpp:92-128) on the device: the exact-n check
 * with the reference's "keeps" message, the group fit in double, the codes
 * and the 2bit-CSR index stream.  raw_out (may be NULL) receives the
 * reference-layout arrays; out (may be NULL) the device matrix, as
 * egt_dev_packed_create would build it from those arrays. */
EGT_API egt_status egt_gpu_quantize_pack(const float* w_dev, const uint8_t* mask_dev, uint32_t rows,
                                         uint32_t cols, int n, const uint32_t* group_sizes,
                                         const egt_gpu_packed_out* raw_out, void* stream,
                                         egt_dev_packed** out);

/* ---------------- row shards with a fused all-gather ---------
 * Replaces the NCCL all-gather after a row-sharded spmv (the reference is
 * single-process: spmv packed.cpp:211-220 over the whole matrix).  Each rank
 * owns one peer buffer: a 512-byte control block (arrival counters of up to
 * 8 ranks, a gather sequence number, a done counter, an error word) followed
 * by y (M x ldy floats, the FULL output).  Buffers are exported with CUDA IPC
 * handles (64 opaque bytes, exchanged by the caller, e.g. over
 * torch.distributed) and opened by every other rank; a peer group lists all
 * ranks' buffers in rank order (this rank's own pointer at `rank`).
 * egt_spmv_allgather runs the shard's product and stores every y row into
 * every rank's buffer over NVLink; its last CTA signals the peers and waits
 * until all ranks' slices have landed here, so the gathered y is complete
 * when the kernel is.  EGT_PEER_NOWAIT skips that wait (then egt_peer_wait
 * must follow, e.g. when several ranks share one GPU in a test).  A wait
 * bounded at 2 s records a timeout that egt_peer_group_check reports. */
#define EGT_PEER_NOWAIT 4u
#define EGT_PEER_CTRL_BYTES 512u
#define EGT_MAX_PEERS 8u
typedef struct egt_ipc_handle {
  uint8_t bytes[64];
} egt_ipc_handle;
typedef struct egt_peer_group egt_peer_group; /* opaque; buffers must outlive it */
EGT_API egt_status egt_peer_buffer_alloc(size_t y_floats, void** buf_dev, egt_ipc_handle* handle);
EGT_API egt_status egt_peer_buffer_free(void* buf_dev);
EGT_API egt_status egt_peer_buffer_open(const egt_ipc_handle* handle, void** buf_dev);
EGT_API egt_status egt_peer_buffer_close(void* buf_dev);
EGT_API egt_status egt_peer_group_create(uint32_t world, uint32_t rank, void* const* bufs_dev,
                                         egt_peer_group** out);
EGT_API egt_status egt_peer_group_destroy(egt_peer_group* g);
/* The gathered output in this rank's buffer (M x ldy floats). */
EGT_API float* egt_peer_group_y(const egt_peer_group* g);
/* y rows [row0, row0 + shard.rows) of every token, gathered on all ranks.
 * flags: EGT_SPMV_INDEPENDENT, EGT_PEER_NOWAIT.  Tiled path only. */
EGT_API egt_status egt_spmv_allgather(const egt_dev_packed* shard, const float* x_dev, uint32_t M,
                                      uint32_t ldx, egt_peer_group* g, uint32_t row0, uint32_t ldy,
                                      uint32_t flags, void* stream);
/* Stream-ordered wait for every rank's current slice (after EGT_PEER_NOWAIT). */
EGT_API egt_status egt_peer_wait(egt_peer_group* g, void* stream);
/* Synchronizes the device; EGT_EINTERNAL ("peer wait timed out") if a wait
 * gave up. */
EGT_API egt_status egt_peer_group_check(egt_peer_group* g);

/* ---------------- EGTQ compressed-model files -> device layers ------------
 * parse_compressed (egtq_io.cpp:221-235, read_layer :110-210) with the
 * reference's checks and FormatError messages ("<context>: ..."); upload is
 * the mixed dispatch on the layer's (pattern, storage) keys without
 * re-packing: the file's kept INT4 codes are the device stream's value bytes
 * and its (verified) index section the index words.  Dense fp layers are not
 * on the SparseGemv path (EGT_EINVAL). */
typedef struct egt_egtq egt_egtq;
typedef struct egt_egtq_layer_info {
  const char* name;          /* valid while the egt_egtq lives */
  uint8_t pattern;           /* SparsityPattern: 0 dense, 1 one-of-four, 2 two-of-four */
  uint8_t has_quant;         /* 1 INT4 codes + group tables, 0 fp values */
  uint8_t has_index;         /* the file carried the 2bit-CSR index section */
  uint32_t rows, cols;
} egt_egtq_layer_info;
EGT_API egt_status egt_egtq_parse(const uint8_t* bytes, size_t n, const char* context, egt_egtq** out);
EGT_API uint32_t egt_egtq_layer_count(const egt_egtq* e);
EGT_API egt_status egt_egtq_query(const egt_egtq* e, uint32_t i, egt_egtq_layer_info* info);
EGT_API egt_status egt_egtq_upload(const egt_egtq* e, uint32_t i, void* stream, egt_dev_packed** out);
/* flags: EGT_UPLOAD_ROUND_FP16 (sparse-FP layers whose f32 values fp16
 * cannot hold exactly are rounded instead of rejected) */
EGT_API egt_status egt_egtq_upload_ex(const egt_egtq* e, uint32_t i, uint32_t flags, void* stream,
                                      egt_dev_packed** out);
EGT_API egt_status egt_egtq_destroy(egt_egtq* e);

/* ---------------- host encoder (C++; byte-identical to the reference) ----
 * Masks are PruneMask bitmaps (bit r*cols+c, LSB-first). */

/* fit_group (compress.cpp:77-90). */
EGT_API void egt_host_fit_group(const double* values, size_t count, float* scale, uint8_t* zero_point);

/* Number of quant groups sum_r ceil(cols/g_r); 0 if some g_r == 0. */
EGT_API size_t egt_host_group_count(uint32_t rows, uint32_t cols, const uint32_t* group_sizes);

/* quantize_matrix (compress.cpp:157-208). mask_bits NULL = all retained.
 * group_offsets[rows+1], scales/zero_points[group_count], codes[rows*cols]. */
EGT_API egt_status egt_host_quantize(const float* w, uint32_t rows, uint32_t cols,
                             const uint32_t* group_sizes, const uint8_t* mask_bits,
                             uint32_t* group_offsets, float* scales, uint8_t* zero_points,
                             uint8_t* codes, size_t* n_codes);

/* pack(mask, QuantizedMatrix, n, m) (packed.cpp:92-128).  codes are dense
 * (rows*cols, dense_codes=1) or kept-only.  words[ceil(nnz/8)],
 * value_bytes[ceil(nnz/2)]. */
EGT_API egt_status egt_host_pack_int4(const uint8_t* mask_bits, uint32_t rows, uint32_t cols, int n,
                              int m, const uint8_t* codes, size_t n_codes, int dense_codes,
                              uint16_t* words, size_t* n_words, uint8_t* value_bytes,
                              size_t* n_value_bytes);

/* pack(mask, Matrix, n, m) (packed.cpp:130-141): words + kept values. */
EGT_API egt_status egt_host_pack_f32(const uint8_t* mask_bits, uint32_t rows, uint32_t cols, int n, int m,
                             const float* w, uint16_t* words, size_t* n_words, float* values,
                             size_t* n_values);

/* footprint (packed.cpp:222-240): out = {index, value, scale, packed,
 * baseline} bytes. */
EGT_API egt_status egt_host_footprint(const egt_packed_view* view, uint64_t out[5], double* ratio);

#ifdef __cplusplus
}
#endif

#endif /* EGT_B200_H */
