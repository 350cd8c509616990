/*
 * egt_oracle.h -- CPU restatement of the reference SparseGemv path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product (paper_2605_11582_b200) never
 * links or calls anything under oracle/.
 *
 * Every function restates one reference function line by line in plain C
 * (no FMA contraction, f32/f64 exactly where the reference uses them) and
 * cites the reference file:line it follows (paths relative to the reference
 * tree's proj/ directory).
 *
 * Parity pinning: the restatement is pinned (a) against the reference's own
 * known-answer tests (0x7200, ramp fit, [-1,1] fit, hand spmv = 1.0,
 * footprint 29/136; see tests/test_oracle_golden.py) and (b) against
 * fixtures produced by the UNMODIFIED reference sources compiled into
 * oracle/_ref/libegt_ref.so (oracle/build_ref.sh, tests/golden/make_golden.py).
 *
 * Error codes mirror the reference's three exception classes:
 *   0 ok, 1 std::invalid_argument, 2 FormatError, 3 InvariantError.
 */
#ifndef EGT_ORACLE_H
#define EGT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { EGTO_OK = 0, EGTO_EINVAL = 1, EGTO_EFORMAT = 2, EGTO_EINVARIANT = 3 };

/* Message of the last failing call on this thread. */
const char* egto_last_error(void);

/* PackedSparseMatrix (packed.hpp:37-67) as a flat view. kind: 0 f32, 1 int4. */
typedef struct {
  uint8_t n, m;
  uint32_t rows, cols;
  uint8_t kind;
  const uint16_t* index_words; size_t n_index_words;
  const uint8_t* value_bytes;  size_t n_value_bytes;
  const uint32_t* group_sizes; size_t n_group_sizes;   /* rows */
  const uint32_t* group_offsets; size_t n_group_offsets; /* rows + 1 */
  const float* scales;         size_t n_scales;
  const uint8_t* zero_points;  size_t n_zero_points;
  const float* values;         size_t n_values;
} egto_packed;

/* compress.cpp:77-101 */
void egto_fit_group(const double* values, size_t count, float* scale, uint8_t* zero_point);
uint8_t egto_encode_value(double value, float scale, uint8_t zero_point);
float egto_decode_value(uint8_t code, float scale, uint8_t zero_point);

/* PruneMask bit helpers (compress.cpp:48-59): LSB-first bitmap over r*cols+c. */
int egto_mask_at(const uint8_t* bits, uint32_t cols, uint32_t r, uint32_t c);

/* Total groups = sum_r ceil(cols / g_r) (compress.cpp:170-176); 0 on a zero g. */
size_t egto_group_count(uint32_t rows, uint32_t cols, const uint32_t* group_sizes);

/* quantize_impl (compress.cpp:157-197). mask_bits may be NULL (all kept).
 * Outputs: group_offsets[rows+1], scales/zero_points[group_count],
 * codes[<= rows*cols] one per byte for retained positions, *n_codes. */
int egto_quantize(const float* w, uint32_t rows, uint32_t cols,
                  const uint32_t* group_sizes, const uint8_t* mask_bits,
                  uint32_t* group_offsets, float* scales, uint8_t* zero_points,
                  uint8_t* codes, size_t* n_codes);

/* dequantize (compress.cpp:210-228): dense [rows x cols], dropped -> 0. */
int egto_dequantize(uint32_t rows, uint32_t cols, const uint32_t* group_sizes,
                    const uint32_t* group_offsets, const float* scales,
                    const uint8_t* zero_points, const uint8_t* mask_bits,
                    const uint8_t* codes, size_t n_codes, float* out);

/* check_pattern + check_mask_shape + IndexStreamWriter (packed.cpp:27-88).
 * words must hold ceil(nnz/8) entries. */
int egto_pack_index(const uint8_t* mask_bits, uint32_t rows, uint32_t cols,
                    int n, int m, uint16_t* words, size_t* n_words);

/* pack(mask, QuantizedMatrix) value stream (packed.cpp:92-128).
 * dense_codes != 0: codes has rows*cols entries (quant.mask empty);
 * otherwise codes covers exactly the kept positions. */
int egto_pack_codes(const uint8_t* mask_bits, uint32_t rows, uint32_t cols,
                    int n, const uint8_t* codes, size_t n_codes, int dense_codes,
                    uint8_t* value_bytes, size_t* n_value_bytes);

/* pack(mask, Matrix) value stream (packed.cpp:130-141). */
int egto_pack_values(const uint8_t* mask_bits, uint32_t rows, uint32_t cols,
                     const float* w, float* values, size_t* n_values);

/* check_packed + offset monotonicity of for_each_nonzero (packed.cpp:145-184). */
int egto_check_packed(const egto_packed* p);

/* unpack (packed.cpp:197-209): values[rows*cols], mask_bits[ceil(rows*cols/8)]. */
int egto_unpack(const egto_packed* p, float* values, uint8_t* mask_bits);

/* spmv (packed.cpp:211-220): y[rows], f32 left to right per row. */
int egto_spmv(const egto_packed* p, const float* x, size_t x_len, float* y);

/* footprint (packed.cpp:222-240): out[0..4] = index, value, scale, packed,
 * baseline bytes; *ratio = packed / baseline. */
int egto_footprint(const egto_packed* p, uint64_t out[5], double* ratio);

/* quant_dense_gemv (packed.cpp:266-281), dense codes one per byte. */
void egto_quant_dense_gemv(uint32_t rows, uint32_t cols, const uint32_t* group_sizes,
                           const uint32_t* group_offsets, const float* scales,
                           const uint8_t* zero_points, const uint8_t* codes,
                           const float* x, float* y);

/* magnitude_mask (packed.cpp:245-264): exactly n kept per group of m by |w|,
 * ties to the lower column. bits must be zeroed, ceil(rows*cols/8) bytes. */
/* importance_scores (compress.cpp:230-244) and prune_nm (:246-278). */
int egto_importance(const float* w, const float* x_norms, const float* grad_abs, uint32_t rows,
                    uint32_t cols, float* scores);
int egto_prune_nm(const float* scores, uint32_t rows, uint32_t cols, int n, int m, uint8_t* bits);
void egto_magnitude_mask(const float* w, uint32_t rows, uint32_t cols, int n, int m,
                         uint8_t* bits);

/* ---- verify substrate: forward_impl (model.cpp:118-202) ---- */
typedef struct {
  uint32_t vocab_size, d_model, n_layers, n_heads, d_ff, max_positions;
} egto_model_config;

/* sinusoidal_positions (model.cpp:44-54): out[max_positions x d_model]. */
void egto_sinusoidal_positions(uint32_t max_positions, uint32_t d_model, float* out);

/* forward (model.cpp:358-361 -> forward_impl :118-202).
 * layer_weights: n_layers*6 pointers in the order wq, wk, wv, wo, ff1, ff2
 * (each [out x in] row-major, model.hpp:47-51). mask: n*n bytes (0/1).
 * logits: [n x vocab]. */
int egto_forward(const egto_model_config* cfg, const float* embedding,
                 const float* const* layer_weights, const float* head,
                 const float* positions, const int* tokens, const int* pos,
                 const uint8_t* mask, int n, float* logits);

/* log_softmax (model.cpp:370-377) of one row. */
void egto_log_softmax(const float* logits, size_t len, float* out);

#ifdef __cplusplus
}
#endif

#endif /* EGT_ORACLE_H */
