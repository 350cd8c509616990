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
 * synchronous.  Device memory is allocated on the current device. */
EGT_API egt_status egt_dev_packed_create(const egt_packed_view* view, void* stream, egt_dev_packed** out);

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
EGT_API egt_status egt_spmv_ex(const egt_dev_packed* h, const float* x_dev, float* y_dev, uint32_t M,
                               uint32_t ldx, uint32_t ldy, uint32_t flags, void* stream);

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
EGT_API void egt_tune_force_plan(int rb, int s, int nw, int nst, int ch);

/* Number of kernels the library has launched on this thread (a counter the
 * benchmark reads to report gpu_launches). */
EGT_API uint64_t egt_launch_count(void);

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
