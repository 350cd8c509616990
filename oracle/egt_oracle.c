/*
 * egt_oracle.c -- CPU restatement of the reference SparseGemv path.
 *
 * TEST INFRASTRUCTURE ONLY (see egt_oracle.h).  Compiled with
 * -O2 -ffp-contract=off so every f32 operation rounds exactly where the
 * reference's does (the reference build has no FMA: plain x86-64 target).
 * Reference citations are relative to the reference tree's proj/ directory.
 */
#include "egt_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* egto_last_error(void) { return g_err; }

static const double kScaleFloor = 1e-8; /* compress.hpp:33 */

/* ---------------------------------------------------------------- quant */

/* fit_group, compress.cpp:77-90.  Fit in double; store f32 / u8. */
void egto_fit_group(const double* values, size_t count, float* scale, uint8_t* zero_point) {
  if (count == 0) { /* :79 scale floor, zero point 0 */
    *scale = (float)kScaleFloor;
    *zero_point = 0;
    return;
  }
  double mn = values[0], mx = values[0];
  for (size_t i = 0; i < count; ++i) { /* :81-84 */
    if (values[i] < mn) mn = values[i];
    if (values[i] > mx) mx = values[i];
  }
  double s = (mx - mn) / 15.0; /* :85 */
  if (s < kScaleFloor) s = kScaleFloor;
  double zp = round(-mn / s); /* :86 round half away from zero */
  if (zp < 0.0) zp = 0.0;
  if (zp > 15.0) zp = 15.0;
  *scale = (float)s;
  *zero_point = (uint8_t)zp;
}

/* encode_value, compress.cpp:92-96: uses the float-rounded scale. */
uint8_t egto_encode_value(double value, float scale, uint8_t zero_point) {
  double code = round(value / (double)scale) + (double)zero_point;
  if (code < 0.0) code = 0.0;
  if (code > 15.0) code = 15.0;
  return (uint8_t)code;
}

/* decode_value, compress.cpp:98-101: (f32(code) - f32(zp)) * scale in f32. */
float egto_decode_value(uint8_t code, float scale, uint8_t zero_point) {
  float a = (float)code - (float)zero_point;
  return a * scale;
}

int egto_mask_at(const uint8_t* bits, uint32_t cols, uint32_t r, uint32_t c) {
  size_t i = (size_t)r * cols + c; /* compress.cpp:48-51 */
  return (bits[i / 8] >> (i % 8)) & 1;
}

static void mask_set(uint8_t* bits, uint32_t cols, uint32_t r, uint32_t c) {
  size_t i = (size_t)r * cols + c; /* compress.cpp:53-59 */
  bits[i / 8] |= (uint8_t)(1u << (i % 8));
}

size_t egto_group_count(uint32_t rows, uint32_t cols, const uint32_t* gs) {
  size_t total = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    if (gs[r] == 0) return 0;
    total += (cols + gs[r] - 1) / gs[r];
  }
  return total;
}

/* quantize_impl, compress.cpp:157-197. */
int egto_quantize(const float* w, uint32_t rows, uint32_t cols, const uint32_t* gs,
                  const uint8_t* mask_bits, uint32_t* goff, float* scales, uint8_t* zps,
                  uint8_t* codes, size_t* n_codes) {
  goff[0] = 0; /* :170-176 */
  for (uint32_t r = 0; r < rows; ++r) {
    if (gs[r] == 0) return fail(EGTO_EINVAL, "quantize: zero group size");
    goff[r + 1] = goff[r] + (cols + gs[r] - 1) / gs[r];
  }
  double* group = (double*)malloc(sizeof(double) * (cols ? cols : 1));
  size_t nc = 0;
  for (uint32_t r = 0; r < rows; ++r) { /* :182-195 */
    const uint32_t g = gs[r];
    uint32_t gi = 0;
    for (uint32_t start = 0; start < cols; start += g, ++gi) {
      uint32_t end = start + g < cols ? start + g : cols;
      size_t cnt = 0;
      for (uint32_t c = start; c < end; ++c)
        if (!mask_bits || egto_mask_at(mask_bits, cols, r, c))
          group[cnt++] = (double)w[(size_t)r * cols + c];
      float s;
      uint8_t zp;
      egto_fit_group(group, cnt, &s, &zp);
      scales[goff[r] + gi] = s;
      zps[goff[r] + gi] = zp;
      for (uint32_t c = start; c < end; ++c)
        if (!mask_bits || egto_mask_at(mask_bits, cols, r, c))
          codes[nc++] = egto_encode_value((double)w[(size_t)r * cols + c], s, zp);
    }
  }
  free(group);
  *n_codes = nc;
  return EGTO_OK;
}

/* dequantize, compress.cpp:210-228. */
int egto_dequantize(uint32_t rows, uint32_t cols, const uint32_t* gs, const uint32_t* goff,
                    const float* scales, const uint8_t* zps, const uint8_t* mask_bits,
                    const uint8_t* codes, size_t n_codes, float* out) {
  memset(out, 0, sizeof(float) * (size_t)rows * cols);
  size_t ci = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    const uint32_t g = gs[r];
    for (uint32_t c = 0; c < cols; ++c) {
      if (mask_bits && !egto_mask_at(mask_bits, cols, r, c)) continue;
      uint32_t gi = c / g;
      if (ci >= n_codes)
        return fail(EGTO_EINVARIANT, "dequantize: fewer codes than retained positions");
      out[(size_t)r * cols + c] =
          egto_decode_value(codes[ci++], scales[goff[r] + gi], zps[goff[r] + gi]);
    }
  }
  if (ci != n_codes)
    return fail(EGTO_EINVARIANT, "dequantize: more codes than retained positions");
  return EGTO_OK;
}

/* ---------------------------------------------------------------- pack */

/* check_pattern, packed.cpp:27-32 */
static int check_pattern(int n, int m) {
  if (m != 4) return fail(EGTO_EINVAL, "pack: group width must be 4");
  if (n == m) return fail(EGTO_EINVAL, "pack: dense pattern unsupported");
  if (n < 1 || n > m) return fail(EGTO_EINVAL, "pack: keep count must be in [1, group width)");
  return EGTO_OK;
}

/* check_mask_shape, packed.cpp:34-49 */
static int check_mask_shape(const uint8_t* bits, uint32_t rows, uint32_t cols, int n, int m) {
  if (cols % (uint32_t)m != 0)
    return fail(EGTO_EINVAL, "pack: columns must be a multiple of the group width");
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t start = 0; start < cols; start += (uint32_t)m) {
      int kept = 0;
      for (uint32_t c = start; c < start + (uint32_t)m; ++c) kept += egto_mask_at(bits, cols, r, c);
      if (kept != n)
        return fail(EGTO_EINVAL, "pack: group at row %u, column %u keeps %d entries (want %d)", r,
                    start, kept, n);
    }
  return EGTO_OK;
}

/* IndexStreamWriter + pack_common, packed.cpp:51-88: each kept column's
 * in-group offset c % m, 8 per u16 word, slot i at bits [15-2i, 14-2i],
 * final word zero-padded. */
int egto_pack_index(const uint8_t* bits, uint32_t rows, uint32_t cols, int n, int m,
                    uint16_t* words, size_t* n_words) {
  int rc = check_pattern(n, m);
  if (rc) return rc;
  rc = check_mask_shape(bits, rows, cols, n, m);
  if (rc) return rc;
  uint16_t word = 0;
  int slot = 0;
  size_t nw = 0;
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t c = 0; c < cols; ++c)
      if (egto_mask_at(bits, cols, r, c)) {
        word |= (uint16_t)((c % (uint32_t)m) << (14 - 2 * slot)); /* :53-56 */
        if (++slot == 8) {
          words[nw++] = word;
          word = 0;
          slot = 0;
        }
      }
  if (slot > 0) words[nw++] = word; /* :57-60 */
  *n_words = nw;
  return EGTO_OK;
}

/* pack(mask, QuantizedMatrix) code stream, packed.cpp:107-126: codes two per
 * byte, low nibble first, in stream order. */
int egto_pack_codes(const uint8_t* bits, uint32_t rows, uint32_t cols, int n,
                    const uint8_t* codes, size_t n_codes, int dense_codes, uint8_t* vb,
                    size_t* n_vb) {
  size_t emitted = 0, ci = 0, nb = 0;
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t c = 0; c < cols; ++c) {
      uint8_t code;
      if (dense_codes) {
        size_t at = (size_t)r * cols + c;
        if (at >= n_codes) return fail(EGTO_EINVAL, "pack: dense code index out of range");
        code = codes[at];
        if (!egto_mask_at(bits, cols, r, c)) continue;
      } else {
        if (!egto_mask_at(bits, cols, r, c)) continue;
        if (ci >= n_codes) return fail(EGTO_EINVAL, "pack: kept code index out of range");
        code = codes[ci++];
      }
      if (emitted % 2 == 0)
        vb[nb++] = code;
      else
        vb[nb - 1] |= (uint8_t)(code << 4);
      ++emitted;
    }
  size_t nnz = (size_t)rows * cols * (size_t)n / 4;
  if (emitted != nnz) return fail(EGTO_EINVARIANT, "pack: nonzero count mismatch");
  *n_vb = nb;
  return EGTO_OK;
}

/* pack(mask, Matrix), packed.cpp:130-141 (value stream only). */
int egto_pack_values(const uint8_t* bits, uint32_t rows, uint32_t cols, const float* w,
                     float* values, size_t* n_values) {
  size_t k = 0;
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t c = 0; c < cols; ++c)
      if (egto_mask_at(bits, cols, r, c)) values[k++] = w[(size_t)r * cols + c];
  *n_values = k;
  return EGTO_OK;
}

/* ---------------------------------------------------------------- walk */

static size_t p_nnz(const egto_packed* p) { return (size_t)p->rows * p->cols * p->n / p->m; }

/* offset_at, packed.hpp:64-66 */
static uint32_t offset_at(const egto_packed* p, size_t k) {
  return (p->index_words[k / 8] >> (14 - 2 * (k % 8))) & 0x3u;
}

/* check_packed, packed.cpp:145-166 */
static int check_sizes(const egto_packed* p) {
  if (p->m != 4) return fail(EGTO_EFORMAT, "packed matrix: group width must be 4");
  if (p->n < 1 || p->n >= p->m) return fail(EGTO_EFORMAT, "packed matrix: bad keep count");
  if (p->cols % p->m != 0)
    return fail(EGTO_EFORMAT, "packed matrix: columns not a multiple of the group width");
  size_t nnz = p_nnz(p);
  if (p->n_index_words != (nnz + 7) / 8)
    return fail(EGTO_EFORMAT, "packed matrix: index word count mismatch");
  if (p->kind == 1) {
    if (p->n_value_bytes != (nnz + 1) / 2)
      return fail(EGTO_EFORMAT, "packed matrix: value byte count mismatch");
    if (p->n_group_sizes != p->rows || p->n_group_offsets != (size_t)p->rows + 1)
      return fail(EGTO_EFORMAT, "packed matrix: group table size mismatch");
    if (p->n_scales != p->group_offsets[p->rows] || p->n_zero_points != p->n_scales)
      return fail(EGTO_EFORMAT, "packed matrix: scale table size mismatch");
  } else {
    if (p->n_values != nnz) return fail(EGTO_EFORMAT, "packed matrix: value count mismatch");
  }
  return EGTO_OK;
}

/* packed_value, packed.cpp:186-193.  The reference indexes its tables
 * unchecked; the restatement reports out-of-range tables as FormatError
 * instead of reading past them. */
static int packed_value(const egto_packed* p, uint32_t r, uint32_t col, size_t k, float* v) {
  if (p->kind == 0) {
    *v = p->values[k];
    return EGTO_OK;
  }
  uint8_t code = (uint8_t)((p->value_bytes[k / 2] >> ((k % 2) * 4)) & 0xf);
  uint32_t g = p->group_sizes[r];
  if (g == 0) return fail(EGTO_EFORMAT, "packed matrix: zero group size");
  size_t gi = (size_t)p->group_offsets[r] + col / g;
  if (gi >= p->n_scales) return fail(EGTO_EFORMAT, "packed matrix: group index out of range");
  *v = egto_decode_value(code, p->scales[gi], p->zero_points[gi]);
  return EGTO_OK;
}

int egto_check_packed(const egto_packed* p) {
  int rc = check_sizes(p);
  if (rc) return rc;
  const size_t row_nnz = (size_t)p->cols * p->n / p->m;
  size_t k = 0;
  for (uint32_t r = 0; r < p->rows; ++r) { /* for_each_nonzero, packed.cpp:169-184 */
    uint32_t prev = 0;
    for (size_t j = 0; j < row_nnz; ++j, ++k) {
      uint32_t off = offset_at(p, k);
      if (j % p->n != 0 && off <= prev)
        return fail(EGTO_EFORMAT, "packed matrix: in-group offsets not increasing");
      prev = off;
    }
  }
  return EGTO_OK;
}

/* unpack, packed.cpp:197-209 */
int egto_unpack(const egto_packed* p, float* values, uint8_t* mask_bits) {
  int rc = check_sizes(p);
  if (rc) return rc;
  memset(values, 0, sizeof(float) * (size_t)p->rows * p->cols);
  memset(mask_bits, 0, ((size_t)p->rows * p->cols + 7) / 8);
  const size_t row_nnz = (size_t)p->cols * p->n / p->m;
  size_t k = 0;
  for (uint32_t r = 0; r < p->rows; ++r) {
    uint32_t prev = 0;
    for (size_t j = 0; j < row_nnz; ++j, ++k) {
      uint32_t off = offset_at(p, k);
      if (j % p->n != 0 && off <= prev)
        return fail(EGTO_EFORMAT, "packed matrix: in-group offsets not increasing");
      prev = off;
      uint32_t col = (uint32_t)(j / p->n) * p->m + off; /* :180 */
      float v;
      rc = packed_value(p, r, col, k, &v);
      if (rc) return rc;
      mask_set(mask_bits, p->cols, r, col);
      values[(size_t)r * p->cols + col] = v;
    }
  }
  return EGTO_OK;
}

/* spmv, packed.cpp:211-220: y(r) += packed_value * x(col), f32, left to right. */
int egto_spmv(const egto_packed* p, const float* x, size_t x_len, float* y) {
  int rc = check_sizes(p);
  if (rc) return rc;
  if (x_len != p->cols) return fail(EGTO_EINVAL, "spmv: input length differs from columns");
  const size_t row_nnz = (size_t)p->cols * p->n / p->m;
  size_t k = 0;
  for (uint32_t r = 0; r < p->rows; ++r) {
    uint32_t prev = 0;
    float acc = 0.0f;
    for (size_t j = 0; j < row_nnz; ++j, ++k) {
      uint32_t off = offset_at(p, k);
      if (j % p->n != 0 && off <= prev)
        return fail(EGTO_EFORMAT, "packed matrix: in-group offsets not increasing");
      prev = off;
      uint32_t col = (uint32_t)(j / p->n) * p->m + off;
      float v;
      rc = packed_value(p, r, col, k, &v);
      if (rc) return rc;
      float prod = v * x[col];
      acc = acc + prod; /* :217 */
    }
    y[r] = acc;
  }
  return EGTO_OK;
}

/* footprint, packed.cpp:222-240 */
int egto_footprint(const egto_packed* p, uint64_t out[5], double* ratio) {
  if (p->n == p->m) return fail(EGTO_EINVAL, "footprint: dense pattern unsupported");
  int rc = check_sizes(p);
  if (rc) return rc;
  uint64_t index_b = (uint64_t)p->n_index_words * 2, value_b = 0, scale_b = 0;
  if (p->kind == 1) {
    value_b = p->n_value_bytes;
    scale_b = (uint64_t)p->n_scales * 4 + p->n_zero_points;
  } else {
    value_b = (uint64_t)p->n_values * 4;
  }
  uint64_t packed = index_b + value_b + scale_b;
  uint64_t base = (uint64_t)p_nnz(p) * 4 + ((uint64_t)p->rows + 1) * 4;
  out[0] = index_b;
  out[1] = value_b;
  out[2] = scale_b;
  out[3] = packed;
  out[4] = base;
  *ratio = (double)packed / (double)base;
  return EGTO_OK;
}

/* quant_dense_gemv, packed.cpp:266-281 */
void egto_quant_dense_gemv(uint32_t rows, uint32_t cols, const uint32_t* gs, const uint32_t* goff,
                           const float* scales, const uint8_t* zps, const uint8_t* codes,
                           const float* x, float* y) {
  size_t k = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    const uint32_t g = gs[r];
    float acc = 0.0f;
    for (uint32_t c = 0; c < cols; ++c) {
      uint32_t gi = c / g;
      float v = egto_decode_value(codes[k++], scales[goff[r] + gi], zps[goff[r] + gi]);
      float prod = v * x[c];
      acc = acc + prod;
    }
    y[r] = acc;
  }
}

/* magnitude_mask, packed.cpp:245-264: sort by |w| desc, ties to lower col. */
void egto_magnitude_mask(const float* w, uint32_t rows, uint32_t cols, int n, int m,
                         uint8_t* bits) {
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t start = 0; start < cols; start += (uint32_t)m) {
      float a[8];
      uint32_t idx[8];
      int cnt = 0;
      for (uint32_t c = start; c < start + (uint32_t)m; ++c, ++cnt) {
        a[cnt] = fabsf(w[(size_t)r * cols + c]);
        idx[cnt] = c;
      }
      /* insertion sort with the reference's comparator (stable outcome). */
      for (int i = 1; i < cnt; ++i)
        for (int j = i; j > 0; --j) {
          int before = (a[j] != a[j - 1]) ? (a[j] > a[j - 1]) : (idx[j] < idx[j - 1]);
          if (!before) break;
          float ta = a[j]; a[j] = a[j - 1]; a[j - 1] = ta;
          uint32_t ti = idx[j]; idx[j] = idx[j - 1]; idx[j - 1] = ti;
        }
      for (int i = 0; i < n; ++i) mask_set(bits, cols, r, idx[i]);
    }
}

/* importance_scores, compress.cpp:230-244: |w| * x_norms[c] + |w| * grad_abs,
 * two f32 products and one f32 sum (no contraction: -ffp-contract=off). */
int egto_importance(const float* w, const float* x_norms, const float* grad_abs, uint32_t rows,
                    uint32_t cols, float* scores) {
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t c = 0; c < cols; ++c) {
      const size_t i = (size_t)r * cols + c;
      const float a = fabsf(w[i]);
      const float p = a * x_norms[c];
      const float q = a * grad_abs[i];
      scores[i] = p + q;
    }
  return 0;
}

/* prune_nm, compress.cpp:246-278: per row, per group of m columns (the last
 * may be short), keep the min(n, #positive) largest scores; ties to the lower
 * column.  bits: PruneMask bitmap, zeroed here. */
int egto_prune_nm(const float* scores, uint32_t rows, uint32_t cols, int n, int m, uint8_t* bits) {
  if (m != 4) return fail(1, "prune_nm: group width must be 4");
  if (n < 1 || n >= m) return fail(1, "prune_nm: keep count must be in [1, group width)");
  memset(bits, 0, ((size_t)rows * cols + 7) / 8);
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t start = 0; start < cols; start += (uint32_t)m) {
      const uint32_t end = start + (uint32_t)m < cols ? start + (uint32_t)m : cols;
      float a[4];
      uint32_t idx[4];
      int cnt = 0;
      for (uint32_t c = start; c < end; ++c) {
        const float v = scores[(size_t)r * cols + c];
        if (v > 0.0f) {
          a[cnt] = v;
          idx[cnt++] = c;
        }
      }
      for (int i = 1; i < cnt; ++i)
        for (int j = i; j > 0; --j) {
          int before = (a[j] != a[j - 1]) ? (a[j] > a[j - 1]) : (idx[j] < idx[j - 1]);
          if (!before) break;
          float ta = a[j]; a[j] = a[j - 1]; a[j - 1] = ta;
          uint32_t ti = idx[j]; idx[j] = idx[j - 1]; idx[j - 1] = ti;
        }
      for (int i = 0; i < n && i < cnt; ++i) mask_set(bits, cols, r, idx[i]);
    }
  return 0;
}

/* ---------------------------------------------------------------- model */

/* sinusoidal_positions, model.cpp:44-54 (double math, stored f32). */
void egto_sinusoidal_positions(uint32_t max_positions, uint32_t d_model, float* out) {
  for (uint32_t pos = 0; pos < max_positions; ++pos)
    for (uint32_t i = 0; i < d_model; ++i) {
      double expo = (double)(2 * (i / 2)) / (double)d_model;
      double angle = (double)pos / pow(10000.0, expo);
      out[(size_t)pos * d_model + i] = (float)(i % 2 == 0 ? sin(angle) : cos(angle));
    }
}

static const float kNormEps = 1e-6f; /* model.cpp:27 */

/* rmsnorm, model.cpp:57-67 */
static void rmsnorm(const float* x, int n, int d, float* y) {
  for (int r = 0; r < n; ++r) {
    const float* xr = x + (size_t)r * d;
    float ss = 0.0f;
    for (int c = 0; c < d; ++c) ss += xr[c] * xr[c];
    float inv = 1.0f / sqrtf(ss / (float)d + kNormEps);
    for (int c = 0; c < d; ++c) y[(size_t)r * d + c] = xr[c] * inv;
  }
}

/* out[n x o] = a[n x i] * W^T, W [o x i] (the X * W^T products, model.cpp:156-195). */
static void linear(const float* a, int n, int in, const float* w, int o, float* out) {
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < o; ++j) {
      const float* ar = a + (size_t)r * in;
      const float* wj = w + (size_t)j * in;
      float s = 0.0f;
      for (int c = 0; c < in; ++c) s += ar[c] * wj[c];
      out[(size_t)r * o + j] = s;
    }
}

static float sigmoidf_(float x) { return 1.0f / (1.0f + expf(-x)); } /* model.cpp:80 */

int egto_forward(const egto_model_config* cfg, const float* embedding,
                 const float* const* lw, const float* head, const float* positions,
                 const int* tokens, const int* pos, const uint8_t* mask, int n, float* logits) {
  if (n == 0) return fail(EGTO_EINVAL, "forward: empty token sequence"); /* :123 */
  for (int i = 0; i < n; ++i) {
    if (tokens[i] < 0 || (uint32_t)tokens[i] >= cfg->vocab_size)
      return fail(EGTO_EINVAL, "forward: token out of range");
    if (pos[i] < 0 || (uint32_t)pos[i] >= cfg->max_positions)
      return fail(EGTO_EINVAL, "forward: position out of range");
  }
  const int d = (int)cfg->d_model, dff = (int)cfg->d_ff, H = (int)cfg->n_heads;
  const int dh = d / H;
  const float att_scale = 1.0f / sqrtf((float)dh); /* :139 */
  size_t nd = (size_t)n * d;
  float* x = malloc(sizeof(float) * nd);
  float* a = malloc(sizeof(float) * nd);
  float* q = malloc(sizeof(float) * nd);
  float* k = malloc(sizeof(float) * nd);
  float* v = malloc(sizeof(float) * nd);
  float* o = malloc(sizeof(float) * nd);
  float* t = malloc(sizeof(float) * nd);
  float* f1 = malloc(sizeof(float) * (size_t)n * dff);
  float* s = malloc(sizeof(float) * (size_t)n);
  for (int i = 0; i < n; ++i) /* :141-143 */
    for (int c = 0; c < d; ++c)
      x[(size_t)i * d + c] = embedding[(size_t)tokens[i] * d + c] + positions[(size_t)pos[i] * d + c];

  for (uint32_t l = 0; l < cfg->n_layers; ++l) {
    const float* const* w = lw + 6 * l;
    rmsnorm(x, n, d, a);      /* :155 */
    linear(a, n, d, w[0], d, q); /* :156-158 */
    linear(a, n, d, w[1], d, k);
    linear(a, n, d, w[2], d, v);
    memset(o, 0, sizeof(float) * nd);
    for (int h = 0; h < H; ++h) { /* :162-184 */
      for (int qi = 0; qi < n; ++qi) {
        float m = -INFINITY;
        for (int kj = 0; kj < n; ++kj) {
          float dot = 0.0f;
          for (int c = 0; c < dh; ++c) dot += q[(size_t)qi * d + h * dh + c] * k[(size_t)kj * d + h * dh + c];
          s[kj] = dot * att_scale;
          if (mask[(size_t)qi * n + kj] && s[kj] > m) m = s[kj];
        }
        if (!isfinite(m)) continue; /* :173 no visible key: zero row */
        float z = 0.0f;
        for (int kj = 0; kj < n; ++kj) {
          if (!mask[(size_t)qi * n + kj]) { s[kj] = 0.0f; continue; }
          float e = expf(s[kj] - m);
          s[kj] = e;
          z += e;
        }
        for (int kj = 0; kj < n; ++kj) s[kj] = s[kj] / z; /* :181 */
        for (int c = 0; c < dh; ++c) { /* :183 o = a * vh */
          float acc = 0.0f;
          for (int kj = 0; kj < n; ++kj) acc += s[kj] * v[(size_t)kj * d + h * dh + c];
          o[(size_t)qi * d + h * dh + c] = acc;
        }
      }
    }
    linear(o, n, d, w[3], d, t); /* :186 x_mid = x + o * wo^T */
    for (size_t i = 0; i < nd; ++i) x[i] = x[i] + t[i];
    rmsnorm(x, n, d, a);         /* :187 */
    linear(a, n, d, w[4], dff, f1); /* :188 */
    for (size_t i = 0; i < (size_t)n * dff; ++i) f1[i] = f1[i] * sigmoidf_(f1[i]); /* :189 */
    linear(f1, n, dff, w[5], d, t); /* :190 */
    for (size_t i = 0; i < nd; ++i) x[i] = x[i] + t[i];
  }
  rmsnorm(x, n, d, a); /* :194 */
  linear(a, n, d, head, (int)cfg->vocab_size, logits); /* :195 */
  free(x); free(a); free(q); free(k); free(v); free(o); free(t); free(f1); free(s);
  return EGTO_OK;
}

/* log_softmax, model.cpp:370-377: max in f32, sum of exp in double. */
void egto_log_softmax(const float* logits, size_t len, float* out) {
  float m = -INFINITY;
  for (size_t i = 0; i < len; ++i)
    if (logits[i] > m) m = logits[i];
  double z = 0.0;
  for (size_t i = 0; i < len; ++i) z += exp((double)(logits[i] - m));
  float lz = (float)log(z);
  for (size_t i = 0; i < len; ++i) out[i] = logits[i] - m - lz;
}
