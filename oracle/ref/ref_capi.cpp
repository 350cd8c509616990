// extern "C" wrappers over the UNMODIFIED reference sources (packed.cpp,
// compress.cpp, egtq_io.cpp, io.cpp under /root/reference/proj/src), built by
// oracle/build_ref.sh into oracle/_ref/libegt_ref.so.  This file is written
// for this repo; it only converts flat buffers to the reference's value types
// and back, and maps its exceptions to status codes.  Test infrastructure
// only: it checks the restatement in oracle/egt_oracle.c and is the
// "reference" CPU arm of bench.py.
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>

#include "egt/compress.hpp"
#include "egt/packed.hpp"
#include "../egt_oracle.h"

namespace {
thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const egt::FormatError& e) {
    g_err = e.what();
    return 2;
  } catch (const egt::InvariantError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

egt::PruneMask make_mask(const uint8_t* bits, uint32_t rows, uint32_t cols) {
  egt::PruneMask m;
  m.rows = rows;
  m.cols = cols;
  m.bits.assign(bits, bits + (static_cast<size_t>(rows) * cols + 7) / 8);
  return m;
}

egt::Matrix make_matrix(const float* w, uint32_t rows, uint32_t cols) {
  egt::Matrix m(rows, cols);
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t c = 0; c < cols; ++c) m(r, c) = w[static_cast<size_t>(r) * cols + c];
  return m;
}

egt::PackedSparseMatrix make_packed(const egto_packed* p) {
  egt::PackedSparseMatrix q;
  q.n = p->n;
  q.m = p->m;
  q.rows = p->rows;
  q.cols = p->cols;
  q.kind = p->kind ? egt::PackedValueKind::kInt4 : egt::PackedValueKind::kFloat32;
  if (p->index_words) q.index_words.assign(p->index_words, p->index_words + p->n_index_words);
  if (p->value_bytes) q.value_bytes.assign(p->value_bytes, p->value_bytes + p->n_value_bytes);
  if (p->group_sizes) q.group_sizes.assign(p->group_sizes, p->group_sizes + p->n_group_sizes);
  if (p->group_offsets)
    q.group_offsets.assign(p->group_offsets, p->group_offsets + p->n_group_offsets);
  if (p->scales) q.scales.assign(p->scales, p->scales + p->n_scales);
  if (p->zero_points) q.zero_points.assign(p->zero_points, p->zero_points + p->n_zero_points);
  if (p->values) q.values.assign(p->values, p->values + p->n_values);
  return q;
}

egt::QuantizedMatrix make_quant(uint32_t rows, uint32_t cols, const uint32_t* gs,
                                const uint32_t* goff, const float* scales, const uint8_t* zps,
                                size_t n_groups, const uint8_t* qmask, const uint8_t* codes,
                                size_t n_codes) {
  egt::QuantizedMatrix q;
  q.rows = rows;
  q.cols = cols;
  q.group_sizes.assign(gs, gs + rows);
  q.group_offsets.assign(goff, goff + rows + 1);
  q.scales.assign(scales, scales + n_groups);
  q.zero_points.assign(zps, zps + n_groups);
  if (qmask) q.mask.assign(qmask, qmask + (static_cast<size_t>(rows) * cols + 7) / 8);
  q.codes.assign(codes, codes + n_codes);
  return q;
}
}  // namespace

void ref_set_error(const std::string& m) { g_err = m; }  // ref_model_capi.cpp

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_fit_group(const double* v, size_t n, float* scale, uint8_t* zp) {
  egt::GroupParams p = egt::fit_group(std::vector<double>(v, v + n));
  *scale = p.scale;
  *zp = p.zero_point;
}

uint8_t ref_encode_value(double v, float scale, uint8_t zp) {
  return egt::encode_value(v, egt::GroupParams{scale, zp});
}

float ref_decode_value(uint8_t code, float scale, uint8_t zp) {
  return egt::decode_value(code, egt::GroupParams{scale, zp});
}

int ref_quantize(const float* w, uint32_t rows, uint32_t cols, const uint32_t* gs,
                 const uint8_t* mask_bits, uint32_t* goff, float* scales, uint8_t* zps,
                 uint8_t* codes, size_t* n_codes) {
  return guarded([&] {
    egt::Matrix m = make_matrix(w, rows, cols);
    egt::GroupQuantSpec spec;
    spec.group_sizes.assign(gs, gs + rows);
    egt::QuantizedMatrix q = mask_bits
                                 ? egt::quantize_matrix(m, spec, make_mask(mask_bits, rows, cols))
                                 : egt::quantize_matrix(m, spec);
    std::copy(q.group_offsets.begin(), q.group_offsets.end(), goff);
    std::copy(q.scales.begin(), q.scales.end(), scales);
    std::copy(q.zero_points.begin(), q.zero_points.end(), zps);
    std::copy(q.codes.begin(), q.codes.end(), codes);
    *n_codes = q.codes.size();
  });
}

int ref_dequantize(uint32_t rows, uint32_t cols, const uint32_t* gs, const uint32_t* goff,
                   const float* scales, const uint8_t* zps, size_t n_groups,
                   const uint8_t* mask_bits, const uint8_t* codes, size_t n_codes, float* out) {
  return guarded([&] {
    egt::Matrix d = egt::dequantize(
        make_quant(rows, cols, gs, goff, scales, zps, n_groups, mask_bits, codes, n_codes));
    for (uint32_t r = 0; r < rows; ++r)
      for (uint32_t c = 0; c < cols; ++c) out[static_cast<size_t>(r) * cols + c] = d(r, c);
  });
}

// pack(mask, QuantizedMatrix, n, m) (packed.cpp:92-128).
int ref_pack_int4(const uint8_t* mask_bits, uint32_t rows, uint32_t cols, int n, int m,
                  uint32_t q_rows, uint32_t q_cols, const uint32_t* gs, const uint32_t* goff,
                  const float* scales, const uint8_t* zps, size_t n_groups,
                  const uint8_t* qmask, const uint8_t* codes, size_t n_codes, uint16_t* words,
                  size_t* n_words, uint8_t* vbytes, size_t* n_vbytes) {
  return guarded([&] {
    egt::QuantizedMatrix q =
        make_quant(q_rows, q_cols, gs, goff, scales, zps, n_groups, qmask, codes, n_codes);
    egt::PackedSparseMatrix p = egt::pack(make_mask(mask_bits, rows, cols), q, n, m);
    std::copy(p.index_words.begin(), p.index_words.end(), words);
    *n_words = p.index_words.size();
    std::copy(p.value_bytes.begin(), p.value_bytes.end(), vbytes);
    *n_vbytes = p.value_bytes.size();
  });
}

// pack(mask, Matrix, n, m) (packed.cpp:130-141).
int ref_pack_f32(const uint8_t* mask_bits, uint32_t rows, uint32_t cols, int n, int m,
                 const float* w, uint32_t w_rows, uint32_t w_cols, uint16_t* words,
                 size_t* n_words, float* values, size_t* n_values) {
  return guarded([&] {
    egt::PackedSparseMatrix p =
        egt::pack(make_mask(mask_bits, rows, cols), make_matrix(w, w_rows, w_cols), n, m);
    std::copy(p.index_words.begin(), p.index_words.end(), words);
    *n_words = p.index_words.size();
    std::copy(p.values.begin(), p.values.end(), values);
    *n_values = p.values.size();
  });
}

int ref_unpack(const egto_packed* p, float* values, uint8_t* mask_bits) {
  return guarded([&] {
    egt::UnpackResult u = egt::unpack(make_packed(p));
    for (uint32_t r = 0; r < p->rows; ++r)
      for (uint32_t c = 0; c < p->cols; ++c)
        values[static_cast<size_t>(r) * p->cols + c] = u.values(r, c);
    std::copy(u.mask.bits.begin(), u.mask.bits.end(), mask_bits);
  });
}

int ref_spmv(const egto_packed* p, const float* x, size_t x_len, float* y) {
  return guarded([&] {
    egt::Vector xv(static_cast<Eigen::Index>(x_len));
    for (size_t i = 0; i < x_len; ++i) xv(static_cast<Eigen::Index>(i)) = x[i];
    egt::Vector yv = egt::spmv(make_packed(p), xv);
    for (Eigen::Index i = 0; i < yv.size(); ++i) y[i] = yv(i);
  });
}

int ref_footprint(const egto_packed* p, uint64_t out[5], double* ratio) {
  return guarded([&] {
    egt::FootprintReport f = egt::footprint(make_packed(p));
    out[0] = f.index_bytes;
    out[1] = f.value_bytes;
    out[2] = f.scale_bytes;
    out[3] = f.packed_bytes;
    out[4] = f.baseline_bytes;
    *ratio = f.ratio;
  });
}

// bench_spmv (packed.cpp:310-383) for one shape: 4 rows of (median, p95, bytes).
int ref_bench_spmv(uint32_t rows, uint32_t cols, int reps, uint64_t seed, uint64_t* median_ns,
                   uint64_t* p95_ns, uint64_t* bytes) {
  return guarded([&] {
    std::vector<egt::BenchRow> out = egt::bench_spmv({{rows, cols}}, reps, seed);
    for (size_t i = 0; i < out.size(); ++i) {
      median_ns[i] = out[i].median_ns;
      p95_ns[i] = out[i].p95_ns;
      bytes[i] = out[i].bytes;
    }
  });
}

// A reference PackedSparseMatrix kept alive across timing calls.
void* ref_packed_new(const egto_packed* p) {
  try {
    return new egt::PackedSparseMatrix(make_packed(p));
  } catch (...) {
    return nullptr;
  }
}

void ref_packed_free(void* h) { delete static_cast<egt::PackedSparseMatrix*>(h); }

// Times the reference spmv on `threads` host threads, each repeatedly calling
// spmv on the shared immutable matrix (SPEC: concurrent spmv calls over shared
// packed data are safe).  Every thread does `calls` products after one warm-up;
// returns wall seconds for the whole batch and the last y of thread 0.
int ref_spmv_timed(void* h, const float* x, size_t x_len, int calls, int threads,
                   double* seconds, float* y_out) {
  return guarded([&] {
    const auto& p = *static_cast<egt::PackedSparseMatrix*>(h);
    egt::Vector xv(static_cast<Eigen::Index>(x_len));
    for (size_t i = 0; i < x_len; ++i) xv(static_cast<Eigen::Index>(i)) = x[i];
    egt::Vector warm = egt::spmv(p, xv);
    std::vector<std::thread> pool;
    std::vector<float> sink(static_cast<size_t>(threads), 0.0f);
    auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        for (int i = 0; i < calls; ++i) {
          egt::Vector yv = egt::spmv(p, xv);
          sink[static_cast<size_t>(t)] += yv(0);
          if (t == 0 && i == calls - 1 && y_out)
            for (Eigen::Index r = 0; r < yv.size(); ++r) y_out[r] = yv(r);
        }
      });
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    (void)warm;
  });
}

// EGTQ files written by the reference's own serialize_compressed
// (egtq_io.cpp:212-219): layer i has name names[i], pattern patterns[i]
// (0 dense, 1 one-of-four, 2 two-of-four), storage quant[i]; weights w[i]
// (rows x cols), keep bitmap masks[i] (NULL for dense) and uniform group size
// groups[i] (quantize_matrix with the mask, compress.cpp:157-197).
int ref_egtq_serialize(int n_layers, const char* const* names, const uint8_t* patterns, const uint8_t* quant,
                       const uint32_t* rows, const uint32_t* cols, const float* const* w,
                       const uint8_t* const* masks, const uint32_t* groups, uint8_t* out, size_t cap,
                       size_t* len) {
  return guarded([&] {
    egt::CompressedModel model;
    for (int i = 0; i < n_layers; ++i) {
      egt::CompressedLayer L;
      L.name = names[i];
      L.pattern = static_cast<egt::SparsityPattern>(patterns[i]);
      L.has_quant = quant[i] != 0;
      L.mask = masks[i] ? make_mask(masks[i], rows[i], cols[i]) : egt::PruneMask::all_kept(rows[i], cols[i]);
      egt::Matrix m = make_matrix(w[i], rows[i], cols[i]);
      if (L.has_quant) {
        egt::GroupQuantSpec spec;
        spec.group_sizes.assign(rows[i], groups[i]);
        L.quant = masks[i] ? egt::quantize_matrix(m, spec, L.mask) : egt::quantize_matrix(m, spec);
      } else {
        L.dense_values = m;
        for (uint32_t r = 0; r < rows[i]; ++r)
          for (uint32_t c = 0; c < cols[i]; ++c)
            if (!L.mask.at(r, c)) L.dense_values(r, c) = 0.0f;
      }
      model.layers.push_back(std::move(L));
    }
    const std::string bytes = egt::serialize_compressed(model);
    *len = bytes.size();
    if (bytes.size() > cap) throw std::invalid_argument("ref_egtq_serialize: buffer too small");
    std::memcpy(out, bytes.data(), bytes.size());
  });
}

// parse_compressed (egtq_io.cpp:221-235) on a byte buffer: layer count, or
// the FormatError.
int ref_egtq_parse(const uint8_t* bytes, size_t n, uint32_t* n_layers) {
  return guarded([&] {
    egt::CompressedModel m = egt::parse_compressed(std::string(reinterpret_cast<const char*>(bytes), n), "egtq");
    *n_layers = static_cast<uint32_t>(m.layers.size());
  });
}

// importance_scores (compress.cpp:230-244): |w| x_norm[c] + |w| grad_abs.
int ref_importance(const float* w, const float* x_norms, const float* grad_abs, uint32_t rows,
                   uint32_t cols, float* scores) {
  return guarded([&] {
    egt::Vector xn(cols);
    for (uint32_t c = 0; c < cols; ++c) xn(c) = x_norms[c];
    egt::ImportanceMatrix im = egt::importance_scores(make_matrix(w, rows, cols), xn,
                                                      make_matrix(grad_abs, rows, cols));
    for (uint32_t r = 0; r < rows; ++r)
      for (uint32_t c = 0; c < cols; ++c) scores[static_cast<size_t>(r) * cols + c] = im.scores(r, c);
  });
}

// prune_nm (compress.cpp:246-278): PruneMask bitmap of the top-n positive
// scores of every group of m columns.
int ref_prune_nm(const float* scores, uint32_t rows, uint32_t cols, int n, int m, uint8_t* mask_bits) {
  return guarded([&] {
    egt::ImportanceMatrix im;
    im.scores = make_matrix(scores, rows, cols);
    egt::PruneMask pm = egt::prune_nm(make_matrix(scores, rows, cols), im, n, m);
    std::copy(pm.bits.begin(), pm.bits.end(), mask_bits);
  });
}

}  // extern "C"
