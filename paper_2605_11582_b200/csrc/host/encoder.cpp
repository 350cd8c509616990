// Host encoder + C++ drop-in API (egt_b200/packed.hpp).  The encoder restates
// the reference's byte layout exactly; tests/test_host_encoder.py checks it
// byte for byte against the reference sources (oracle/_ref) and the golden
// vectors.  Citations are relative to the reference's proj/ directory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>

#include "egt_b200/packed.hpp"

#define EGT_EXPORT extern "C" EGT_API

namespace egt_b200 {

// ------------------------------------------------------------ PruneMask
// compress.cpp:36-65
PruneMask PruneMask::all_kept(uint32_t rows, uint32_t cols) {
  PruneMask m;
  m.rows = rows;
  m.cols = cols;
  const size_t total = static_cast<size_t>(rows) * cols;
  m.bits.assign((total + 7) / 8, 0xff);
  for (size_t i = total; i < m.bits.size() * 8; ++i)
    m.bits[i / 8] &= static_cast<uint8_t>(~(1u << (i % 8)));
  return m;
}
bool PruneMask::at(uint32_t r, uint32_t c) const {
  const size_t i = static_cast<size_t>(r) * cols + c;
  return (bits[i / 8] >> (i % 8)) & 1;
}
void PruneMask::set(uint32_t r, uint32_t c, bool keep) {
  const size_t i = static_cast<size_t>(r) * cols + c;
  if (keep)
    bits[i / 8] |= static_cast<uint8_t>(1u << (i % 8));
  else
    bits[i / 8] &= static_cast<uint8_t>(~(1u << (i % 8)));
}
size_t PruneMask::kept_count() const {
  size_t n = 0;
  for (uint8_t b : bits) n += static_cast<size_t>(__builtin_popcount(b));
  return n;
}

// ------------------------------------------------------------ group fit
// compress.cpp:77-101: fit in double, store f32 / u8.
GroupParams fit_group(const std::vector<double>& values) {
  GroupParams p;
  if (values.empty()) return p;
  double mn = values[0], mx = values[0];
  for (double v : values) {
    mn = std::min(mn, v);
    mx = std::max(mx, v);
  }
  const double scale = std::max(kScaleFloor, (mx - mn) / 15.0);
  const double zp = std::clamp(std::round(-mn / scale), 0.0, 15.0);
  p.scale = static_cast<float>(scale);
  p.zero_point = static_cast<uint8_t>(zp);
  return p;
}
uint8_t encode_value(double value, const GroupParams& params) {
  const double code = std::round(value / static_cast<double>(params.scale)) +
                      static_cast<double>(params.zero_point);
  return static_cast<uint8_t>(std::clamp(code, 0.0, 15.0));
}
float decode_value(uint8_t code, const GroupParams& params) {
  return (static_cast<float>(code) - static_cast<float>(params.zero_point)) * params.scale;
}

// ------------------------------------------------------------ quantize
namespace {
QuantizedMatrix quantize_impl(const Matrix& w, const GroupQuantSpec& spec, const PruneMask* mask) {
  const uint32_t rows = w.rows, cols = w.cols;  // compress.cpp:157-197
  if (spec.group_sizes.size() != rows)
    throw std::invalid_argument("quantize: group spec length differs from rows");
  if (mask && (mask->rows != rows || mask->cols != cols))
    throw std::invalid_argument("quantize: mask shape differs from matrix");
  QuantizedMatrix q;
  q.rows = rows;
  q.cols = cols;
  q.group_sizes = spec.group_sizes;
  q.group_offsets.resize(rows + 1);
  q.group_offsets[0] = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    const uint32_t g = spec.group_sizes[r];
    if (g == 0) throw std::invalid_argument("quantize: zero group size");
    q.group_offsets[r + 1] = q.group_offsets[r] + (cols + g - 1) / g;
  }
  q.scales.resize(q.group_offsets[rows]);
  q.zero_points.resize(q.group_offsets[rows]);
  if (mask) q.mask = mask->bits;
  std::vector<double> group;
  for (uint32_t r = 0; r < rows; ++r) {
    const uint32_t g = spec.group_sizes[r];
    for (uint32_t start = 0, gi = 0; start < cols; start += g, ++gi) {
      const uint32_t end = std::min(start + g, cols);
      group.clear();
      for (uint32_t c = start; c < end; ++c)
        if (!mask || mask->at(r, c)) group.push_back(w(r, c));
      const GroupParams p = fit_group(group);
      q.scales[q.group_offsets[r] + gi] = p.scale;
      q.zero_points[q.group_offsets[r] + gi] = p.zero_point;
      for (uint32_t c = start; c < end; ++c)
        if (!mask || mask->at(r, c)) q.codes.push_back(encode_value(w(r, c), p));
    }
  }
  return q;
}
}  // namespace

QuantizedMatrix quantize_matrix(const Matrix& w, const GroupQuantSpec& spec) {
  return quantize_impl(w, spec, nullptr);
}
QuantizedMatrix quantize_matrix(const Matrix& w, const GroupQuantSpec& spec, const PruneMask& mask) {
  return quantize_impl(w, spec, &mask);
}

Matrix dequantize(const QuantizedMatrix& q) {  // compress.cpp:210-228
  Matrix out(q.rows, q.cols);
  size_t ci = 0;
  for (uint32_t r = 0; r < q.rows; ++r) {
    const uint32_t g = q.group_sizes[r];
    for (uint32_t c = 0; c < q.cols; ++c) {
      if (!q.mask.empty()) {
        const size_t i = static_cast<size_t>(r) * q.cols + c;
        if (!((q.mask[i / 8] >> (i % 8)) & 1)) continue;
      }
      const uint32_t gi = c / g;
      if (ci >= q.codes.size())
        throw InvariantError("dequantize: fewer codes than retained positions");
      out(r, c) = decode_value(q.codes[ci++], GroupParams{q.scales[q.group_offsets[r] + gi],
                                                          q.zero_points[q.group_offsets[r] + gi]});
    }
  }
  if (ci != q.codes.size()) throw InvariantError("dequantize: more codes than retained positions");
  return out;
}

// ------------------------------------------------------------ pack
namespace {
void check_pattern(int n, int m) {  // packed.cpp:27-32
  if (m != 4) throw std::invalid_argument("pack: group width must be 4");
  if (n == m) throw std::invalid_argument("pack: dense pattern unsupported");
  if (n < 1 || n > m) throw std::invalid_argument("pack: keep count must be in [1, group width)");
}

void check_mask_shape(const PruneMask& mask, int n, int m) {  // packed.cpp:34-49
  if (mask.cols % m != 0)
    throw std::invalid_argument("pack: columns must be a multiple of the group width");
  for (uint32_t r = 0; r < mask.rows; ++r)
    for (uint32_t start = 0; start < mask.cols; start += m) {
      int kept = 0;
      for (uint32_t c = start; c < start + static_cast<uint32_t>(m); ++c) kept += mask.at(r, c) ? 1 : 0;
      if (kept != n) {
        std::ostringstream os;
        os << "pack: group at row " << r << ", column " << start << " keeps " << kept
           << " entries (want " << n << ")";
        throw std::invalid_argument(os.str());
      }
    }
}

// The 2bit-CSR index stream (packed.cpp:51-88): in-group offset c % m of
// each kept column, eight per u16 word, slot i in bits [15-2i, 14-2i].
PackedSparseMatrix pack_index(const PruneMask& mask, int n, int m) {
  check_pattern(n, m);
  check_mask_shape(mask, n, m);
  PackedSparseMatrix p;
  p.n = static_cast<uint8_t>(n);
  p.m = static_cast<uint8_t>(m);
  p.rows = mask.rows;
  p.cols = mask.cols;
  p.index_words.reserve((p.nnz() + 7) / 8);
  uint16_t word = 0;
  int slot = 0;
  for (uint32_t r = 0; r < mask.rows; ++r)
    for (uint32_t c = 0; c < mask.cols; ++c)
      if (mask.at(r, c)) {
        word |= static_cast<uint16_t>((c % m) << (14 - 2 * slot));
        if (++slot == 8) {
          p.index_words.push_back(word);
          word = 0;
          slot = 0;
        }
      }
  if (slot > 0) p.index_words.push_back(word);
  return p;
}
}  // namespace

PackedSparseMatrix pack(const PruneMask& mask, const QuantizedMatrix& quant, int n, int m) {
  if (quant.rows != mask.rows || quant.cols != mask.cols)  // packed.cpp:92-128
    throw std::invalid_argument("pack: quantized shape differs from mask");
  const bool dense_codes = quant.mask.empty();
  if (!dense_codes && quant.mask != mask.bits)
    throw std::invalid_argument("pack: quantized mask differs from prune mask");
  PackedSparseMatrix p = pack_index(mask, n, m);
  p.kind = PackedValueKind::kInt4;
  p.group_sizes = quant.group_sizes;
  p.group_offsets = quant.group_offsets;
  p.scales = quant.scales;
  p.zero_points = quant.zero_points;
  p.value_bytes.reserve((p.nnz() + 1) / 2);
  size_t emitted = 0, ci = 0;
  for (uint32_t r = 0; r < mask.rows; ++r)
    for (uint32_t c = 0; c < mask.cols; ++c) {
      uint8_t code = 0;
      if (dense_codes) {
        code = quant.codes.at(static_cast<size_t>(r) * mask.cols + c);
        if (!mask.at(r, c)) continue;
      } else {
        if (!mask.at(r, c)) continue;
        code = quant.codes.at(ci++);
      }
      if (emitted % 2 == 0)
        p.value_bytes.push_back(code);
      else
        p.value_bytes.back() |= static_cast<uint8_t>(code << 4);
      ++emitted;
    }
  if (emitted != p.nnz()) throw InvariantError("pack: nonzero count mismatch");
  return p;
}

PackedSparseMatrix pack(const PruneMask& mask, const Matrix& values, int n, int m) {
  if (values.rows != mask.rows || values.cols != mask.cols)  // packed.cpp:130-141
    throw std::invalid_argument("pack: value shape differs from mask");
  PackedSparseMatrix p = pack_index(mask, n, m);
  p.kind = PackedValueKind::kFloat32;
  p.values.reserve(p.nnz());
  for (uint32_t r = 0; r < mask.rows; ++r)
    for (uint32_t c = 0; c < mask.cols; ++c)
      if (mask.at(r, c)) p.values.push_back(values(r, c));
  return p;
}

egt_packed_view view_of(const PackedSparseMatrix& p) {
  egt_packed_view v{};
  v.n = p.n;
  v.m = p.m;
  v.rows = p.rows;
  v.cols = p.cols;
  v.kind = static_cast<uint8_t>(p.kind);
  v.index_words = p.index_words.data();
  v.n_index_words = p.index_words.size();
  v.value_bytes = p.value_bytes.data();
  v.n_value_bytes = p.value_bytes.size();
  v.group_sizes = p.group_sizes.data();
  v.n_group_sizes = p.group_sizes.size();
  v.group_offsets = p.group_offsets.data();
  v.n_group_offsets = p.group_offsets.size();
  v.scales = p.scales.data();
  v.n_scales = p.scales.size();
  v.zero_points = p.zero_points.data();
  v.n_zero_points = p.zero_points.size();
  v.values = p.values.data();
  v.n_values = p.values.size();
  return v;
}

FootprintReport footprint(const PackedSparseMatrix& p) {  // packed.cpp:222-240
  if (p.n == p.m) throw std::invalid_argument("footprint: dense pattern unsupported");
  const egt_packed_view v = view_of(p);
  uint64_t out[5];
  double ratio = 0.0;
  check(egt_host_footprint(&v, out, &ratio));
  FootprintReport f;
  f.index_bytes = out[0];
  f.value_bytes = out[1];
  f.scale_bytes = out[2];
  f.packed_bytes = out[3];
  f.baseline_bytes = out[4];
  f.ratio = ratio;
  return f;
}

// ------------------------------------------------------------ device side
void throw_status(egt_status st) {
  const std::string msg = egt_last_error();
  switch (st) {
    case EGT_EINVAL: throw std::invalid_argument(msg);
    case EGT_EFORMAT: throw FormatError(msg);
    case EGT_ECUDA: throw CudaError(msg);
    default: throw InvariantError(msg);
  }
}

DeviceMatrix::DeviceMatrix(egt_dev_packed* h) : h_(h, [](egt_dev_packed* p) { egt_dev_packed_destroy(p); }) {}

DeviceMatrix::DeviceMatrix(const PackedSparseMatrix& p, void* stream) {
  const egt_packed_view v = view_of(p);
  egt_dev_packed* h = nullptr;
  check(egt_dev_packed_create(&v, stream, &h));
  h_.reset(h, [](egt_dev_packed* q) { egt_dev_packed_destroy(q); });
}

DeviceMatrix::DeviceMatrix(const QuantizedMatrix& q, void* stream) {
  if (!q.mask.empty()) throw std::invalid_argument("dense int4: quantized matrix has a prune mask");
  egt_quant_view v{};
  v.rows = q.rows;
  v.cols = q.cols;
  v.group_sizes = q.group_sizes.data();
  v.group_offsets = q.group_offsets.data();
  v.scales = q.scales.data();
  v.n_scales = q.scales.size();
  v.zero_points = q.zero_points.data();
  v.codes = q.codes.data();
  v.n_codes = q.codes.size();
  egt_dev_packed* h = nullptr;
  check(egt_dev_dense_i4_create(&v, stream, &h));
  h_.reset(h, [](egt_dev_packed* p) { egt_dev_packed_destroy(p); });
}

DeviceMatrix DeviceMatrix::slice_rows(uint32_t r0, uint32_t r1) const {
  egt_dev_packed* s = nullptr;
  check(egt_dev_packed_slice_rows(h_.get(), r0, r1, &s));
  return DeviceMatrix(s);
}

egt_dev_packed_info DeviceMatrix::info() const {
  egt_dev_packed_info i{};
  check(egt_dev_packed_query(h_.get(), &i));
  return i;
}

Vector spmv(const DeviceMatrix& w, const Vector& x, void* stream) {
  const egt_dev_packed_info i = w.info();
  Vector y(i.rows, 0.0f);
  check(egt_spmv_host(w.handle(), x.data(), x.size(), y.data(), stream));
  return y;
}

Vector spmv(const PackedSparseMatrix& packed, const Vector& x) {
  if (x.size() != packed.cols) throw std::invalid_argument("spmv: input length differs from columns");
  return spmv(DeviceMatrix(packed), x);
}

UnpackResult unpack(const DeviceMatrix& w, void* stream) {
  const egt_dev_packed_info i = w.info();
  const size_t n = static_cast<size_t>(i.rows) * i.cols;
  UnpackResult out;
  out.values = Matrix(i.rows, i.cols);
  out.mask.rows = i.rows;
  out.mask.cols = i.cols;
  out.mask.bits.assign((n + 7) / 8, 0);
  if (n == 0) return out;
  float* dw = nullptr;
  uint8_t* dm = nullptr;
  const size_t mask_words = (n + 31) / 32 * 4;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMalloc(&dw, n * sizeof(float) + mask_words) != cudaSuccess)
    throw CudaError("unpack: device allocation failed");
  dm = reinterpret_cast<uint8_t*>(dw + n);
  egt_status st = egt_dequant(w.handle(), dw, dm, stream);
  cudaError_t e = cudaSuccess;
  if (st == EGT_OK) {
    e = cudaMemcpyAsync(out.values.data.data(), dw, n * sizeof(float), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out.mask.bits.data(), dm, out.mask.bits.size(), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  cudaFree(dw);
  if (st != EGT_OK) throw_status(st);
  if (e != cudaSuccess) throw CudaError(std::string("unpack: ") + cudaGetErrorString(e));
  return out;
}

UnpackResult unpack(const PackedSparseMatrix& packed) { return unpack(DeviceMatrix(packed)); }

}  // namespace egt_b200

// ---------------------------------------------------------------- C-ABI
namespace egt_impl {
void set_last_error(const std::string& msg);  // capi.cu: shared egt_last_error()
}

namespace {

template <class Fn>
egt_status host_guard(Fn&& fn) {
  try {
    fn();
    return EGT_OK;
  } catch (const std::invalid_argument& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EINVAL;
  } catch (const egt_b200::FormatError& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EFORMAT;
  } catch (const std::exception& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EINTERNAL;
  }
}

egt_b200::PruneMask mask_of(const uint8_t* bits, uint32_t rows, uint32_t cols) {
  egt_b200::PruneMask m;
  m.rows = rows;
  m.cols = cols;
  m.bits.assign(bits, bits + (static_cast<size_t>(rows) * cols + 7) / 8);
  return m;
}
}  // namespace

EGT_EXPORT void egt_host_fit_group(const double* values, size_t count, float* scale, uint8_t* zp) {
  const egt_b200::GroupParams p = egt_b200::fit_group(std::vector<double>(values, values + count));
  *scale = p.scale;
  *zp = p.zero_point;
}

EGT_EXPORT size_t egt_host_group_count(uint32_t rows, uint32_t cols, const uint32_t* gs) {
  size_t total = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    if (gs[r] == 0) return 0;
    total += (cols + gs[r] - 1) / gs[r];
  }
  return total;
}

EGT_EXPORT egt_status egt_host_quantize(const float* w, uint32_t rows, uint32_t cols,
                                        const uint32_t* gs, const uint8_t* mask_bits,
                                        uint32_t* goff, float* scales, uint8_t* zps, uint8_t* codes,
                                        size_t* n_codes) {
  return host_guard([&] {
    egt_b200::Matrix m(rows, cols);
    std::memcpy(m.data.data(), w, m.data.size() * sizeof(float));
    egt_b200::GroupQuantSpec spec;
    spec.group_sizes.assign(gs, gs + rows);
    const egt_b200::QuantizedMatrix q = mask_bits
                                            ? egt_b200::quantize_matrix(m, spec, mask_of(mask_bits, rows, cols))
                                            : egt_b200::quantize_matrix(m, spec);
    std::copy(q.group_offsets.begin(), q.group_offsets.end(), goff);
    std::copy(q.scales.begin(), q.scales.end(), scales);
    std::copy(q.zero_points.begin(), q.zero_points.end(), zps);
    std::copy(q.codes.begin(), q.codes.end(), codes);
    *n_codes = q.codes.size();
  });
}

EGT_EXPORT egt_status egt_host_pack_int4(const uint8_t* mask_bits, uint32_t rows, uint32_t cols,
                                         int n, int m, const uint8_t* codes, size_t n_codes,
                                         int dense_codes, uint16_t* words, size_t* n_words,
                                         uint8_t* value_bytes, size_t* n_value_bytes) {
  return host_guard([&] {
    egt_b200::PruneMask mask = mask_of(mask_bits, rows, cols);
    egt_b200::QuantizedMatrix q;
    q.rows = rows;
    q.cols = cols;
    if (!dense_codes) q.mask = mask.bits;
    q.codes.assign(codes, codes + n_codes);
    const egt_b200::PackedSparseMatrix p = egt_b200::pack(mask, q, n, m);
    std::copy(p.index_words.begin(), p.index_words.end(), words);
    *n_words = p.index_words.size();
    std::copy(p.value_bytes.begin(), p.value_bytes.end(), value_bytes);
    *n_value_bytes = p.value_bytes.size();
  });
}

EGT_EXPORT egt_status egt_host_pack_f32(const uint8_t* mask_bits, uint32_t rows, uint32_t cols,
                                        int n, int m, const float* w, uint16_t* words,
                                        size_t* n_words, float* values, size_t* n_values) {
  return host_guard([&] {
    egt_b200::Matrix mat(rows, cols);
    std::memcpy(mat.data.data(), w, mat.data.size() * sizeof(float));
    const egt_b200::PackedSparseMatrix p = egt_b200::pack(mask_of(mask_bits, rows, cols), mat, n, m);
    std::copy(p.index_words.begin(), p.index_words.end(), words);
    *n_words = p.index_words.size();
    std::copy(p.values.begin(), p.values.end(), values);
    *n_values = p.values.size();
  });
}

EGT_EXPORT egt_status egt_host_footprint(const egt_packed_view* v, uint64_t out[5], double* ratio) {
  return host_guard([&] {  // packed.cpp:222-240 (check_packed sizes first)
    if (v->n == v->m) throw std::invalid_argument("footprint: dense pattern unsupported");
    if (v->m != 4) throw egt_b200::FormatError("packed matrix: group width must be 4");
    if (v->n < 1 || v->n >= v->m) throw egt_b200::FormatError("packed matrix: bad keep count");
    if (v->cols % v->m != 0)
      throw egt_b200::FormatError("packed matrix: columns not a multiple of the group width");
    const uint64_t nnz = static_cast<uint64_t>(v->rows) * v->cols * v->n / v->m;
    if (v->n_index_words != (nnz + 7) / 8)
      throw egt_b200::FormatError("packed matrix: index word count mismatch");
    uint64_t value_b = 0, scale_b = 0;
    if (v->kind == EGT_KIND_INT4) {
      if (v->n_value_bytes != (nnz + 1) / 2)
        throw egt_b200::FormatError("packed matrix: value byte count mismatch");
      if (v->n_group_sizes != v->rows || v->n_group_offsets != static_cast<size_t>(v->rows) + 1)
        throw egt_b200::FormatError("packed matrix: group table size mismatch");
      if (v->n_scales != v->group_offsets[v->rows] || v->n_zero_points != v->n_scales)
        throw egt_b200::FormatError("packed matrix: scale table size mismatch");
      value_b = v->n_value_bytes;
      scale_b = v->n_scales * 4 + v->n_zero_points;
    } else {
      if (v->n_values != nnz) throw egt_b200::FormatError("packed matrix: value count mismatch");
      value_b = v->n_values * 4;
    }
    out[0] = v->n_index_words * 2;
    out[1] = value_b;
    out[2] = scale_b;
    out[3] = out[0] + out[1] + out[2];
    out[4] = nnz * 4 + (static_cast<uint64_t>(v->rows) + 1) * 4;
    *ratio = static_cast<double>(out[3]) / static_cast<double>(out[4]);
  });
}
