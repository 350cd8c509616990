// EGTQ compressed-model files -> device-resident layers.
//
// The reference's reader (egtq_io.cpp:110-210 read_layer, :221-235
// parse_compressed, over io.cpp:64-124 ByteReader) is restated here with the
// same checks and the same FormatError messages ("<context>: <message>",
// "truncated while reading <what>").  The file already holds the device's
// source stream for a pruned INT4 layer: the kept codes nibble-packed in row
// order ARE PackedSparseMatrix::value_bytes, and the optional index section IS
// index_words (the reader verifies it against the keep bitmap, as the
// reference does).  Upload is therefore the mixed dispatch on the layer's
// (pattern, storage) keys without re-quantizing or
// re-packing:
//   (2:4 | 1:4, quant)  -> egt_dev_packed_create, INT4 2bit-CSR
//   (dense,     quant)  -> egt_dev_dense_i4_create (quant_dense_gemv arm)
//   (2:4 | 1:4, fp)     -> egt_dev_packed_create, F32 view (FP16 on device)
//   (dense,     fp)     -> EGT_EINVAL: not on the SparseGemv path
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "egt_b200.h"
#include "egt_b200/packed.hpp"

namespace egt_b200 {

namespace {

constexpr uint32_t kCompressedVersion = 1;  // egtq_io.cpp:29

// Little-endian reader with the reference's messages (io.cpp:64-124).
class ByteReader {
 public:
  ByteReader(const uint8_t* data, size_t n, std::string context) : d_(data), n_(n), ctx_(std::move(context)) {}
  [[noreturn]] void fail(const std::string& message) const { throw FormatError(ctx_ + ": " + message); }
  void require(size_t k, const char* what) const {
    if (n_ - pos_ < k) throw FormatError(ctx_ + ": truncated while reading " + what);
  }
  uint8_t u8(const char* what) {
    require(1, what);
    return d_[pos_++];
  }
  uint16_t u16(const char* what) {
    require(2, what);
    const uint16_t v = static_cast<uint16_t>(d_[pos_] | (d_[pos_ + 1] << 8));
    pos_ += 2;
    return v;
  }
  uint32_t u32(const char* what) {
    require(4, what);
    uint32_t v = 0;
    for (int i = 3; i >= 0; --i) v = (v << 8) | d_[pos_ + i];
    pos_ += 4;
    return v;
  }
  uint64_t u64(const char* what) {
    require(8, what);
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | d_[pos_ + i];
    pos_ += 8;
    return v;
  }
  float f32(const char* what) {
    const uint32_t bits = u32(what);
    float v;
    std::memcpy(&v, &bits, sizeof(v));
    return v;
  }
  const uint8_t* raw(size_t len, const char* what) {
    require(len, what);
    const uint8_t* p = d_ + pos_;
    pos_ += len;
    return p;
  }
  std::string str16(const char* what) {
    const uint16_t len = u16(what);
    const uint8_t* p = raw(len, what);
    return std::string(reinterpret_cast<const char*>(p), len);
  }
  bool at_end() const { return pos_ == n_; }

 private:
  const uint8_t* d_;
  size_t n_;
  size_t pos_ = 0;
  std::string ctx_;
};

int keep_count(uint8_t pattern) { return pattern == 2 ? 2 : pattern == 1 ? 1 : 4; }  // compress.cpp pattern_keep_count

size_t mask_bytes(uint32_t rows, uint32_t cols) { return (static_cast<size_t>(rows) * cols + 7) / 8; }

bool mask_packable(const PruneMask& mask, int n) {  // egtq_io.cpp:31-42
  if (mask.cols % 4 != 0) return false;
  for (uint32_t r = 0; r < mask.rows; ++r)
    for (uint32_t start = 0; start < mask.cols; start += 4) {
      int kept = 0;
      for (uint32_t c = start; c < start + 4; ++c) kept += mask.at(r, c) ? 1 : 0;
      if (kept != n) return false;
    }
  return true;
}

std::vector<uint16_t> index_stream(const PruneMask& mask, int n) {  // egtq_io.cpp:44-46
  return pack(mask, Matrix(mask.rows, mask.cols), n, 4).index_words;
}

}  // namespace

struct EgtqLayer {
  std::string name;
  uint8_t pattern = 0;  // SparsityPattern: 0 dense, 1 one-of-four, 2 two-of-four
  bool has_quant = true;
  uint32_t rows = 0, cols = 0;
  PruneMask mask;
  QuantizedMatrix quant;              // tables; codes stay nibble-packed in packed_codes
  std::vector<uint8_t> packed_codes;  // (n_kept + 1) / 2 bytes, low nibble first
  uint64_t n_codes = 0;
  std::vector<float> kept_values;     // fp storage, row-major over kept positions
  bool has_index = false;
  std::vector<uint16_t> index_words;
};

// read_layer, egtq_io.cpp:110-210.
EgtqLayer read_layer(ByteReader& r) {
  EgtqLayer L;
  L.name = r.str16("layer name");
  const uint8_t pattern = r.u8("pattern tag");
  if (pattern > 2) r.fail("bad pattern tag " + std::to_string(pattern));
  L.pattern = pattern;
  const uint8_t storage = r.u8("storage tag");
  if (storage > 1) r.fail("bad storage tag " + std::to_string(storage));
  L.has_quant = storage == 1;
  const uint32_t rows = r.u32("rows");
  const uint32_t cols = r.u32("cols");
  if (rows == 0 || cols == 0) r.fail("empty shape for layer " + L.name);
  L.rows = rows;
  L.cols = cols;
  if (L.has_quant) {
    QuantizedMatrix& q = L.quant;
    q.rows = rows;
    q.cols = cols;
    q.group_sizes.resize(rows);
    q.group_offsets.assign(rows + 1, 0);
    for (uint32_t i = 0; i < rows; ++i) {
      const uint32_t g = q.group_sizes[i] = r.u32("group size");
      if (g == 0) r.fail("zero group size for layer " + L.name);
      q.group_offsets[i + 1] = q.group_offsets[i] + (cols + g - 1) / g;
    }
    const uint32_t n_groups = r.u32("group count");
    if (n_groups != q.group_offsets[rows]) r.fail("group count differs from group sizes for layer " + L.name);
    q.scales.resize(n_groups);
    for (uint32_t i = 0; i < n_groups; ++i) q.scales[i] = r.f32("scale");
    q.zero_points.resize(n_groups);
    for (uint32_t i = 0; i < n_groups; ++i) {
      q.zero_points[i] = r.u8("zero point");
      if (q.zero_points[i] > 15) r.fail("zero point out of range");
    }
    L.n_codes = r.u64("code count");
    const uint8_t* pc = r.raw((L.n_codes + 1) / 2, "codes");
    L.packed_codes.assign(pc, pc + (L.n_codes + 1) / 2);
    if (L.n_codes % 2 == 1 && (L.packed_codes.back() >> 4) != 0) r.fail("nonzero padding nibble in codes");
  } else {
    const uint64_t n_kept = r.u64("value count");
    L.kept_values.resize(n_kept);
    for (uint64_t i = 0; i < n_kept; ++i) L.kept_values[i] = r.f32("kept value");
  }
  if (L.pattern == 0) {
    L.mask = PruneMask::all_kept(rows, cols);
  } else {
    L.mask.rows = rows;
    L.mask.cols = cols;
    const uint8_t* b = r.raw(mask_bytes(rows, cols), "keep bitmap");
    L.mask.bits.assign(b, b + mask_bytes(rows, cols));
    const size_t total = static_cast<size_t>(rows) * cols;
    for (size_t i = total; i < L.mask.bits.size() * 8; ++i)
      if ((L.mask.bits[i / 8] >> (i % 8)) & 1) r.fail("nonzero padding bit in keep bitmap");
  }
  const size_t kept = L.mask.kept_count();
  if (L.has_quant) {
    const size_t expect = L.pattern == 0 ? static_cast<size_t>(rows) * cols : kept;
    if (L.n_codes != expect) r.fail("code count differs from keep bitmap for layer " + L.name);
  } else if (L.kept_values.size() != kept) {
    r.fail("value count differs from keep bitmap for layer " + L.name);
  }
  if (L.pattern != 0 && L.has_quant) {
    const uint8_t has_index = r.u8("index section tag");
    if (has_index > 1) r.fail("bad index section tag");
    if (has_index == 1) {
      const uint8_t n = r.u8("index keep count");
      const uint8_t m = r.u8("index group width");
      if (m != 4 || n != keep_count(L.pattern)) r.fail("index pattern differs from layer pattern");
      const uint32_t n_words = r.u32("index word count");
      L.index_words.resize(n_words);
      for (uint32_t i = 0; i < n_words; ++i) L.index_words[i] = r.u16("index word");
      if (!mask_packable(L.mask, n))
        r.fail("index section present but keep bitmap is not exact-" + std::to_string(n));
      if (L.index_words != index_stream(L.mask, n)) r.fail("index stream differs from keep bitmap for layer " + L.name);
      L.has_index = true;
    }
  }
  return L;
}

// parse_compressed, egtq_io.cpp:221-235.
std::vector<EgtqLayer> parse_compressed(const uint8_t* data, size_t n, const std::string& context) {
  ByteReader r(data, n, context);
  const uint8_t* magic = r.raw(4, "magic");
  if (std::memcmp(magic, "EGTQ", 4) != 0) r.fail("bad magic (want EGTQ)");
  const uint32_t version = r.u32("version");
  if (version != kCompressedVersion) r.fail("unsupported version " + std::to_string(version));
  const uint32_t count = r.u32("layer count");
  std::vector<EgtqLayer> layers;
  layers.reserve(count);
  for (uint32_t i = 0; i < count; ++i) layers.push_back(read_layer(r));
  if (!r.at_end()) r.fail("trailing bytes after last layer");
  return layers;
}

}  // namespace egt_b200

// ---------------------------------------------------------------- C-ABI
struct egt_egtq {
  std::vector<egt_b200::EgtqLayer> layers;
};

namespace egt_impl {
void set_last_error(const std::string& msg);  // capi.cu
}

namespace {
template <class Fn>
egt_status egtq_guard(Fn&& fn) {
  try {
    return fn();
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
}  // namespace

extern "C" {

EGT_API egt_status egt_egtq_parse(const uint8_t* bytes, size_t n, const char* context, egt_egtq** out) {
  return egtq_guard([&] {
    if (!out || (!bytes && n)) throw std::invalid_argument("egtq: null argument");
    *out = nullptr;
    auto e = new egt_egtq();
    try {
      e->layers = egt_b200::parse_compressed(bytes, n, context ? context : "egtq");
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
    return EGT_OK;
  });
}

EGT_API uint32_t egt_egtq_layer_count(const egt_egtq* e) { return e ? static_cast<uint32_t>(e->layers.size()) : 0; }

EGT_API egt_status egt_egtq_query(const egt_egtq* e, uint32_t i, egt_egtq_layer_info* info) {
  return egtq_guard([&] {
    if (!e || !info || i >= e->layers.size()) throw std::invalid_argument("egtq: layer index out of range");
    const egt_b200::EgtqLayer& L = e->layers[i];
    info->name = L.name.c_str();
    info->pattern = L.pattern;
    info->has_quant = L.has_quant ? 1 : 0;
    info->has_index = L.has_index ? 1 : 0;
    info->rows = L.rows;
    info->cols = L.cols;
    return EGT_OK;
  });
}

EGT_API egt_status egt_egtq_upload(const egt_egtq* e, uint32_t i, void* stream, egt_dev_packed** out) {
  return egt_egtq_upload_ex(e, i, 0u, stream, out);
}

EGT_API egt_status egt_egtq_upload_ex(const egt_egtq* e, uint32_t i, uint32_t flags, void* stream,
                                      egt_dev_packed** out) {
  return egtq_guard([&]() -> egt_status {
    if (!e || !out || i >= e->layers.size()) throw std::invalid_argument("egtq: layer index out of range");
    *out = nullptr;
    const egt_b200::EgtqLayer& L = e->layers[i];
    if (L.has_quant && L.pattern == 0) {
      // dense INT4: one code per byte for the quant view
      std::vector<uint8_t> codes(L.n_codes);
      for (uint64_t k = 0; k < L.n_codes; ++k) codes[k] = (L.packed_codes[k / 2] >> ((k % 2) * 4)) & 0xF;
      egt_quant_view v{};
      v.rows = L.rows;
      v.cols = L.cols;
      v.group_sizes = L.quant.group_sizes.data();
      v.group_offsets = L.quant.group_offsets.data();
      v.scales = L.quant.scales.data();
      v.n_scales = L.quant.scales.size();
      v.zero_points = L.quant.zero_points.data();
      v.codes = codes.data();
      v.n_codes = codes.size();
      return egt_dev_dense_i4_create(&v, stream, out);
    }
    if (!L.has_quant && L.pattern == 0)
      throw std::invalid_argument("egtq: dense fp layer " + L.name + " is not on the SparseGemv path");
    const int n = egt_b200::keep_count(L.pattern);
    egt_b200::PackedSparseMatrix p;
    if (L.has_quant) {
      // the file's kept codes are value_bytes; its index section (or, when
      // absent, pack's own stream and its "keeps" check) is index_words
      p = L.has_index ? egt_b200::PackedSparseMatrix{} : egt_b200::pack(L.mask, egt_b200::Matrix(L.rows, L.cols), n, 4);
      p.n = static_cast<uint8_t>(n);
      p.m = 4;
      p.rows = L.rows;
      p.cols = L.cols;
      p.kind = egt_b200::PackedValueKind::kInt4;
      if (L.has_index) p.index_words = L.index_words;
      p.values.clear();
      p.value_bytes = L.packed_codes;
      p.group_sizes = L.quant.group_sizes;
      p.group_offsets = L.quant.group_offsets;
      p.scales = L.quant.scales;
      p.zero_points = L.quant.zero_points;
    } else {
      egt_b200::Matrix dense(L.rows, L.cols);
      size_t vi = 0;
      for (uint32_t r = 0; r < L.rows; ++r)
        for (uint32_t c = 0; c < L.cols; ++c)
          if (L.mask.at(r, c)) dense(r, c) = L.kept_values[vi++];
      p = egt_b200::pack(L.mask, dense, n, 4);
    }
    const egt_packed_view v = egt_b200::view_of(p);
    return egt_dev_packed_create_ex(&v, flags, stream, out);
  });
}

EGT_API egt_status egt_egtq_destroy(egt_egtq* e) {
  delete e;
  return EGT_OK;
}

}  // extern "C"
