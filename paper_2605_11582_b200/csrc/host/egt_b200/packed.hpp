// C++ drop-in for the reference's SparseGemv host API (namespace egt in
// proj/include/egt/packed.hpp and compress.hpp), re-implemented without Eigen.
// Same type names, argument meaning and exception classes; the products run
// on the B200 through the C-ABI in include/egt_b200.h.
//
//   reference (proj/include/egt/...)            here (namespace egt_b200)
//   PruneMask            compress.hpp:36-45      PruneMask
//   GroupQuantSpec       compress.hpp:49-51      GroupQuantSpec
//   QuantizedMatrix      compress.hpp:59-71      QuantizedMatrix
//   GroupParams, fit_group/encode/decode :76-83  same
//   quantize_matrix / dequantize :96-100         same
//   PackedSparseMatrix   packed.hpp:37-67        PackedSparseMatrix
//   pack (both)          packed.hpp:72-74        pack
//   unpack               packed.hpp:81           unpack (device dequant)
//   spmv                 packed.hpp:85           spmv (device), DeviceMatrix
//   footprint            packed.hpp:98           footprint
//   FormatError / InvariantError common.hpp:38-47 same
#pragma once
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "egt_b200.h"

// The C++ drop-in is exported from libegt_b200.so (the library builds with
// -fvisibility=hidden): consumers link -legt_b200 and include this header.
#pragma GCC visibility push(default)
namespace egt_b200 {

class FormatError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class InvariantError : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline constexpr double kScaleFloor = 1e-8;

// Row-major dense f32 matrix (the reference's egt::Matrix role).
struct Matrix {
  uint32_t rows = 0, cols = 0;
  std::vector<float> data;
  Matrix() = default;
  Matrix(uint32_t r, uint32_t c) : rows(r), cols(c), data(static_cast<size_t>(r) * c, 0.0f) {}
  float& operator()(uint32_t r, uint32_t c) { return data[static_cast<size_t>(r) * cols + c]; }
  float operator()(uint32_t r, uint32_t c) const { return data[static_cast<size_t>(r) * cols + c]; }
};
using Vector = std::vector<float>;

struct PruneMask {
  uint32_t rows = 0, cols = 0;
  std::vector<uint8_t> bits;  // bit (r*cols + c), LSB-first
  static PruneMask all_kept(uint32_t rows, uint32_t cols);
  bool at(uint32_t r, uint32_t c) const;
  void set(uint32_t r, uint32_t c, bool keep);
  size_t kept_count() const;
};

struct GroupQuantSpec {
  std::vector<uint32_t> group_sizes;
};

struct QuantizedMatrix {
  uint32_t rows = 0, cols = 0;
  std::vector<uint32_t> group_sizes;
  std::vector<uint32_t> group_offsets;
  std::vector<float> scales;
  std::vector<uint8_t> zero_points;
  std::vector<uint8_t> mask;   // empty = all retained
  std::vector<uint8_t> codes;  // one per retained position
};

struct GroupParams {
  float scale = static_cast<float>(kScaleFloor);
  uint8_t zero_point = 0;
};

GroupParams fit_group(const std::vector<double>& values);
uint8_t encode_value(double value, const GroupParams& params);
float decode_value(uint8_t code, const GroupParams& params);

QuantizedMatrix quantize_matrix(const Matrix& w, const GroupQuantSpec& spec);
QuantizedMatrix quantize_matrix(const Matrix& w, const GroupQuantSpec& spec, const PruneMask& mask);
Matrix dequantize(const QuantizedMatrix& q);

enum class PackedValueKind : uint8_t { kFloat32 = 0, kInt4 = 1 };

struct PackedSparseMatrix {
  uint8_t n = 2, m = 4;
  uint32_t rows = 0, cols = 0;
  PackedValueKind kind = PackedValueKind::kInt4;
  std::vector<uint16_t> index_words;
  std::vector<uint8_t> value_bytes;
  std::vector<uint32_t> group_sizes;
  std::vector<uint32_t> group_offsets;
  std::vector<float> scales;
  std::vector<uint8_t> zero_points;
  std::vector<float> values;
  size_t nnz() const { return static_cast<size_t>(rows) * cols * n / m; }
  size_t row_nnz() const { return static_cast<size_t>(cols) * n / m; }
  uint32_t offset_at(size_t k) const { return (index_words[k / 8] >> (14 - 2 * (k % 8))) & 0x3u; }
};

PackedSparseMatrix pack(const PruneMask& mask, const QuantizedMatrix& quant, int n, int m);
PackedSparseMatrix pack(const PruneMask& mask, const Matrix& values, int n, int m);

struct FootprintReport {
  size_t index_bytes = 0, value_bytes = 0, scale_bytes = 0, packed_bytes = 0, baseline_bytes = 0;
  double ratio = 0.0;
};
FootprintReport footprint(const PackedSparseMatrix& packed);

// bench_spmv / bench_csv (packed.hpp:100-113, packed.cpp:310-393): the
// reference harness with its seeded inputs and analytic bytes; the timing
// columns are device nanoseconds per product (CUDA events, inputs resident).
struct BenchShape {
  uint32_t rows = 0;
  uint32_t cols = 0;
};
struct BenchRow {
  std::string variant;  // dense-fp | quant-dense | packed-2:4 | packed-1:4
  uint32_t rows = 0;
  uint32_t cols = 0;
  std::string pattern;
  uint64_t median_ns = 0;
  uint64_t p95_ns = 0;
  uint64_t bytes = 0;
};
std::vector<BenchRow> bench_spmv(const std::vector<BenchShape>& shapes, int reps, uint64_t seed);
std::string bench_csv(const std::vector<BenchRow>& rows);

// Throws the exception class the reference would for an egt_status.
// Layer-adaptive sparsity (compress.hpp:115-119, plan_sparsity
// compress.cpp:298-326): the mixed-dispatch keys of a compressed stack.
enum class SparsityPattern : uint8_t { kDense = 0, kOneOfFour = 1, kTwoOfFour = 2 };
std::vector<SparsityPattern> plan_sparsity(const std::vector<const Matrix*>& scores,
                                           const std::vector<const Matrix*>& weights, double rho_s);

[[noreturn]] void throw_status(egt_status st);
inline void check(egt_status st) {
  if (st != EGT_OK) throw_status(st);
}

egt_packed_view view_of(const PackedSparseMatrix& p);

// A packed matrix resident on the current CUDA device (immutable; safe to
// share across threads and streams).  Row shards are zero-copy.
class DeviceMatrix {
 public:
  explicit DeviceMatrix(const PackedSparseMatrix& p, void* stream = nullptr);
  // dense INT4 layer (quant_dense_gemv semantics); quant.mask must be empty
  explicit DeviceMatrix(const QuantizedMatrix& dense_quant, void* stream = nullptr);
  DeviceMatrix slice_rows(uint32_t r0, uint32_t r1) const;
  egt_dev_packed_info info() const;
  const egt_dev_packed* handle() const { return h_.get(); }

 private:
  explicit DeviceMatrix(egt_dev_packed* h);
  std::shared_ptr<egt_dev_packed> h_;
};

struct UnpackResult {
  Matrix values;
  PruneMask mask;
};

// y = W x on the device (upload of x, product, download of y).
Vector spmv(const DeviceMatrix& w, const Vector& x, void* stream = nullptr);
// The reference signature: uploads the matrix, computes, releases it.
Vector spmv(const PackedSparseMatrix& packed, const Vector& x);
// Bit-exact device unpack (packed.cpp:197-209).
UnpackResult unpack(const DeviceMatrix& w, void* stream = nullptr);
UnpackResult unpack(const PackedSparseMatrix& packed);

}  // namespace egt_b200
#pragma GCC visibility pop
