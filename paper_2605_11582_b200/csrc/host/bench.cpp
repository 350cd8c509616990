// bench_spmv / bench_csv (packed.cpp:242-393, packed.hpp:100-113) on the
// B200: the reference's micro-benchmark harness with the same seeded inputs,
// variants and analytic bytes, timing the device products.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "egt_b200/packed.hpp"

#define EGT_EXPORT extern "C" EGT_API

namespace egt_impl {
void set_last_error(const std::string& msg);
}

namespace egt_b200 {
namespace {

// magnitude_mask (packed.cpp:244-262): exactly n kept per group of m, the
// largest |w| first, ties to the lower column.
PruneMask magnitude_mask(const Matrix& w, int n, int m) {
  PruneMask mask;
  mask.rows = w.rows;
  mask.cols = w.cols;
  mask.bits.assign((static_cast<size_t>(mask.rows) * mask.cols + 7) / 8, 0);
  std::vector<std::pair<float, uint32_t>> e;
  for (uint32_t r = 0; r < w.rows; ++r)
    for (uint32_t start = 0; start < w.cols; start += static_cast<uint32_t>(m)) {
      e.clear();
      for (uint32_t c = start; c < start + static_cast<uint32_t>(m); ++c) e.emplace_back(std::fabs(w(r, c)), c);
      std::sort(e.begin(), e.end(), [](const auto& a, const auto& b) {
        if (a.first != b.first) return a.first > b.first;
        return a.second < b.second;
      });
      for (int i = 0; i < n; ++i) mask.set(r, e[i].second, true);
    }
  return mask;
}

struct Stats {
  uint64_t median_ns = 0, p95_ns = 0;
};

// time_reps (packed.cpp:288-304) with device time: one warm-up, then each
// product bracketed by CUDA events on the stream.
template <class Fn>
Stats time_reps(int reps, cudaStream_t s, Fn&& fn) {
  fn();
  std::vector<cudaEvent_t> ev(2 * static_cast<size_t>(reps));
  for (auto& e : ev) cudaEventCreate(&e);
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(ev[2 * i], s);
    fn();
    cudaEventRecord(ev[2 * i + 1], s);
  }
  cudaStreamSynchronize(s);
  std::vector<uint64_t> ns(reps);
  for (int i = 0; i < reps; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
    ns[i] = static_cast<uint64_t>(std::llround(ms * 1e6));
  }
  for (auto& e : ev) cudaEventDestroy(e);
  std::sort(ns.begin(), ns.end());
  Stats st;
  st.median_ns = ns[ns.size() / 2];
  st.p95_ns = ns[std::min(ns.size() - 1, ns.size() * 95 / 100)];
  return st;
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

std::vector<BenchRow> bench_spmv(const std::vector<BenchShape>& shapes, int reps, uint64_t seed) {
  if (reps < 1) throw std::invalid_argument("bench: repetitions must be positive");
  std::vector<BenchRow> out;
  cudaStream_t s = nullptr;
  cuda_ok(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "bench: stream");
  struct Guard {
    cudaStream_t s;
    ~Guard() { cudaStreamDestroy(s); }
  } guard{s};
  for (size_t si = 0; si < shapes.size(); ++si) {
    const BenchShape& shape = shapes[si];
    if (shape.rows == 0 || shape.cols == 0) throw std::invalid_argument("bench: shape dimensions must be positive");
    if (shape.cols % 4 != 0) throw std::invalid_argument("bench: columns must be a multiple of 4");
    // the reference's inputs, element for element (packed.cpp:323-329)
    std::mt19937_64 rng(seed + 0x9e3779b97f4a7c15ull * (si + 1));
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    Matrix w(shape.rows, shape.cols);
    for (uint32_t r = 0; r < w.rows; ++r)
      for (uint32_t c = 0; c < w.cols; ++c) w(r, c) = dist(rng);
    Vector x(shape.cols);
    for (float& v : x) v = dist(rng);
    GroupQuantSpec spec;
    spec.group_sizes.assign(shape.rows, std::min<uint32_t>(64, shape.cols));

    float *dx = nullptr, *dy = nullptr, *dw = nullptr;
    cuda_ok(cudaMalloc(&dx, x.size() * sizeof(float)), "bench: x");
    cuda_ok(cudaMalloc(&dy, static_cast<size_t>(shape.rows) * sizeof(float)), "bench: y");
    cuda_ok(cudaMemcpy(dx, x.data(), x.size() * sizeof(float), cudaMemcpyHostToDevice), "bench: x upload");
    struct Free {
      float** p[3];
      ~Free() {
        for (float** q : p)
          if (*q) cudaFree(*q);
      }
    } fr{{&dx, &dy, &dw}};

    {  // dense-fp: the f32 matrix resident, one GEMV per product
      cuda_ok(cudaMalloc(&dw, w.data.size() * sizeof(float)), "bench: w");
      cuda_ok(cudaMemcpy(dw, w.data.data(), w.data.size() * sizeof(float), cudaMemcpyHostToDevice), "bench: w upload");
      BenchRow row{"dense-fp", shape.rows, shape.cols, "dense", 0, 0,
                   static_cast<uint64_t>(shape.rows) * shape.cols * 4};
      const Stats t = time_reps(reps, s, [&] { check(egt_gemv_f32(dw, dx, dy, shape.rows, shape.cols, s)); });
      row.median_ns = t.median_ns;
      row.p95_ns = t.p95_ns;
      out.push_back(row);
      cudaFree(dw);
      dw = nullptr;
    }
    {  // quant-dense: INT4 codes of every weight (quant_dense_gemv)
      const QuantizedMatrix q = quantize_matrix(w, spec);
      BenchRow row{"quant-dense", shape.rows, shape.cols, "dense", 0, 0,
                   (static_cast<uint64_t>(shape.rows) * shape.cols + 1) / 2 + q.scales.size() * 4 +
                       q.zero_points.size()};
      const DeviceMatrix d(q, s);
      const Stats t = time_reps(reps, s, [&] {
        check(egt_spmv(d.handle(), dx, dy, 1, shape.cols, shape.rows, s));
      });
      row.median_ns = t.median_ns;
      row.p95_ns = t.p95_ns;
      out.push_back(row);
    }
    for (int n : {2, 1}) {  // packed-2:4, packed-1:4
      const PruneMask mask = magnitude_mask(w, n, 4);
      const QuantizedMatrix q = quantize_matrix(w, spec, mask);
      const PackedSparseMatrix packed = pack(mask, q, n, 4);
      const std::string pat = n == 2 ? "2:4" : "1:4";
      BenchRow row{"packed-" + pat, shape.rows, shape.cols, pat, 0, 0, footprint(packed).packed_bytes};
      const DeviceMatrix d(packed, s);
      const Stats t = time_reps(reps, s, [&] {
        check(egt_spmv(d.handle(), dx, dy, 1, shape.cols, shape.rows, s));
      });
      row.median_ns = t.median_ns;
      row.p95_ns = t.p95_ns;
      out.push_back(row);
    }
  }
  return out;
}

std::string bench_csv(const std::vector<BenchRow>& rows) {  // packed.cpp:385-393
  std::ostringstream os;
  os << "variant,rows,cols,pattern,median_ns,p95_ns,bytes\n";
  for (const BenchRow& r : rows)
    os << r.variant << ',' << r.rows << ',' << r.cols << ',' << r.pattern << ',' << r.median_ns << ',' << r.p95_ns
       << ',' << r.bytes << '\n';
  return os.str();
}

}  // namespace egt_b200

EGT_EXPORT egt_status egt_bench_spmv(const uint32_t* rows, const uint32_t* cols, uint32_t n_shapes, int reps,
                                     uint64_t seed, char* csv, size_t cap, size_t* len) {
  try {
    if (n_shapes && (!rows || !cols)) throw std::invalid_argument("bench: null shape list");
    std::vector<egt_b200::BenchShape> shapes(n_shapes);
    for (uint32_t i = 0; i < n_shapes; ++i) shapes[i] = {rows[i], cols[i]};
    const std::string text = egt_b200::bench_csv(egt_b200::bench_spmv(shapes, reps, seed));
    if (len) *len = text.size();
    if (csv && cap) {
      const size_t k = std::min(cap - 1, text.size());
      std::memcpy(csv, text.data(), k);
      csv[k] = '\0';
    }
    return EGT_OK;
  } catch (const std::invalid_argument& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EINVAL;
  } catch (const std::exception& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EINTERNAL;
  }
}
