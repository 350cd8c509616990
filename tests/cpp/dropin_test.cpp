// Compiled C++ consumer of the drop-in boundary: includes
// the reference-shaped header egt_b200/packed.hpp, links -legt_b200, and runs
// quantize_matrix -> pack -> footprint (host) and, with --gpu, the device
// spmv and unpack, against golden vectors the reference itself produced
// (tests/golden/ref_vectors.npz, flattened by tests/test_cpp_dropin.py).
// Prints one PASS/FAIL line per check (acceptance_main.cpp style) and
// returns the failure count.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "egt_b200/packed.hpp"

namespace {

struct Reader {
  FILE* f;
  template <class T>
  std::vector<T> vec() {
    uint64_t n = 0;
    if (fread(&n, 8, 1, f) != 1) throw std::runtime_error("golden file truncated");
    std::vector<T> v(n);
    if (n && fread(v.data(), sizeof(T), n, f) != n) throw std::runtime_error("golden file truncated");
    return v;
  }
};

int failures = 0;
void expect(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: dropin_test golden.bin [--gpu]\n");
    return 2;
  }
  const bool gpu = argc > 2 && std::string(argv[2]) == "--gpu";
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  Reader rd{f};
  const auto ncases = rd.vec<uint32_t>();
  for (uint32_t c = 0; c < ncases[0]; ++c) {
    const auto meta = rd.vec<uint32_t>();  // rows, cols, n
    const uint32_t rows = meta[0], cols = meta[1];
    const int n = static_cast<int>(meta[2]);
    const auto w = rd.vec<float>();
    const auto x = rd.vec<float>();
    const auto mask_bits = rd.vec<uint8_t>();
    const auto gs = rd.vec<uint32_t>();
    const auto want_scales = rd.vec<float>();
    const auto want_zps = rd.vec<uint8_t>();
    const auto want_words = rd.vec<uint16_t>();
    const auto want_vbytes = rd.vec<uint8_t>();
    const auto want_fp = rd.vec<uint64_t>();  // index, value, scale, packed, baseline bytes
    const auto want_y = rd.vec<float>();
    const auto want_unpack = rd.vec<float>();
    const std::string tag = "case " + std::to_string(c) + " (" + std::to_string(rows) + "x" + std::to_string(cols) +
                            ", " + std::to_string(n) + ":4)";

    egt_b200::Matrix W(rows, cols);
    W.data.assign(w.begin(), w.end());
    egt_b200::PruneMask mask;
    mask.rows = rows;
    mask.cols = cols;
    mask.bits = mask_bits;
    egt_b200::GroupQuantSpec spec;
    spec.group_sizes = gs;
    const egt_b200::QuantizedMatrix q = egt_b200::quantize_matrix(W, spec, mask);
    expect(q.scales.size() == want_scales.size() &&
               std::memcmp(q.scales.data(), want_scales.data(), 4 * q.scales.size()) == 0 && q.zero_points == want_zps,
           tag + ": quantize_matrix scales / zero points bit-identical");
    const egt_b200::PackedSparseMatrix p = egt_b200::pack(mask, q, n, 4);
    expect(p.index_words == want_words, tag + ": pack index words identical");
    expect(p.value_bytes == want_vbytes, tag + ": pack INT4 codes identical");
    const egt_b200::FootprintReport fp = egt_b200::footprint(p);
    expect(fp.index_bytes == want_fp[0] && fp.value_bytes == want_fp[1] && fp.scale_bytes == want_fp[2] &&
               fp.packed_bytes == want_fp[3] && fp.baseline_bytes == want_fp[4],
           tag + ": footprint identical");
    bool threw = false;
    try {
      egt_b200::spmv(p, egt_b200::Vector(cols + 1, 0.f));
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()).find("input length differs from columns") != std::string::npos;
    } catch (...) {
    }
    expect(threw, tag + ": spmv length mismatch throws invalid_argument (packed.cpp:213-214)");
    if (!gpu) continue;
    const egt_b200::DeviceMatrix d(p);
    const egt_b200::Vector y = egt_b200::spmv(d, egt_b200::Vector(x.begin(), x.end()));
    double worst = 0.0;
    for (uint32_t r = 0; r < rows; ++r)
      worst = std::fmax(worst, std::fabs(static_cast<double>(y[r]) - want_y[r]) / (1.0 + std::fabs(want_y[r])));
    expect(worst <= 1e-3, tag + ": device spmv within 1e-3 (1 + |y|), max " + std::to_string(worst));
    const egt_b200::UnpackResult u = egt_b200::unpack(d);
    expect(std::memcmp(u.values.data.data(), want_unpack.data(), 4 * want_unpack.size()) == 0,
           tag + ": device unpack bit-exact");
    expect(u.mask.bits == mask_bits, tag + ": device unpack keep mask");
  }
  std::fclose(f);
  std::printf("%d failure(s)\n", failures);
  return failures;
}
