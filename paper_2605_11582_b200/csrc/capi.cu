// C-ABI entry points (include/egt_b200.h): upload + validation, row slicing,
// launch planning, per-stream split-K workspaces, error mapping.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "egt_b200.h"
#include "handle.h"

using namespace egt_impl;

namespace {

thread_local std::string g_err;
thread_local bool g_pdl = true;

egt_status fail(egt_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(EGT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));        \
  } while (0)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Bump allocator over one cudaMalloc.
struct Carve {
  std::vector<std::pair<size_t*, size_t>> req;
  size_t total = 0;
  size_t add(size_t bytes) {
    size_t off = total;
    total = align_up(total + std::max<size_t>(bytes, 16), 256);
    return off;
  }
};

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// Per (device, stream) split-K workspace; grows, never shrinks.
struct Workspace {
  float* partial = nullptr;
  size_t partial_floats = 0;
  uint32_t* counters = nullptr;
  size_t n_counters = 0;
};
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, Workspace> g_ws;

egt_status get_workspace(cudaStream_t s, size_t floats, size_t counters, Workspace** out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  Workspace& w = g_ws[{dev, s}];
  if (w.partial_floats < floats) {
    if (w.partial) CUDA_TRY(cudaFree(w.partial));
    w.partial = nullptr;
    size_t n = std::max(floats, static_cast<size_t>(1) << 20);
    CUDA_TRY(cudaMalloc(&w.partial, n * sizeof(float)));
    w.partial_floats = n;
  }
  if (w.n_counters < counters) {
    if (w.counters) CUDA_TRY(cudaFree(w.counters));
    w.counters = nullptr;
    size_t n = std::max(counters, static_cast<size_t>(4096));
    CUDA_TRY(cudaMalloc(&w.counters, n * sizeof(uint32_t)));
    CUDA_TRY(cudaMemset(w.counters, 0, n * sizeof(uint32_t)));
    w.n_counters = n;
  }
  *out = &w;
  return EGT_OK;
}

// check_packed (packed.cpp:145-166) on the host view, same messages.
egt_status check_view(const egt_packed_view* v) {
  if (!v) return fail(EGT_EINVAL, "packed matrix: null view");
  if (v->m != 4) return fail(EGT_EFORMAT, "packed matrix: group width must be 4");
  if (v->n < 1 || v->n >= v->m) return fail(EGT_EFORMAT, "packed matrix: bad keep count");
  if (v->cols % v->m != 0)
    return fail(EGT_EFORMAT, "packed matrix: columns not a multiple of the group width");
  const uint64_t nnz = static_cast<uint64_t>(v->rows) * v->cols * v->n / v->m;
  if (v->n_index_words != (nnz + 7) / 8)
    return fail(EGT_EFORMAT, "packed matrix: index word count mismatch");
  if (v->kind == EGT_KIND_INT4) {
    if (v->n_value_bytes != (nnz + 1) / 2)
      return fail(EGT_EFORMAT, "packed matrix: value byte count mismatch");
    if (v->n_group_sizes != v->rows || v->n_group_offsets != static_cast<size_t>(v->rows) + 1)
      return fail(EGT_EFORMAT, "packed matrix: group table size mismatch");
    if (v->n_scales != v->group_offsets[v->rows] || v->n_zero_points != v->n_scales)
      return fail(EGT_EFORMAT, "packed matrix: scale table size mismatch");
  } else if (v->kind == EGT_KIND_F32) {
    if (v->n_values != nnz) return fail(EGT_EFORMAT, "packed matrix: value count mismatch");
  } else {
    return fail(EGT_EFORMAT, "packed matrix: unknown value kind");
  }
  if (nnz > 0 && !v->index_words) return fail(EGT_EINVAL, "packed matrix: null index stream");
  return EGT_OK;
}

// Whether every row's quant groups start on 32-column (k-tile) boundaries.
// Scale entries per k-tile (tiled_format.h ss_entries): every group a
// multiple of 32 columns -> SS in {4, 2, 1}; otherwise, when `half_ok` (INT4
// 2:4) and every group is a multiple of 16 -> SS = 0 (16-column entries, the
// reference's default g_fine = 16).
bool groups_k_aligned(uint32_t rows, uint32_t cols, const uint32_t* gs, int* ss_out, bool half_ok = false) {
  int ss = 4;
  bool half = false;
  for (uint32_t r = 0; r < rows; ++r) {
    const uint32_t g = gs[r];
    if (g >= cols) continue;  // one group per row
    if (g % 32 != 0) {
      if (!half_ok || g % 16 != 0) return false;
      half = true;
      continue;
    }
    const uint32_t kt = g / 32;
    while (kt % ss != 0) ss >>= 1;
  }
  *ss_out = half ? 0 : ss;
  return true;
}

egt_status finish_error_flag(uint32_t* d_err, cudaStream_t s) {
  uint32_t h_err = 0;
  CUDA_TRY(cudaMemcpyAsync(&h_err, d_err, sizeof h_err, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (h_err & 1u) return fail(EGT_EFORMAT, "packed matrix: in-group offsets not increasing");
  if (h_err & 2u) return fail(EGT_EFORMAT, "packed matrix: zero group size");
  if (h_err & 4u) return fail(EGT_EFORMAT, "packed matrix: group table does not cover the row");
  if (h_err & 8u)
    return fail(EGT_EINVAL,
                "packed matrix: values not representable in fp16 (pass EGT_UPLOAD_ROUND_FP16 to round them)");
  return EGT_OK;
}

struct Upload {
  // device pointers into one temporary allocation
  void* base = nullptr;
  uint16_t* words = nullptr;
  uint8_t* codes = nullptr;
  uint8_t* dense = nullptr;
  float* f32 = nullptr;
  __half* f16 = nullptr;
  uint32_t* gs = nullptr;
  uint32_t* goff = nullptr;
  float* scales = nullptr;
  uint8_t* zps = nullptr;
  uint32_t* err = nullptr;
  ~Upload() {
    if (base) cudaFree(base);
  }
};

// Shared tail of create(): decide the path, re-tile if possible, fill info.
egt_status build_handle(int format, uint8_t n, uint8_t kind, uint32_t rows, uint32_t cols,
                        uint64_t nnz, const uint32_t* host_gs, uint64_t n_scales, Upload& up,
                        size_t up_bytes, cudaStream_t s, egt_dev_packed** out) {
  using namespace egt_fmt;
  auto h = std::make_unique<egt_dev_packed>();
  h->rows = rows;
  h->cols = cols;
  h->n = n;
  h->m = 4;
  h->kind = kind;
  h->format = static_cast<uint8_t>(format);
  h->nnz = nnz;
  // weight-side bytes a product must read (footprint, packed.cpp:222-240;
  // FP16 values on the device)
  const uint64_t idx_b = format == I4_DENSE ? 0 : 2 * ((nnz + 7) / 8);
  const uint64_t val_b = kind == EGT_KIND_INT4 ? (nnz + 1) / 2 : 2 * nnz;
  h->algorithmic_bytes = idx_b + val_b + (kind == EGT_KIND_INT4 ? 5 * n_scales : 0);

  int ss = 4;
  static const bool no_g16 = getenv("EGT_NO_TILED_G16") != nullptr;  // tuning: g16 on the reference-order stream
  const bool half_ok = !no_g16 && kind == EGT_KIND_INT4 &&
                       (format == I4_SP24 || (format == I4_SP14 && getenv("EGT_SP14_NATIVE") == nullptr));
  const bool tiled = rows > 0 && cols > 0 && cols % 32 == 0 &&
                     (kind == EGT_KIND_F32 || groups_k_aligned(rows, cols, host_gs, &ss, half_ok));
  // INT4 1:4 on the tiled path is stored as 2:4 with a zero-valued partner per
  // kept entry: one mma.sp per k-tile either way, but without the per-k-tile
  // placement and metadata ALU work (issue-bound otherwise; DESIGN 5).  The
  // algorithmic bytes above stay the 1:4 stream's.
  static const bool sp14_native = getenv("EGT_SP14_NATIVE") != nullptr;
  const bool pad14 = tiled && format == I4_SP14 && !sp14_native;
  if (pad14) {
    format = I4_SP24;
    h->format = static_cast<uint8_t>(I4_SP24);
  }
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  auto store = std::make_shared<DevStorage>();
  store->device = dev;
  if (tiled) {
    TiledStream ts;
    ts.KQ = static_cast<int>((cols + 127) / 128);
    ts.RT = static_cast<int>((rows + 15) / 16);
    ts.SS = kind == EGT_KIND_INT4 ? ss : 4;
    ts.E = ss_entries(ts.SS);
    ts.pad14 = pad14 ? 1 : 0;
    const size_t blocks = static_cast<size_t>(ts.RT) * ts.KQ;
    Carve c;
    const size_t o_vals = c.add(blocks * 32 * val_lane_bytes(format));
    const size_t o_meta = c.add(blocks * 32 * meta_lane_bytes(format));
    const size_t o_sc = has_scales(format) ? c.add(blocks * ts.E * 16 * sizeof(float)) : 0;
    const size_t o_zp = has_scales(format) ? c.add(blocks * ts.E * 16) : 0;
    CUDA_TRY(cudaMalloc(&store->base, c.total));
    store->bytes = c.total;
    uint8_t* b = static_cast<uint8_t*>(store->base);
    CUDA_TRY(cudaMemsetAsync(b, 0, c.total, s));
    ts.vals = b + o_vals;
    ts.meta = b + o_meta;
    ts.scales = has_scales(format) ? reinterpret_cast<float*>(b + o_sc) : nullptr;
    ts.zps = has_scales(format) ? b + o_zp : nullptr;
    RawStream raw;
    raw.words = up.words;
    raw.codes = up.codes;
    raw.dense_codes = up.dense;
    raw.values = up.f16;
    raw.group_sizes = up.gs;
    raw.group_offsets = up.goff;
    raw.scales = up.scales;
    raw.zps = up.zps;
    raw.n_scales = n_scales;
    CUDA_TRY(launch_relayout(raw, format, rows, cols, ts, const_cast<uint8_t*>(ts.vals),
                             const_cast<uint8_t*>(ts.meta), const_cast<float*>(ts.scales),
                             const_cast<uint8_t*>(ts.zps), s));
    CUDA_TRY(cudaStreamSynchronize(s));
    h->path = EGT_PATH_TILED;
    h->tiled = ts;
    h->device_bytes = c.total;
  } else {
    // keep the reference-order upload as the device copy
    store->base = up.base;
    store->bytes = up_bytes;
    up.base = nullptr;  // ownership moves to the handle
    h->path = EGT_PATH_GENERAL;
    if (kind == EGT_KIND_INT4 && format == I4_SP24 && cols % 16 == 0) {
      bool ok = true;
      for (uint32_t r = 0; r < rows && ok; ++r) {
        const uint32_t g = host_gs[r];
        ok = g >= cols || (g >= 16 && (g & (g - 1)) == 0);
      }
      h->grouped_ok = ok ? 1 : 0;
    }
    h->raw.words = up.words;
    h->raw.codes = up.codes;
    h->raw.dense_codes = up.dense;
    h->raw.values = up.f16;
    h->raw.group_sizes = up.gs;
    h->raw.group_offsets = up.goff;
    h->raw.scales = up.scales;
    h->raw.zps = up.zps;
    h->raw.n_scales = n_scales;
    h->device_bytes = up_bytes;
  }
  h->store = std::move(store);
  *out = h.release();
  return EGT_OK;
}

}  // namespace

namespace egt_impl {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace egt_impl

egt_impl::DevStorage::~DevStorage() {
  if (base) {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    cudaFree(base);
    if (cur != device) cudaSetDevice(cur);
  }
}

extern "C" {

int egt_abi_version(void) { return EGT_ABI_VERSION; }
const char* egt_last_error(void) { return g_err.c_str(); }
void egt_set_pdl(int enabled) { g_pdl = enabled != 0; }
uint64_t egt_launch_count(void) { return launch_counter(); }
void egt_tune_force_plan(int rb, int s, int nw, int nst, int ch) { force_plan(rb, s, nw, nst, ch); }
int egt_tune_read_trace(unsigned long long* host, size_t n, int reset) {
  const bool um = getenv("EGT_UMMA_TRACE") != nullptr;
  unsigned long long* b = um ? umma_trace_buffer() : tiled_trace_buffer();
  if (!b) return 1;
  n = std::min<size_t>(n, um ? 1024 : 8 * 4096);
  if (cudaMemcpy(host, b, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess) return 2;
  if (reset) cudaMemset(b, 0, sizeof(unsigned long long) * (um ? 1024 : 8 * 4096));
  return 0;
}

egt_status egt_dev_packed_create(const egt_packed_view* v, void* stream, egt_dev_packed** out) {
  return egt_dev_packed_create_ex(v, 0u, stream, out);
}

egt_status egt_dev_packed_create_ex(const egt_packed_view* v, uint32_t flags, void* stream, egt_dev_packed** out) {
  using namespace egt_fmt;
  if ((flags & ~EGT_UPLOAD_ROUND_FP16) != 0u) return fail(EGT_EINVAL, "egt_dev_packed_create: unknown flags");
  if (!out) return fail(EGT_EINVAL, "egt_dev_packed_create: null output");
  *out = nullptr;
  egt_status st = check_view(v);
  if (st != EGT_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t rows = v->rows, cols = v->cols;
  const uint64_t nnz = static_cast<uint64_t>(rows) * cols * v->n / 4;
  const bool i4 = v->kind == EGT_KIND_INT4;
  const int format = i4 ? (v->n == 2 ? I4_SP24 : I4_SP14) : (v->n == 2 ? F16_SP24 : F16_SP14);
  if (v->n != 1 && v->n != 2) return fail(EGT_EFORMAT, "packed matrix: bad keep count");

  Upload up;
  Carve c;
  const size_t o_words = c.add(v->n_index_words * 2);
  const size_t o_codes = i4 ? c.add(v->n_value_bytes) : 0;
  const size_t o_f32 = i4 ? 0 : c.add(nnz * 4);
  const size_t o_f16 = i4 ? 0 : c.add(nnz * 2);
  const size_t o_gs = i4 ? c.add(rows * 4ull) : 0;
  const size_t o_goff = i4 ? c.add((rows + 1ull) * 4) : 0;
  const size_t o_sc = i4 ? c.add(v->n_scales * 4) : 0;
  const size_t o_zp = i4 ? c.add(v->n_scales) : 0;
  const size_t o_err = c.add(16);
  CUDA_TRY(cudaMalloc(&up.base, c.total));
  uint8_t* b = static_cast<uint8_t*>(up.base);
  up.words = reinterpret_cast<uint16_t*>(b + o_words);
  up.err = reinterpret_cast<uint32_t*>(b + o_err);
  CUDA_TRY(cudaMemsetAsync(up.err, 0, 16, s));
  if (v->n_index_words)
    CUDA_TRY(cudaMemcpyAsync(up.words, v->index_words, v->n_index_words * 2, cudaMemcpyHostToDevice, s));
  if (i4) {
    up.codes = b + o_codes;
    up.gs = reinterpret_cast<uint32_t*>(b + o_gs);
    up.goff = reinterpret_cast<uint32_t*>(b + o_goff);
    up.scales = reinterpret_cast<float*>(b + o_sc);
    up.zps = b + o_zp;
    if (v->n_value_bytes)
      CUDA_TRY(cudaMemcpyAsync(up.codes, v->value_bytes, v->n_value_bytes, cudaMemcpyHostToDevice, s));
    if (rows) {
      CUDA_TRY(cudaMemcpyAsync(up.gs, v->group_sizes, rows * 4ull, cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(up.goff, v->group_offsets, (rows + 1ull) * 4, cudaMemcpyHostToDevice, s));
    }
    if (v->n_scales) {
      CUDA_TRY(cudaMemcpyAsync(up.scales, v->scales, v->n_scales * 4, cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(up.zps, v->zero_points, v->n_scales, cudaMemcpyHostToDevice, s));
    }
    CUDA_TRY(launch_validate_groups(up.gs, up.goff, rows, cols, v->n_scales, up.err, s));
  } else {
    up.f32 = reinterpret_cast<float*>(b + o_f32);
    up.f16 = reinterpret_cast<__half*>(b + o_f16);
    if (nnz) CUDA_TRY(cudaMemcpyAsync(up.f32, v->values, nnz * 4, cudaMemcpyHostToDevice, s));
    CUDA_TRY(launch_f32_to_f16(up.f32, up.f16, nnz, (flags & EGT_UPLOAD_ROUND_FP16) == 0u, up.err, s));
  }
  CUDA_TRY(launch_validate_offsets(up.words, rows, cols, v->n, up.err, s));
  st = finish_error_flag(up.err, s);
  if (st != EGT_OK) return st;
  return build_handle(format, v->n, v->kind, rows, cols, nnz, v->group_sizes, v->n_scales, up,
                      c.total, s, out);
}

egt_status egt_gemv_f32(const float* w, const float* x, float* y, uint32_t rows, uint32_t cols, void* stream) {
  if (static_cast<uint64_t>(rows) * cols && (!w || !x || !y)) return fail(EGT_EINVAL, "gemv: null argument");
  CUDA_TRY(launch_gemv_f32(w, x, y, rows, cols, static_cast<cudaStream_t>(stream)));
  return EGT_OK;
}

egt_status egt_gpu_importance(const float* w, const float* x_norms, const float* grad_abs, uint32_t rows,
                              uint32_t cols, float* scores, void* stream) {
  if (static_cast<uint64_t>(rows) * cols && (!w || !x_norms || !grad_abs || !scores))
    return fail(EGT_EINVAL, "importance: null argument");
  CUDA_TRY(launch_importance(w, x_norms, grad_abs, rows, cols, scores, static_cast<cudaStream_t>(stream)));
  return EGT_OK;
}

egt_status egt_gpu_prune_nm(const float* scores, uint32_t rows, uint32_t cols, int n, int m, uint8_t* mask,
                            void* stream) {
  if (m != 4) return fail(EGT_EINVAL, "prune_nm: group width must be 4");  // compress.cpp:247-249
  if (n < 1 || n >= m) return fail(EGT_EINVAL, "prune_nm: keep count must be in [1, group width)");
  if (static_cast<uint64_t>(rows) * cols && (!scores || !mask)) return fail(EGT_EINVAL, "prune_nm: null argument");
  CUDA_TRY(launch_prune_nm(scores, rows, cols, n, mask, static_cast<cudaStream_t>(stream)));
  return EGT_OK;
}

egt_status egt_gpu_quantize_pack(const float* w, const uint8_t* mask, uint32_t rows, uint32_t cols, int n,
                                 const uint32_t* group_sizes, const egt_gpu_packed_out* raw_out, void* stream,
                                 egt_dev_packed** out) {
  using namespace egt_fmt;
  if (out) *out = nullptr;
  if (!out && !raw_out) return fail(EGT_EINVAL, "gpu pack: nothing to produce");
  // pack's checks (packed.cpp:27-49) and quantize's (compress.cpp:157-176)
  if (n == 4) return fail(EGT_EINVAL, "pack: dense pattern unsupported");
  if (n < 1 || n > 4) return fail(EGT_EINVAL, "pack: keep count must be in [1, group width)");
  if (cols % 4 != 0) return fail(EGT_EINVAL, "pack: columns must be a multiple of the group width");
  if (rows && (!group_sizes || !w || !mask)) return fail(EGT_EINVAL, "gpu pack: null argument");
  std::vector<uint32_t> goff(rows + 1, 0);
  for (uint32_t r = 0; r < rows; ++r) {
    if (group_sizes[r] == 0) return fail(EGT_EINVAL, "quantize: zero group size");
    goff[r + 1] = goff[r] + (cols + group_sizes[r] - 1) / group_sizes[r];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t nnz = static_cast<uint64_t>(rows) * cols * n / 4;
  const uint64_t n_scales = goff[rows];
  Upload up;
  Carve c;
  const size_t o_words = c.add(((nnz + 7) / 8) * 2);
  const size_t o_codes = c.add((nnz + 1) / 2);
  const size_t o_gs = c.add(rows * 4ull);
  const size_t o_goff = c.add((rows + 1ull) * 4);
  const size_t o_sc = c.add(n_scales * 4);
  const size_t o_zp = c.add(n_scales);
  const size_t o_err = c.add(16);
  const size_t o_tmp = c.add(nnz);  // one code per kept entry before nibble packing
  CUDA_TRY(cudaMalloc(&up.base, c.total));
  uint8_t* b = static_cast<uint8_t*>(up.base);
  up.words = reinterpret_cast<uint16_t*>(b + o_words);
  up.codes = b + o_codes;
  up.gs = reinterpret_cast<uint32_t*>(b + o_gs);
  up.goff = reinterpret_cast<uint32_t*>(b + o_goff);
  up.scales = reinterpret_cast<float*>(b + o_sc);
  up.zps = b + o_zp;
  up.err = reinterpret_cast<uint32_t*>(b + o_err);
  auto* first_bad = reinterpret_cast<unsigned long long*>(up.err);
  CUDA_TRY(cudaMemsetAsync(up.err, 0xFF, 8, s));
  CUDA_TRY(cudaMemsetAsync(up.err + 2, 0, 8, s));
  if (rows) {
    CUDA_TRY(cudaMemcpyAsync(up.gs, group_sizes, rows * 4ull, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(up.goff, goff.data(), (rows + 1ull) * 4, cudaMemcpyHostToDevice, s));
  }
  CUDA_TRY(launch_check_nm(mask, rows, cols, n, first_bad, s));
  unsigned long long bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&bad, first_bad, sizeof bad, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (bad != ~0ull) {
    const uint32_t r = static_cast<uint32_t>(bad / (cols / 4)), c0 = static_cast<uint32_t>(bad % (cols / 4)) * 4;
    uint8_t bytes[2] = {0, 0};
    const uint64_t bit = static_cast<uint64_t>(r) * cols + c0;
    const uint64_t nbytes = (static_cast<uint64_t>(rows) * cols + 7) / 8;
    CUDA_TRY(cudaMemcpy(bytes, mask + bit / 8, (bit / 8 + 1 < nbytes) ? 2 : 1, cudaMemcpyDeviceToHost));
    const uint32_t word = bytes[0] | (static_cast<uint32_t>(bytes[1]) << 8);
    int kept = 0;
    for (int j = 0; j < 4; ++j) kept += (word >> ((bit % 8) + j)) & 1u;
    return fail(EGT_EINVAL, "pack: group at row " + std::to_string(r) + ", column " + std::to_string(c0) +
                                " keeps " + std::to_string(kept) + " entries (want " + std::to_string(n) + ")");
  }
  CUDA_TRY(launch_quantize_pack(w, mask, rows, cols, n, up.gs, up.goff, up.scales, up.zps, b + o_tmp, up.codes,
                                up.words, s));
  if (raw_out) {
    if (nnz && (!raw_out->index_words || !raw_out->value_bytes))
      return fail(EGT_EINVAL, "gpu pack: null output array");
    if (nnz) {
      CUDA_TRY(cudaMemcpyAsync(raw_out->index_words, up.words, ((nnz + 7) / 8) * 2, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(raw_out->value_bytes, up.codes, (nnz + 1) / 2, cudaMemcpyDeviceToDevice, s));
    }
    if (raw_out->group_offsets)
      CUDA_TRY(cudaMemcpyAsync(raw_out->group_offsets, up.goff, (rows + 1ull) * 4, cudaMemcpyDeviceToDevice, s));
    if (n_scales && raw_out->scales)
      CUDA_TRY(cudaMemcpyAsync(raw_out->scales, up.scales, n_scales * 4, cudaMemcpyDeviceToDevice, s));
    if (n_scales && raw_out->zero_points)
      CUDA_TRY(cudaMemcpyAsync(raw_out->zero_points, up.zps, n_scales, cudaMemcpyDeviceToDevice, s));
  }
  if (!out) {
    CUDA_TRY(cudaStreamSynchronize(s));
    return EGT_OK;
  }
  CUDA_TRY(cudaMemsetAsync(up.err, 0, 16, s));
  const int format = n == 2 ? I4_SP24 : I4_SP14;
  if (n != 1 && n != 2) return fail(EGT_EINVAL, "pack: keep count must be in [1, group width)");
  return build_handle(format, static_cast<uint8_t>(n), EGT_KIND_INT4, rows, cols, nnz, group_sizes, n_scales, up,
                      c.total, s, out);
}

egt_status egt_dev_dense_i4_create(const egt_quant_view* q, void* stream, egt_dev_packed** out) {
  using namespace egt_fmt;
  if (!out || !q) return fail(EGT_EINVAL, "egt_dev_dense_i4_create: null argument");
  *out = nullptr;
  const uint32_t rows = q->rows, cols = q->cols;
  if (q->n_codes != static_cast<size_t>(rows) * cols)
    return fail(EGT_EINVAL, "dense int4: code count differs from rows x cols");
  if (rows && (!q->group_offsets || q->group_offsets[rows] != q->n_scales))
    return fail(EGT_EFORMAT, "packed matrix: scale table size mismatch");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Upload up;
  Carve c;
  const size_t o_dense = c.add(q->n_codes);
  const size_t o_gs = c.add(rows * 4ull);
  const size_t o_goff = c.add((rows + 1ull) * 4);
  const size_t o_sc = c.add(q->n_scales * 4);
  const size_t o_zp = c.add(q->n_scales);
  const size_t o_err = c.add(16);
  CUDA_TRY(cudaMalloc(&up.base, c.total));
  uint8_t* b = static_cast<uint8_t*>(up.base);
  up.dense = b + o_dense;
  up.gs = reinterpret_cast<uint32_t*>(b + o_gs);
  up.goff = reinterpret_cast<uint32_t*>(b + o_goff);
  up.scales = reinterpret_cast<float*>(b + o_sc);
  up.zps = b + o_zp;
  up.err = reinterpret_cast<uint32_t*>(b + o_err);
  CUDA_TRY(cudaMemsetAsync(up.err, 0, 16, s));
  if (q->n_codes) CUDA_TRY(cudaMemcpyAsync(up.dense, q->codes, q->n_codes, cudaMemcpyHostToDevice, s));
  if (rows) {
    CUDA_TRY(cudaMemcpyAsync(up.gs, q->group_sizes, rows * 4ull, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(up.goff, q->group_offsets, (rows + 1ull) * 4, cudaMemcpyHostToDevice, s));
  }
  if (q->n_scales) {
    CUDA_TRY(cudaMemcpyAsync(up.scales, q->scales, q->n_scales * 4, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(up.zps, q->zero_points, q->n_scales, cudaMemcpyHostToDevice, s));
  }
  CUDA_TRY(launch_validate_groups(up.gs, up.goff, rows, cols, q->n_scales, up.err, s));
  egt_status st = finish_error_flag(up.err, s);
  if (st != EGT_OK) return st;
  return build_handle(I4_DENSE, 4, EGT_KIND_INT4, rows, cols, static_cast<uint64_t>(rows) * cols,
                      q->group_sizes, q->n_scales, up, c.total, s, out);
}

egt_status egt_dev_packed_slice_rows(const egt_dev_packed* h, uint32_t r0, uint32_t r1,
                                     egt_dev_packed** out) {
  if (!h || !out) return fail(EGT_EINVAL, "slice_rows: null argument");
  *out = nullptr;
  if (r0 > r1 || r1 > h->rows) return fail(EGT_EINVAL, "slice_rows: row range outside the matrix");
  auto s = std::make_unique<egt_dev_packed>();
  s->store = h->store;
  s->rows = r1 - r0;
  s->cols = h->cols;
  s->n = h->n;
  s->m = h->m;
  s->kind = h->kind;
  s->format = h->format;
  s->path = h->path;
  s->grouped_ok = h->grouped_ok;
  s->raw = h->raw;
  s->tiled = h->tiled;
  const double frac = h->rows ? static_cast<double>(r1 - r0) / h->rows : 0.0;
  s->nnz = static_cast<uint64_t>(s->rows) * (h->rows ? h->nnz / h->rows : 0);
  s->algorithmic_bytes = static_cast<uint64_t>(frac * h->algorithmic_bytes + 0.5);
  s->device_bytes = static_cast<uint64_t>(frac * h->device_bytes + 0.5);
  if (h->path == EGT_PATH_TILED) {
    if (r0 % 16 != 0 || (r1 % 16 != 0 && r1 != h->rows))
      return fail(EGT_EINVAL, "slice_rows: tiled shards must start and end on 16-row tiles");
    s->tiled.rt_begin = h->tiled.rt_begin + static_cast<int>(r0 / 16);
    s->tiled.RT = static_cast<int>((s->rows + 15) / 16);
  } else {
    s->raw.row_begin = h->raw.row_begin + r0;
  }
  *out = s.release();
  return EGT_OK;
}

egt_status egt_dev_packed_destroy(egt_dev_packed* h) {
  delete h;
  return EGT_OK;
}

egt_status egt_dev_packed_query(const egt_dev_packed* h, egt_dev_packed_info* info) {
  if (!h || !info) return fail(EGT_EINVAL, "query: null argument");
  info->rows = h->rows;
  info->cols = h->cols;
  info->n = h->n;
  info->m = h->m;
  info->kind = h->kind;
  info->format = h->tiled.pad14 ? egt_fmt::I4_SP14 : h->format;  // the stream's format (1:4 stored as 2:4)
  info->path = h->path;
  info->device_bytes = h->device_bytes;
  info->algorithmic_bytes = h->algorithmic_bytes;
  info->nnz = h->nnz;
  return EGT_OK;
}

namespace {
egt_status spmv_impl(const egt_dev_packed* h, const float* x, float* y, uint32_t M, uint32_t ldx, uint32_t ldy,
                     uint32_t flags, const float* res, uint32_t ldr, uint32_t input, float eps,
                     const egt_dev_packed* l2_next, void* stream, const egt_peer_group* pg = nullptr,
                     uint32_t row0 = 0) {
  const bool indep = (flags & EGT_SPMV_INDEPENDENT) != 0;
  if (!h) return fail(EGT_EINVAL, "spmv: null matrix");
  if (M == 0) return EGT_OK;
  if (ldx < h->cols) return fail(EGT_EINVAL, "spmv: input length differs from columns");
  if (M > 1 && ldy < h->rows) return fail(EGT_EINVAL, "spmv: output stride below rows");
  if (input > EGT_INPUT_SILU) return fail(EGT_EINVAL, "spmv: unknown input transform");
  if (res && M > 1 && ldr < h->rows) return fail(EGT_EINVAL, "spmv: residual stride below rows");
  if (h->rows == 0) {
    if (pg) CUDA_TRY(launch_peer_signal(pg, true, (flags & EGT_PEER_NOWAIT) == 0, static_cast<cudaStream_t>(stream)));
    return EGT_OK;
  }
  if (!x || !y) return fail(EGT_EINVAL, "spmv: null vector");
  if (pg && (h->path != EGT_PATH_TILED || h->cols == 0 || M > 16))
    return fail(EGT_EINVAL, "spmv allgather: tiled-path shards with columns, at most 16 tokens");
  if (input == EGT_INPUT_RMSNORM && (ldx % 4 != 0 || h->cols % 4 != 0 || reinterpret_cast<uintptr_t>(x) % 16 != 0))
    return fail(EGT_EINVAL, "spmv: rmsnorm input needs 16-byte aligned rows of a multiple of 4 floats");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LaunchCtx ctx;
  ctx.stream = s;
  ctx.pdl = g_pdl;
  ctx.xform = static_cast<int>(input);
  ctx.eps = eps;
  ctx.res = res;
  ctx.ldr = static_cast<int>(M > 1 ? ldr : h->rows);
  ctx.l2_next = l2_next;
  ctx.out_silu = (flags & EGT_SPMV_OUTPUT_SILU) != 0 ? 1 : 0;
  if (pg) {
    ctx.npeer = static_cast<int>(pg->world);
    ctx.peer_rank = static_cast<int>(pg->rank);
    ctx.peer_row0 = static_cast<int>(row0);
    ctx.peer_wait = (flags & EGT_PEER_NOWAIT) ? 0 : 1;
    ctx.peer_ctrl = pg->ctrl;
    for (uint32_t i = 0; i < pg->world; ++i) {
      ctx.peer_y[i] = pg->y[i];
      ctx.peer_flag[i] = pg->flags[i];
    }
  }
  if (h->cols == 0) {
    for (uint32_t m = 0; m < M; ++m) {
      float* ym = y + static_cast<size_t>(m) * ldy;
      if (res)
        CUDA_TRY(cudaMemcpyAsync(ym, res + static_cast<size_t>(m) * ctx.ldr, h->rows * sizeof(float),
                                 cudaMemcpyDeviceToDevice, s));
      else
        CUDA_TRY(cudaMemsetAsync(ym, 0, h->rows * sizeof(float), s));
    }
    return EGT_OK;
  }
  static const bool no_grouped = getenv("EGT_NO_GROUPED") != nullptr;  // tuning: the warp-per-row kernel
  if (h->path == EGT_PATH_GENERAL && !no_grouped && grouped_stream_ok(h, 1) && !pg && ldx % 4 == 0 &&
      reinterpret_cast<uintptr_t>(x) % 16 == 0) {
    // up to four tokens per launch (x staged in shared memory); more tokens
    // run as several launches over token groups (rows and tokens independent)
    uint32_t mt = 4;
    while (mt > 1 && !grouped_stream_ok(h, static_cast<int>(mt))) --mt;
    for (uint32_t m0 = 0; m0 < M; m0 += mt) {
      const int mc = static_cast<int>(std::min<uint32_t>(mt, M - m0));
      LaunchCtx c2 = ctx;
      if (c2.res) c2.res += static_cast<size_t>(m0) * c2.ldr;
      CUDA_TRY(launch_grouped_stream(h, x + static_cast<size_t>(m0) * ldx, static_cast<int>(ldx), mc,
                                     y + static_cast<size_t>(m0) * ldy, static_cast<int>(ldy), c2));
    }
    return EGT_OK;
  }
  if (h->path == EGT_PATH_GENERAL) {
    if (res || input != EGT_INPUT_NONE || ctx.out_silu)
      return fail(EGT_EINVAL, "spmv: fused input transforms / residual need the tiled path (group sizes % 32 == 0)");
    CUDA_TRY(launch_general(h, x, static_cast<int>(ldx), static_cast<int>(M), y,
                            static_cast<int>(ldy), ctx));
    return EGT_OK;
  }
  if (M > 1 && !pg && (input == EGT_INPUT_NONE || input == EGT_INPUT_RMSNORM) && !plan_forced() && umma_eligible(h, static_cast<int>(M))) {
    // tcgen05 / TMEM many-token kernel (umma_spmm.cu): x stages + per-token
    // range, then split-K partials, in one per-stream workspace
    const int ns = num_sms();
    const size_t xs = (umma_workspace_bytes(h, static_cast<int>(M)) + 255) / 256 * 256;
    const size_t pf = umma_partial_floats(h, static_cast<int>(M), ns);
    Workspace* w = nullptr;
    egt_status st = get_workspace(s, xs / 4 + pf, umma_counters(h, static_cast<int>(M), ns), &w);
    if (st != EGT_OK) return st;
    ctx.partial = w->partial + xs / 4;
    ctx.counters = w->counters;
    CUDA_TRY(launch_umma(h, x, static_cast<int>(ldx), static_cast<int>(M), y, static_cast<int>(ldy),
                         reinterpret_cast<uint8_t*>(w->partial), ctx, ns));
    return EGT_OK;
  }
  static const bool no_wide = getenv("EGT_NO_WIDE") != nullptr;  // tuning: old M > 16 path
  // (16-column groups: the token-tiled kernel below, 16 tokens per block)
  if (M > 16 && !pg && input == EGT_INPUT_NONE && !no_wide && !plan_forced() && h->tiled.SS != 0) {
    Workspace* w = nullptr;
    egt_status st = get_workspace(s, (wide_workspace_bytes(h, static_cast<int>(M)) + 3) / 4, 0, &w);
    if (st != EGT_OK) return st;
    CUDA_TRY(launch_wide(h, x, static_cast<int>(ldx), static_cast<int>(M), y, static_cast<int>(ldy),
                         reinterpret_cast<uint32_t*>(w->partial), ctx, num_sms()));
    return EGT_OK;
  }
  TiledSchedule sc;
  if (plan_forced()) {
    sc = plan_tiled(h, static_cast<int>(M), num_sms(), indep);
  } else {
    std::lock_guard<std::mutex> lk(h->plan_mu);
    const int key = static_cast<int>(M) * 2 + (indep ? 1 : 0);
    auto it = h->plans.find(key);
    if (it == h->plans.end()) {
      it = h->plans.emplace(key, plan_tiled(h, M, num_sms(), indep)).first;
      if (getenv("EGT_DEBUG_PLAN")) {
        const TiledSchedule& p = it->second;
        fprintf(stderr,
                "[egt plan] %ux%u fmt=%d M=%u indep=%d: RB=%d nw=%d KC=%d CH=%d NST=%d S=%d NT=%d grid=(%d,%d,%d) smem=%zu\n",
                h->rows, h->cols, h->format, M, indep ? 1 : 0, p.RB, p.nw, p.KC, p.CH, p.NST, p.S, p.NT,
                p.grid_x, p.grid_y, p.grid_z, p.smem);
      }
    }
    sc = it->second;
  }
  if (sc.smem == 0) return fail(EGT_EINTERNAL, "spmv: no feasible launch plan for this shape and token count");
  // A split-K plan (the planner's fallback when no split-free independent
  // plan fits) always launches dependent: its partials and arrival counters
  // live in the shared workspace, which only stream order protects.
  const bool run_indep = indep && sc.S <= 1;
  if (sc.S > 1) {
    const size_t fl = tiled_workspace_floats(h, sc, M), nc = static_cast<size_t>(sc.grid_x) * sc.grid_z;
    Workspace* w = nullptr;
    egt_status st = get_workspace(s, fl, nc, &w);
    if (st != EGT_OK) return st;
    ctx.partial = w->partial;
    ctx.counters = w->counters;
  }
  CUDA_TRY(launch_tiled(h, sc, x, static_cast<int>(ldx), static_cast<int>(M), y,
                        static_cast<int>(ldy), ctx, run_indep));
  return EGT_OK;
}
}  // namespace

egt_status egt_spmv_ex(const egt_dev_packed* h, const float* x, float* y, uint32_t M, uint32_t ldx,
                       uint32_t ldy, uint32_t flags, void* stream) {
  return spmv_impl(h, x, y, M, ldx, ldy, flags, nullptr, 0, EGT_INPUT_NONE, 0.f, nullptr, stream);
}

egt_status egt_spmm_multi(const egt_dev_packed* const* hs, uint32_t n, const float* x, uint32_t M, uint32_t ldx,
                          float* const* ys, uint32_t ldy, uint32_t input, float eps, void* stream) {
  if (input != EGT_INPUT_NONE && input != EGT_INPUT_RMSNORM)
    return fail(EGT_EINVAL, "spmm multi: input transform must be none or rmsnorm");
  if (!hs || !ys || n == 0 || n > 3) return fail(EGT_EINVAL, "spmm multi: 1 to 3 matrices");
  const egt_dev_packed* h = hs[0];
  if (!h || (!x && M > 0)) return fail(EGT_EINVAL, "spmm multi: null argument");
  bool same = true;
  for (uint32_t i = 0; i < n; ++i) {
    const egt_dev_packed* g = hs[i];
    if (!g || !ys[i]) return fail(EGT_EINVAL, "spmm multi: null argument");
    if (g->cols != h->cols) return fail(EGT_EINVAL, "spmm multi: matrices must share their columns");
    same = same && g->path == h->path && g->rows == h->rows && g->format == h->format &&
           g->tiled.KQ == h->tiled.KQ && g->tiled.SS == h->tiled.SS && g->tiled.pad14 == h->tiled.pad14;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n > 1 && same && M > 1 && h->cols > 0 && h->rows > 0 && umma_eligible(h, static_cast<int>(M))) {
    if (ldx < h->cols || ldy < h->rows) return fail(EGT_EINVAL, "spmm multi: leading dimension too small");
    LaunchCtx ctx;
    ctx.stream = s;
    ctx.pdl = g_pdl;
    ctx.xform = static_cast<int>(input);
    ctx.eps = eps;
    const int ns = num_sms();
    const size_t xs = (umma_workspace_bytes(h, static_cast<int>(M)) + 255) / 256 * 256;
    const size_t pf = umma_partial_floats(h, static_cast<int>(M), ns);
    Workspace* w = nullptr;
    egt_status st = get_workspace(s, xs / 4 + pf, umma_counters(h, static_cast<int>(M), ns), &w);
    if (st != EGT_OK) return st;
    ctx.partial = w->partial + xs / 4;
    ctx.counters = w->counters;
    CUDA_TRY(launch_umma_multi(hs, static_cast<int>(n), x, static_cast<int>(ldx), static_cast<int>(M), ys,
                               static_cast<int>(ldy), reinterpret_cast<uint8_t*>(w->partial), ctx, ns));
    return EGT_OK;
  }
  for (uint32_t i = 0; i < n; ++i) {
    const egt_status st = egt_spmv_fused(hs[i], x, ys[i], M, ldx, ldy, nullptr, 0, input, eps,
                                         i ? EGT_SPMV_INDEPENDENT : 0u, nullptr, stream);
    if (st != EGT_OK) return st;
  }
  return EGT_OK;
}

egt_status egt_spmv_fused_multi(const egt_dev_packed* const* hs, uint32_t n, const float* x, float* const* ys,
                                uint32_t input, float eps, uint32_t flags, void* stream) {
  if (!hs || !ys || n == 0 || n > 3) return fail(EGT_EINVAL, "spmv multi: 1 to 3 matrices");
  const egt_dev_packed* h = hs[0];
  if (!h || !x) return fail(EGT_EINVAL, "spmv multi: null argument");
  for (uint32_t i = 0; i < n; ++i) {
    const egt_dev_packed* g = hs[i];
    if (!g || !ys[i]) return fail(EGT_EINVAL, "spmv multi: null argument");
    if (g->path != EGT_PATH_TILED || g->rows != h->rows || g->cols != h->cols || g->format != h->format ||
        g->tiled.KQ != h->tiled.KQ || g->tiled.SS != h->tiled.SS)
      return fail(EGT_EINVAL, "spmv multi: matrices must share shape, format and group layout on the tiled path");
  }
  if (n > 1 && h->rows % 16 != 0) return fail(EGT_EINVAL, "spmv multi: rows must be a multiple of 16");
  if (input > EGT_INPUT_SILU) return fail(EGT_EINVAL, "spmv: unknown input transform");
  if (n == 1) return spmv_impl(h, x, ys[0], 1, h->cols, h->rows, flags, nullptr, 0, input, eps, nullptr, stream);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LaunchCtx ctx;
  ctx.stream = s;
  ctx.pdl = g_pdl;
  ctx.xform = static_cast<int>(input);
  ctx.eps = eps;
  ctx.out_silu = (flags & EGT_SPMV_OUTPUT_SILU) != 0 ? 1 : 0;
  ctx.nseg = static_cast<int>(n);
  for (uint32_t i = 0; i < n; ++i) {
    ctx.segs[i] = hs[i];
    ctx.seg_y[i] = ys[i];
  }
  const bool indep = (flags & EGT_SPMV_INDEPENDENT) != 0;
  const TiledSchedule sc = plan_tiled_rt(h, h->tiled.RT * static_cast<int>(n), 1, num_sms(), indep);
  if (sc.smem == 0) return fail(EGT_EINTERNAL, "spmv: no feasible launch plan for this shape and token count");
  const bool run_indep = indep && sc.S <= 1;  // split-K plans launch dependent (see spmv_impl)
  if (sc.S > 1) {
    const size_t fl = static_cast<size_t>(sc.S) * h->tiled.RT * n * 16, nc = static_cast<size_t>(sc.grid_x) * sc.grid_z;
    Workspace* w = nullptr;
    egt_status st = get_workspace(s, fl, nc, &w);
    if (st != EGT_OK) return st;
    ctx.partial = w->partial;
    ctx.counters = w->counters;
  }
  CUDA_TRY(launch_tiled(h, sc, x, static_cast<int>(h->cols), 1, ys[0], static_cast<int>(h->rows), ctx, run_indep));
  return EGT_OK;
}

egt_status egt_spmv_allgather(const egt_dev_packed* shard, const float* x, uint32_t M, uint32_t ldx,
                              egt_peer_group* g, uint32_t row0, uint32_t ldy, uint32_t flags, void* stream) {
  if (!g) return fail(EGT_EINVAL, "spmv allgather: null peer group");
  if (!shard) return fail(EGT_EINVAL, "spmv: null matrix");
  if (static_cast<uint64_t>(row0) + shard->rows > ldy)
    return fail(EGT_EINVAL, "spmv allgather: shard rows past the gathered output stride");
  if (M == 0) return EGT_OK;
  // With peers, calls on one group share the arrival counter (peer_ctrl[1])
  // and the sequence target: two calls in flight at once would mix their
  // counts, so exchanging calls always launch dependent (stream-ordered).
  const uint32_t keep = g->world > 1 ? EGT_PEER_NOWAIT : (EGT_SPMV_INDEPENDENT | EGT_PEER_NOWAIT);
  return spmv_impl(shard, x, g->y[g->rank], M, ldx, ldy, flags & keep, nullptr,
                   0, EGT_INPUT_NONE, 0.f, nullptr, stream, g, row0);
}

egt_status egt_spmv_fused(const egt_dev_packed* h, const float* x, float* y, uint32_t M, uint32_t ldx,
                          uint32_t ldy, const float* residual, uint32_t ldr, uint32_t input, float eps,
                          uint32_t flags, const egt_dev_packed* l2_next, void* stream) {
  return spmv_impl(h, x, y, M, ldx, ldy, flags, residual, ldr, input, eps, l2_next, stream);
}

egt_status egt_spmv(const egt_dev_packed* h, const float* x, float* y, uint32_t M, uint32_t ldx,
                    uint32_t ldy, void* stream) {
  return egt_spmv_ex(h, x, y, M, ldx, ldy, 0u, stream);
}

egt_status egt_spmv_host(const egt_dev_packed* h, const float* x_host, size_t x_len, float* y_host,
                         void* stream) {
  if (!h) return fail(EGT_EINVAL, "spmv: null matrix");
  if (x_len != h->cols) return fail(EGT_EINVAL, "spmv: input length differs from columns");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  float* dx = nullptr;
  float* dy = nullptr;
  const size_t xb = std::max<size_t>(h->cols, 1) * sizeof(float);
  const size_t yb = std::max<size_t>(h->rows, 1) * sizeof(float);
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dx), xb + yb, s));
  dy = dx + std::max<size_t>(h->cols, 1);
  egt_status st = EGT_OK;
  cudaError_t e = cudaMemcpyAsync(dx, x_host, h->cols * sizeof(float), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    st = egt_spmv(h, dx, dy, 1, h->cols, h->rows, stream);
    if (st == EGT_OK)
      e = cudaMemcpyAsync(y_host, dy, h->rows * sizeof(float), cudaMemcpyDeviceToHost, s);
  }
  cudaFreeAsync(dx, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (st != EGT_OK) return st;
  if (e != cudaSuccess) return fail(EGT_ECUDA, std::string("spmv_host: ") + cudaGetErrorString(e));
  return EGT_OK;
}

egt_status egt_dequant(const egt_dev_packed* h, float* w, uint8_t* mask, void* stream) {
  if (!h || (!w && h->rows && h->cols)) return fail(EGT_EINVAL, "dequant: null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n = static_cast<size_t>(h->rows) * h->cols;
  if (n == 0) return EGT_OK;
  CUDA_TRY(cudaMemsetAsync(w, 0, n * sizeof(float), s));
  if (mask) {
    // the kernel ORs whole 32-bit words: the buffer holds ceil(n/32) words
    CUDA_TRY(cudaMemsetAsync(mask, 0, (n + 31) / 32 * 4, s));
  }
  CUDA_TRY(launch_dequant(h, w, mask, s));
  return EGT_OK;
}

}  // extern "C"
