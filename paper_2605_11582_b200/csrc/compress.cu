// GPU compression: the step before the SparseGemv path,
// for re-compressing 7B/70B-sized layers on the device.  Byte-identical to
// the host encoder (csrc/host/encoder.cpp) and the reference:
//   importance_scores  compress.cpp:230-244
//   prune_nm           compress.cpp:246-278
//   quantize_impl      compress.cpp:157-197 (fit_group :77-90, encode :92-96)
//   pack (INT4)        packed.cpp:92-128 (index stream :51-88, check :34-49)
// Everything is elementwise or per (row, group): HBM-bound, one pass over
// the weights for the fit + codes, no sort (ranks within a group of 4 are
// computed by comparison).
#include "device_common.cuh"
#include "handle.h"

namespace egt_impl {
namespace {

__device__ __forceinline__ bool mask_bit(const uint8_t* m, uint64_t i) { return (m[i >> 3] >> (i & 7)) & 1u; }

__global__ void importance_kernel(const float* __restrict__ w, const float* __restrict__ xn,
                                  const float* __restrict__ g, uint32_t rows, uint32_t cols,
                                  float* __restrict__ out) {
  const uint64_t n = static_cast<uint64_t>(rows) * cols;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float a = fabsf(w[i]);
    // two f32 products then one f32 sum, no contraction (the reference's order)
    out[i] = __fadd_rn(__fmul_rn(a, xn[i % cols]), __fmul_rn(a, g[i]));
  }
}

// One thread per mask byte: each of its 8 bits decides membership in the
// top-min(n, #positive) of its group of 4 (ties to the lower column) by
// counting the group's entries that sort before it.
__global__ void prune_kernel(const float* __restrict__ sc, uint32_t rows, uint32_t cols, int n,
                             uint8_t* __restrict__ mask) {
  const uint64_t total = static_cast<uint64_t>(rows) * cols;
  const uint64_t nbytes = (total + 7) / 8;
  for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < nbytes;
       b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t byte = 0;
    for (int k = 0; k < 8; ++k) {
      const uint64_t i = b * 8 + k;
      if (i >= total) break;
      const uint32_t r = static_cast<uint32_t>(i / cols), c = static_cast<uint32_t>(i % cols);
      const float v = sc[i];
      if (!(v > 0.0f)) continue;
      const uint32_t start = c & ~3u, end = min(start + 4u, cols);
      int before = 0;
      for (uint32_t o = start; o < end; ++o) {
        if (o == c) continue;
        const float u = sc[static_cast<uint64_t>(r) * cols + o];
        if (u > 0.0f && (u > v || (u == v && o < c))) ++before;
      }
      if (before < n) byte |= 1u << k;
    }
    mask[b] = static_cast<uint8_t>(byte);
  }
}

// check_mask_shape (packed.cpp:34-49): the first (row-major) group of 4 that
// does not keep exactly n entries.
__global__ void check_nm_kernel(const uint8_t* __restrict__ mask, uint32_t rows, uint32_t cols, int n,
                                unsigned long long* first_bad) {
  const uint64_t quads = static_cast<uint64_t>(rows) * (cols / 4);
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < quads;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i0 = (q / (cols / 4)) * cols + (q % (cols / 4)) * 4;
    int kept = 0;
    for (int j = 0; j < 4; ++j) kept += mask_bit(mask, i0 + j);
    if (kept != n) atomicMin(first_bad, static_cast<unsigned long long>(q));
  }
}

// fit_group + encode_value per (row, group): one warp per group, a block per
// row.  min / max of the retained values are exact in f32; the fit itself is
// in double as in the reference; codes use the f32-rounded scale.  codes[k]
// = code of the k-th kept entry of the matrix (row-major), one byte each.
__global__ void __launch_bounds__(256) quantize_kernel(const float* __restrict__ w, const uint8_t* __restrict__ mask,
                                                       uint32_t cols, int n, const uint32_t* __restrict__ gs,
                                                       const uint32_t* __restrict__ goff, float* __restrict__ scales,
                                                       uint8_t* __restrict__ zps, uint8_t* __restrict__ codes) {
  const uint32_t r = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint32_t g = gs[r];
  const uint32_t ngroups = goff[r + 1] - goff[r];
  const uint64_t row0 = static_cast<uint64_t>(r) * cols;
  const uint64_t k_row = static_cast<uint64_t>(r) * (cols / 4) * n;
  for (uint32_t gi = warp; gi < ngroups; gi += nw) {
    const uint32_t start = gi * g, end = min(start + g, cols);
    float mn = INFINITY, mx = -INFINITY;
    int cnt = 0;
    for (uint32_t c = start + lane; c < end; c += 32)
      if (mask_bit(mask, row0 + c)) {
        const float v = w[row0 + c];
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
        ++cnt;
      }
    for (int off = 16; off > 0; off >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    }
    float scale = 1e-8f;  // GroupParams defaults for a group with nothing retained
    uint32_t zp = 0;
    if (cnt > 0) {
      const double sd = fmax(1e-8, __dsub_rn(static_cast<double>(mx), static_cast<double>(mn)) / 15.0);
      zp = static_cast<uint32_t>(fmin(fmax(round(-static_cast<double>(mn) / sd), 0.0), 15.0));
      scale = static_cast<float>(sd);
    }
    if (lane == 0) {
      scales[goff[r] + gi] = scale;
      zps[goff[r] + gi] = static_cast<uint8_t>(zp);
    }
    for (uint32_t c = start + lane; c < end; c += 32)
      if (mask_bit(mask, row0 + c)) {
        const uint32_t q0 = c & ~3u;
        int rank = 0;
        for (uint32_t o = q0; o < c; ++o) rank += mask_bit(mask, row0 + o);
        const double code = round(static_cast<double>(w[row0 + c]) / static_cast<double>(scale)) +
                            static_cast<double>(zp);
        codes[k_row + static_cast<uint64_t>(q0 / 4) * n + rank] =
            static_cast<uint8_t>(fmin(fmax(code, 0.0), 15.0));
      }
  }
}

// value bytes: two codes per byte, the first in the low nibble.
__global__ void nibble_kernel(const uint8_t* __restrict__ codes, uint64_t nnz, uint8_t* __restrict__ out) {
  const uint64_t nb = (nnz + 1) / 2;
  for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < nb;
       b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t lo = codes[2 * b];
    const uint32_t hi = 2 * b + 1 < nnz ? codes[2 * b + 1] : 0u;
    out[b] = static_cast<uint8_t>(lo | (hi << 4));
  }
}

// 2bit-CSR index words: kept slot k (row-major) -> offset in its group of 4,
// eight per u16, slot i in bits [15-2i, 14-2i], the last word zero-padded.
__global__ void index_kernel(const uint8_t* __restrict__ mask, uint32_t cols, int n, uint64_t nnz,
                             uint16_t* __restrict__ words) {
  const uint64_t nwords = (nnz + 7) / 8;
  const uint64_t row_nnz = static_cast<uint64_t>(cols / 4) * n;
  for (uint64_t wi = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; wi < nwords;
       wi += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t word = 0;
    for (int slot = 0; slot < 8; ++slot) {
      const uint64_t k = wi * 8 + slot;
      if (k >= nnz) break;
      const uint64_t r = k / row_nnz, l = k % row_nnz;
      const uint64_t base = r * cols + (l / n) * 4;
      int j = static_cast<int>(l % n), off = 0;
      for (; off < 4; ++off)
        if (mask_bit(mask, base + off) && j-- == 0) break;
      word |= static_cast<uint32_t>(off & 3) << (14 - 2 * slot);
    }
    words[wi] = static_cast<uint16_t>(word);
  }
}

inline int grid_for(uint64_t items, int threads) {
  const uint64_t b = (items + threads - 1) / threads;
  return static_cast<int>(std::min<uint64_t>(std::max<uint64_t>(b, 1), 148ull * 16));
}

}  // namespace

cudaError_t launch_importance(const float* w, const float* xn, const float* g, uint32_t rows, uint32_t cols,
                              float* out, cudaStream_t s) {
  const uint64_t n = static_cast<uint64_t>(rows) * cols;
  if (n == 0) return cudaSuccess;
  importance_kernel<<<grid_for(n, 256), 256, 0, s>>>(w, xn, g, rows, cols, out);
  return cudaGetLastError();
}

cudaError_t launch_prune_nm(const float* scores, uint32_t rows, uint32_t cols, int n, uint8_t* mask,
                            cudaStream_t s) {
  const uint64_t nb = (static_cast<uint64_t>(rows) * cols + 7) / 8;
  if (nb == 0) return cudaSuccess;
  prune_kernel<<<grid_for(nb, 256), 256, 0, s>>>(scores, rows, cols, n, mask);
  return cudaGetLastError();
}

cudaError_t launch_check_nm(const uint8_t* mask, uint32_t rows, uint32_t cols, int n,
                            unsigned long long* first_bad, cudaStream_t s) {
  const uint64_t q = static_cast<uint64_t>(rows) * (cols / 4);
  if (q == 0) return cudaSuccess;
  check_nm_kernel<<<grid_for(q, 256), 256, 0, s>>>(mask, rows, cols, n, first_bad);
  return cudaGetLastError();
}

cudaError_t launch_quantize_pack(const float* w, const uint8_t* mask, uint32_t rows, uint32_t cols, int n,
                                 const uint32_t* gs, const uint32_t* goff, float* scales, uint8_t* zps,
                                 uint8_t* codes_tmp, uint8_t* value_bytes, uint16_t* words, cudaStream_t s) {
  const uint64_t nnz = static_cast<uint64_t>(rows) * cols * n / 4;
  if (rows == 0) return cudaSuccess;
  quantize_kernel<<<rows, 256, 0, s>>>(w, mask, cols, n, gs, goff, scales, zps, codes_tmp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || nnz == 0) return e;
  nibble_kernel<<<grid_for((nnz + 1) / 2, 256), 256, 0, s>>>(codes_tmp, nnz, value_bytes);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  index_kernel<<<grid_for((nnz + 7) / 8, 256), 256, 0, s>>>(mask, cols, n, nnz, words);
  return cudaGetLastError();
}

}  // namespace egt_impl
