// Upload-time validation and re-tiling, the general (reference-order) CUDA-core
// SpGEMV, and the bit-exact device unpack.
#include "device_common.cuh"
#include "handle.h"
#include "egt_b200.h"

namespace egt_impl {
using namespace egt_dev;
using namespace egt_fmt;

uint64_t& launch_counter() {
  static thread_local uint64_t n = 0;
  return n;
}

// offset_at (packed.hpp:64-66)
__device__ __forceinline__ uint32_t offset_at(const uint16_t* words, uint64_t k) {
  return (static_cast<uint32_t>(words[k >> 3]) >> (14 - 2 * (k & 7))) & 3u;
}
__device__ __forceinline__ uint32_t nibble_at(const uint8_t* codes, uint64_t k) {
  return (codes[k >> 1] >> (4 * (k & 1))) & 0xFu;
}
// decode_value (compress.cpp:98-101), with explicit rounding so nothing is
// contracted: (f32(code) - f32(zp)) * scale.
__device__ __forceinline__ float decode(uint32_t code, uint32_t zp, float scale) {
  return __fmul_rn(__fsub_rn(static_cast<float>(code), static_cast<float>(zp)), scale);
}

// ------------------------------------------------------------- validation
// for_each_nonzero's order check (packed.cpp:176-178): within a group of n
// kept entries the offsets strictly increase.  Done once at upload.
__global__ void validate_offsets_kernel(const uint16_t* words, uint32_t rows, uint32_t cols, int n,
                                        uint32_t* err) {
  const uint64_t groups = static_cast<uint64_t>(rows) * (cols / 4);
  for (uint64_t G = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; G < groups;
       G += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = G * n;
    uint32_t prev = offset_at(words, k);
    for (int i = 1; i < n; ++i) {
      const uint32_t off = offset_at(words, k + i);
      if (off <= prev) atomicOr(err, 1u);
      prev = off;
    }
  }
}

// Group tables must index inside the scale table for every column (the
// reference indexes them unchecked, packed.cpp:189-191).
__global__ void validate_groups_kernel(const uint32_t* gs, const uint32_t* goff, uint32_t rows,
                                       uint32_t cols, uint64_t n_scales, uint32_t* err) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const uint32_t g = gs[r];
  if (g == 0) {
    atomicOr(err, 2u);
    return;
  }
  const uint64_t ng = (static_cast<uint64_t>(cols) + g - 1) / g;
  if (static_cast<uint64_t>(goff[r]) + ng > n_scales) atomicOr(err, 4u);
}

cudaError_t launch_validate_offsets(const uint16_t* words, uint32_t rows, uint32_t cols, int n,
                                    uint32_t* err, cudaStream_t s) {
  if (n < 2 || rows == 0 || cols == 0) return cudaSuccess;
  validate_offsets_kernel<<<1184, 256, 0, s>>>(words, rows, cols, n, err);
  ++launch_counter();
  return cudaGetLastError();
}

cudaError_t launch_validate_groups(const uint32_t* gs, const uint32_t* goff, uint32_t rows,
                                   uint32_t cols, uint64_t n_scales, uint32_t* err,
                                   cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  validate_groups_kernel<<<(rows + 255) / 256, 256, 0, s>>>(gs, goff, rows, cols, n_scales, err);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------- re-tiling
// One thread per (row tile, k-quad, lane): gathers exactly the bits the lane
// will consume (tiled_format.h) from the reference-order stream.
struct RelayoutArgs {
  RawStream raw;
  int format;
  uint32_t rows, cols;
  int KQ, RT, SS, E;
  uint8_t* vals;
  uint8_t* meta;
  float* scales;
  uint8_t* zps;
  int pad14;  // raw stream is INT4 1:4, written as 2:4 with zero-valued partners
};

__device__ __forceinline__ bool group_valid(const RelayoutArgs& a, uint32_t r, uint32_t G) {
  return r < a.rows && G * 4 < a.cols;
}

__global__ void relayout_kernel(const RelayoutArgs a) {
  const uint64_t total = static_cast<uint64_t>(a.RT) * a.KQ * 32;
  const uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (idx >= total) return;
  const int lane = static_cast<int>(idx & 31);
  const uint64_t blk = idx >> 5;
  const int kq = static_cast<int>(blk % a.KQ);
  const int rt = static_cast<int>(blk / a.KQ);
  const int g = lane >> 2, t = lane & 3;
  const int f = a.format;
  const int n = a.pad14 ? 1 : keep_n(f);
  const uint64_t row_nnz = static_cast<uint64_t>(a.cols) * (n == 4 ? 4 : n) / 4;
  const RawStream& raw = a.raw;
  // INT4 1:4 as 2:4: the kept entry at offset o of its group of 4 is paired
  // with a partner carrying the group's zero point (so c - z = 0 exactly):
  // o = 0,1,2 -> (o, o+1) kept first; o = 3 -> (1, 3) kept second.
  auto pad_pair = [&](uint32_t r, uint32_t G, uint32_t* c0, uint32_t* c1, uint32_t* nib) {
    const uint64_t R = raw.row_begin + r;
    const uint64_t k = R * row_nnz + G;
    const uint32_t off = offset_at(raw.words, k), code = nibble_at(raw.codes, k);
    const uint32_t col = G * 4 + off;
    const uint32_t z = raw.zps[raw.group_offsets[R] + col / raw.group_sizes[R]];
    if (off < 3) {
      *c0 = code, *c1 = z, *nib = off | ((off + 1) << 2);
    } else {
      *c0 = z, *c1 = code, *nib = 1u | (3u << 2);
    }
  };

  if (f == I4_SP24 || f == F16_SP24) {
    uint32_t v[16] = {0};
    for (int j = 0; j < 4; ++j)
      for (int h = 0; h < 2; ++h)
        for (int q = 0; q < 2; ++q) {
          const uint32_t r = rt * 16 + g + 8 * h;
          const uint32_t G = (kq * 4 + j) * 8 + t + 4 * q;
          const int p = h + 2 * q;
          if (!group_valid(a, r, G)) {
            continue;  // codes 0 / values 0 (scale 0 / x 0 make them inert)
          }
          const uint64_t k0 = (raw.row_begin + r) * row_nnz + 2ull * G;
          if (a.pad14) {
            uint32_t c0, c1, nib;
            pad_pair(r, G, &c0, &c1, &nib);
            v[j] |= c0 << (4 * p);
            v[j] |= c1 << (16 + 4 * p);
          } else if (f == I4_SP24) {
            v[j] |= nibble_at(raw.codes, k0) << (4 * p);
            v[j] |= nibble_at(raw.codes, k0 + 1) << (16 + 4 * p);
          } else {
            v[4 * j + p] = static_cast<uint32_t>(__half_as_ushort(raw.values[k0])) |
                           (static_cast<uint32_t>(__half_as_ushort(raw.values[k0 + 1])) << 16);
          }
        }
    const int VB = val_lane_bytes(f);
    uint32_t* vo = reinterpret_cast<uint32_t*>(a.vals + blk * 32 * VB + lane * VB);
    for (int i = 0; i < VB / 4; ++i) vo[i] = v[i];
    // mma.sp metadata: lane t = 2*sel + hh of a quad holds groups
    // [4hh, 4hh+4) of its k-tile, row g in bits [0,16) and row g+8 in [16,32).
    uint32_t m[2];
    for (int sl = 0; sl < 2; ++sl) {
      const int j = (t >> 1) + 2 * sl, hh = t & 1;
      uint32_t word = 0;
      for (int h = 0; h < 2; ++h)
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t r = rt * 16 + g + 8 * h;
          const uint32_t G = (kq * 4 + j) * 8 + 4 * hh + q4;
          uint32_t nib = 0x4u;  // (0,1): a valid ordered pattern for padding
          if (group_valid(a, r, G)) {
            if (a.pad14) {
              uint32_t c0, c1;
              pad_pair(r, G, &c0, &c1, &nib);
            } else {
              const uint64_t k0 = (raw.row_begin + r) * row_nnz + 2ull * G;
              nib = offset_at(raw.words, k0) | (offset_at(raw.words, k0 + 1) << 2);
            }
          }
          word |= nib << (16 * h + 4 * q4);
        }
      m[sl] = word;
    }
    uint32_t* mo = reinterpret_cast<uint32_t*>(a.meta + blk * 32 * 8 + lane * 8);
    mo[0] = m[0];
    mo[1] = m[1];
  } else if (f == I4_SP14 || f == F16_SP14) {
    uint32_t v[8] = {0};
    uint32_t ms = 0;
    for (int j = 0; j < 4; ++j)
      for (int h = 0; h < 2; ++h)
        for (int q = 0; q < 2; ++q) {
          const uint32_t r = rt * 16 + g + 8 * h;
          const uint32_t G = (kq * 4 + j) * 8 + t + 4 * q;
          if (!group_valid(a, r, G)) continue;
          const uint64_t k = (raw.row_begin + r) * row_nnz + G;
          const uint32_t off = offset_at(raw.words, k);
          ms |= (off & 1u) << (4 * j + h + 2 * q);
          if (f == I4_SP14) {
            v[j >> 1] |= nibble_at(raw.codes, k) << (4 * (2 * (j & 1) + q) + 16 * h);
          } else {
            v[2 * j + q] |= static_cast<uint32_t>(__half_as_ushort(raw.values[k])) << (16 * h);
          }
        }
    for (int sl = 0; sl < 2; ++sl) {  // high offset bits, metadata-holder order
      const int j = (t >> 1) + 2 * sl, hh = t & 1;
      for (int h = 0; h < 2; ++h)
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t r = rt * 16 + g + 8 * h;
          const uint32_t G = (kq * 4 + j) * 8 + 4 * hh + q4;
          if (!group_valid(a, r, G)) continue;
          const uint64_t k = (raw.row_begin + r) * row_nnz + G;
          ms |= ((offset_at(raw.words, k) >> 1) & 1u) << (16 + 8 * sl + 4 * h + q4);
        }
    }
    const int VB = val_lane_bytes(f);
    uint32_t* vo = reinterpret_cast<uint32_t*>(a.vals + blk * 32 * VB + lane * VB);
    for (int i = 0; i < VB / 4; ++i) vo[i] = v[i];
    *reinterpret_cast<uint32_t*>(a.meta + blk * 32 * 4 + lane * 4) = ms;
  } else {  // I4_DENSE: 8 k16 tiles per k-quad
    uint32_t v[8] = {0};
    for (int w = 0; w < 8; ++w)
      for (int h = 0; h < 2; ++h)
        for (int q = 0; q < 2; ++q) {
          const uint32_t r = rt * 16 + g + 8 * h;
          const uint32_t c = kq * 128 + 16 * w + 2 * t + 8 * q;
          const int p = h + 2 * q;
          if (r >= a.rows || c >= a.cols) continue;
          const uint64_t k = static_cast<uint64_t>(raw.row_begin + r) * a.cols + c;
          v[w] |= static_cast<uint32_t>(raw.dense_codes[k] & 0xF) << (4 * p);
          v[w] |= static_cast<uint32_t>(raw.dense_codes[k + 1] & 0xF) << (16 + 4 * p);
        }
    uint32_t* vo = reinterpret_cast<uint32_t*>(a.vals + blk * 32 * 32 + lane * 32);
    for (int i = 0; i < 8; ++i) vo[i] = v[i];
  }
}

// Per (row tile, k-quad, scale entry, row): the group covering k-tiles
// [e*SS, (e+1)*SS) of the quad, or (SS = 0) columns [16e, 16e + 16).  Group
// boundaries are multiples of 32 columns on the tiled path (16 with SS = 0),
// so an entry never straddles two groups.
__global__ void relayout_scales_kernel(const RelayoutArgs a) {
  const uint64_t total = static_cast<uint64_t>(a.RT) * a.KQ * a.E * 16;
  const uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (idx >= total) return;
  const int slot = static_cast<int>(idx & 15);
  const uint64_t be = idx >> 4;
  const int e = static_cast<int>(be % a.E);
  const uint64_t blk = be / a.E;
  const int kq = static_cast<int>(blk % a.KQ);
  const int rt = static_cast<int>(blk / a.KQ);
  const int g = slot >> 1, h = slot & 1;
  const uint32_t r = rt * 16 + g + 8 * h;
  const uint32_t col = kq * 128 + (a.SS ? e * a.SS * 32 : e * 16);
  float s = 0.f;
  uint8_t z = 0;
  if (r < a.rows && col < a.cols) {
    const uint32_t R = a.raw.row_begin + r;
    const uint64_t gi = static_cast<uint64_t>(a.raw.group_offsets[R]) + col / a.raw.group_sizes[R];
    s = a.raw.scales[gi];
    z = a.raw.zps[gi];
  }
  a.scales[idx] = s;
  a.zps[idx] = z;
}

cudaError_t launch_relayout(const RawStream& raw, int format, uint32_t rows, uint32_t cols,
                            const TiledStream& dst, uint8_t* vals, uint8_t* meta, float* scales,
                            uint8_t* zps, cudaStream_t s) {
  RelayoutArgs a;
  a.raw = raw;
  a.format = format;
  a.rows = rows;
  a.cols = cols;
  a.KQ = dst.KQ;
  a.RT = dst.RT;
  a.SS = dst.SS;
  a.E = dst.E;
  a.vals = vals;
  a.meta = meta;
  a.scales = scales;
  a.zps = zps;
  a.pad14 = dst.pad14;
  const uint64_t total = static_cast<uint64_t>(dst.RT) * dst.KQ * 32;
  relayout_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(a);
  ++launch_counter();
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess || !has_scales(format)) return err;
  const uint64_t tot_s = static_cast<uint64_t>(dst.RT) * dst.KQ * dst.E * 16;
  relayout_scales_kernel<<<static_cast<unsigned>((tot_s + 255) / 256), 256, 0, s>>>(a);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------- general path
// Reference-order stream, one warp per output row, lanes stride over the
// row's kept entries; any group size, any cols % 4 == 0.  Used when the
// group sizes are not multiples of 32 (the tiled path's k-tile).
struct GeneralArgs {
  RawStream raw;
  int kind;  // 0 sparse INT4, 1 sparse FP16, 2 dense INT4
  uint32_t rows, cols;
  int n;
  const float* x;
  int ldx, M;
  float* y;
  int ldy;
};

__global__ void __launch_bounds__(256) general_spmm_kernel(const GeneralArgs a) {
  pdl_wait();  // general path: always dependent; launch the next kernel once the inputs are complete
  pdl_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r = blockIdx.x * 8 + warp;
  if (r >= a.rows) return;
  const uint64_t R = a.raw.row_begin + r;
  const uint64_t row_nnz = a.kind == 2 ? a.cols : static_cast<uint64_t>(a.cols) * a.n / 4;
  const uint32_t gsz = a.kind == 1 ? 1u : a.raw.group_sizes[R];
  const uint32_t gbase = a.kind == 1 ? 0u : a.raw.group_offsets[R];
  for (int m0 = 0; m0 < a.M; m0 += 8) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (uint64_t j = lane; j < row_nnz; j += 32) {
      const uint64_t k = R * row_nnz + j;
      uint32_t col;
      float v;
      if (a.kind == 2) {
        col = static_cast<uint32_t>(j);
        const uint32_t gi = gbase + col / gsz;
        v = decode(a.raw.dense_codes[k], a.raw.zps[gi], a.raw.scales[gi]);
      } else {
        col = static_cast<uint32_t>(j / a.n) * 4 + offset_at(a.raw.words, k);
        if (a.kind == 0) {
          const uint32_t gi = gbase + col / gsz;
          v = decode(nibble_at(a.raw.codes, k), a.raw.zps[gi], a.raw.scales[gi]);
        } else {
          v = __half2float(a.raw.values[k]);
        }
      }
#pragma unroll
      for (int mm = 0; mm < 8; ++mm)
        if (m0 + mm < a.M) acc[mm] = fmaf(v, a.x[static_cast<size_t>(m0 + mm) * a.ldx + col], acc[mm]);
    }
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
      const float s = warp_sum(acc[mm]);
      if (lane == 0 && m0 + mm < a.M) a.y[static_cast<size_t>(m0 + mm) * a.ldy + r] = s;
    }
  }
}

cudaError_t launch_general(const egt_dev_packed* h, const float* x, int ldx, int M, float* y,
                           int ldy, const LaunchCtx& ctx) {
  GeneralArgs a;
  a.raw = h->raw;
  a.kind = h->format == I4_DENSE ? 2 : (h->kind == 0 ? 1 : 0);
  a.rows = h->rows;
  a.cols = h->cols;
  a.n = h->n;
  a.x = x;
  a.ldx = ldx;
  a.M = M;
  a.y = y;
  a.ldy = ldy;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((h->rows + 7) / 8);
  cfg.blockDim = dim3(256);
  cfg.stream = ctx.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  void* args[] = {&a};
  cudaError_t err = cudaLaunchKernelExC(&cfg, reinterpret_cast<void*>(&general_spmm_kernel), args);
  if (err == cudaSuccess) ++launch_counter();
  return err;
}

// ------------------------------------------------------------- grouped stream
// INT4 2:4 in the reference's own stream order with power-of-two group sizes
// >= 16 -- the reference's default fine groups (config.hpp:50-51, g_fine =
// 16) do not fit the tiled path's 32-column k-tiles.  A lane takes chunks of
// 8 kept entries: one u16 index word, one u32 of codes, and (16 columns,
// 16-aligned) exactly one group, so one scale / zero point per chunk:
//   y_r += s_g * sum_j (c_j - z_g) x[col_j]      (c - z exact in f32)
// x (after the fused rmsnorm / silu) is staged once per block in shared
// memory with one pad float per 16 (lane stride 16 floats -> 17: no bank
// conflicts).  Bytes per 8 entries at g16: 4 codes + 2 index + 5 table.
struct GroupedArgs {
  RawStream raw;
  uint32_t rows, cols;
  const float* x;
  int ldx, M;
  float* y;
  int ldy;
  const float* res;
  int ldr, xform, out_silu;
  float eps;
};
// one row per warp, 8 chunks per lane in flight (~45 KB of weights in
// flight per SM at full occupancy: the bandwidth-delay product of HBM)
// (16 rows per block: x staged once per 16 rows; two blocks per SM)
constexpr int kGroupedRowsPerWarp = 1, kGroupedWarps = 16, kGroupedMaxX = 24 * 1024;  // x floats staged

__device__ __forceinline__ int xpad(int c) { return c + (c >> 4); }

template <int M>
__global__ void __launch_bounds__(32 * kGroupedWarps, 2) grouped_stream_kernel(const GroupedArgs a) {
  extern __shared__ float xs[];  // [M][cols + cols / 16]
  pdl_wait();
  pdl_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ldxs = xpad(static_cast<int>(a.cols));
  // ---- stage x (rmsnorm: inv_m over the whole row, model.cpp:57-67)
  __shared__ float s_red[kGroupedWarps][M];
  float inv[M];
#pragma unroll
  for (int m = 0; m < M; ++m) inv[m] = 1.f;
  // x into registers first (float4s, every load of a thread in flight
  // together: x staging is on the critical path of a dependent product),
  // then the row sums (rmsnorm), then the transformed values into smem
  constexpr int kXV = 6;  // float4s per thread per token: cols <= 4 * 512 * 6
  const int n4 = static_cast<int>(a.cols / 4);
  for (int m = 0; m < M; ++m) {
    float4 v[kXV];
    const float4* xr = reinterpret_cast<const float4*>(a.x + static_cast<size_t>(m) * a.ldx);
#pragma unroll
    for (int u = 0; u < kXV; ++u) {
      const int j = static_cast<int>(threadIdx.x) + u * static_cast<int>(blockDim.x);
      v[u] = j < n4 ? __ldg(xr + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float iv = 1.f;
    if (a.xform == EGT_INPUT_RMSNORM) {
      float ss = 0.f;
#pragma unroll
      for (int u = 0; u < kXV; ++u)
        ss = fmaf(v[u].x, v[u].x, fmaf(v[u].y, v[u].y, fmaf(v[u].z, v[u].z, fmaf(v[u].w, v[u].w, ss))));
      ss = warp_sum(ss);
      if (lane == 0) s_red[warp][m] = ss;
      __syncthreads();
      float tot = 0.f;
      for (int w = 0; w < kGroupedWarps; ++w) tot += s_red[w][m];
      iv = 1.0f / sqrtf(tot / static_cast<float>(a.cols) + a.eps);
    }
    inv[m] = iv;
#pragma unroll
    for (int u = 0; u < kXV; ++u) {
      const int j = static_cast<int>(threadIdx.x) + u * static_cast<int>(blockDim.x);
      if (j < n4) {
        float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (a.xform == EGT_INPUT_RMSNORM) e[q] *= iv;
          else if (a.xform == EGT_INPUT_SILU) e[q] = e[q] * (1.0f / (1.0f + expf(-e[q])));  // model.cpp:80-84
        }
        float* dst = xs + m * ldxs + xpad(4 * j);  // 4 j .. 4 j + 3 never straddle a pad (16 | 4 j + 16)
        dst[0] = e[0];
        dst[1] = e[1];
        dst[2] = e[2];
        dst[3] = e[3];
      }
    }
  }
  __syncthreads();
  // ---- rows
  const uint32_t row_nnz = a.cols / 2, nchunk = a.cols / 16;
  for (int i = 0; i < kGroupedRowsPerWarp; ++i) {
    const uint32_t r = (blockIdx.x * kGroupedWarps + warp) * kGroupedRowsPerWarp + i;
    if (r >= a.rows) break;
    const uint64_t R = a.raw.row_begin + r;
    const uint32_t gsz = a.raw.group_sizes[R], gbase = a.raw.group_offsets[R];
    const int lg = gsz >= a.cols ? 31 : __ffs(gsz) - 1;  // one group per row: col >> 31 == 0
    const uint16_t* wr = a.raw.words + R * (row_nnz / 8);
    const uint32_t* cr = reinterpret_cast<const uint32_t*>(a.raw.codes) + R * (row_nnz / 8);
    float acc[M];
#pragma unroll
    for (int m = 0; m < M; ++m) acc[m] = 0.f;
    constexpr int U = 8;  // chunks per lane in flight
    for (uint32_t c0 = lane; c0 < nchunk; c0 += 32 * U) {
      uint32_t w[U], cw[U];
      float s[U];
      uint32_t z[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t c = c0 + 32 * u;
        w[u] = 0u;
        cw[u] = 0u;
        s[u] = 0.f;
        z[u] = 0u;
        if (c < nchunk) {
          w[u] = __ldg(wr + c);
          cw[u] = __ldg(cr + c);
          const uint32_t gi = gbase + ((16 * c) >> lg);
          s[u] = __ldg(a.raw.scales + gi);
          z[u] = __ldg(a.raw.zps + gi);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t c = c0 + 32 * u;
        if (c >= nchunk) break;
        // c - z exactly: 2^23 + c (the code under the exponent of 2^23) minus 2^23 + z
        const float zf = 8388608.0f + static_cast<float>(z[u]);
        // the chunk's 16 columns sit between two pads: xpad(16 c + i) = 17 c + i
        const float* xc = xs + 17 * static_cast<int>(c);
        float part[M];
#pragma unroll
        for (int m = 0; m < M; ++m) part[m] = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = 4 * (j >> 1) + static_cast<int>((w[u] >> (14 - 2 * j)) & 3u);
          const float d = __uint_as_float(0x4B000000u | ((cw[u] >> (4 * j)) & 0xFu)) - zf;
#pragma unroll
          for (int m = 0; m < M; ++m) part[m] = fmaf(d, xc[m * ldxs + col], part[m]);
        }
#pragma unroll
        for (int m = 0; m < M; ++m) acc[m] = fmaf(s[u], part[m], acc[m]);
      }
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const float v = warp_sum(acc[m]);
      if (lane == m) {
        float o = (a.res ? a.res[static_cast<size_t>(m) * a.ldr + r] : 0.f) + v;
        if (a.out_silu) o = o * (1.0f / (1.0f + expf(-o)));  // model.cpp:80-84
        a.y[static_cast<size_t>(m) * a.ldy + r] = o;
      }
    }
  }
}

bool grouped_stream_ok(const egt_dev_packed* h, int M) {
  return h->grouped_ok && M >= 1 && M <= 4 && static_cast<size_t>(M) * (h->cols + h->cols / 16) <= kGroupedMaxX &&
         h->cols <= 4u * 32 * kGroupedWarps * 6;
}

cudaError_t launch_grouped_stream(const egt_dev_packed* h, const float* x, int ldx, int M, float* y, int ldy,
                                  const LaunchCtx& ctx) {
  GroupedArgs a;
  a.raw = h->raw;
  a.rows = h->rows;
  a.cols = h->cols;
  a.x = x;
  a.ldx = ldx;
  a.M = M;
  a.y = y;
  a.ldy = ldy;
  a.res = ctx.res;
  a.ldr = ctx.ldr;
  a.xform = ctx.xform;
  a.out_silu = ctx.out_silu;
  a.eps = ctx.eps;
  void* fn = M == 1 ? reinterpret_cast<void*>(&grouped_stream_kernel<1>)
           : M == 2 ? reinterpret_cast<void*>(&grouped_stream_kernel<2>)
           : M == 3 ? reinterpret_cast<void*>(&grouped_stream_kernel<3>)
                    : reinterpret_cast<void*>(&grouped_stream_kernel<4>);
  const size_t smem = static_cast<size_t>(M) * (h->cols + h->cols / 16) * sizeof(float);
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  const uint32_t rows_per_block = kGroupedWarps * kGroupedRowsPerWarp;
  cfg.gridDim = dim3((h->rows + rows_per_block - 1) / rows_per_block);
  cfg.blockDim = dim3(32 * kGroupedWarps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  void* args[] = {&a};
  err = cudaLaunchKernelExC(&cfg, fn, args);
  if (err == cudaSuccess) ++launch_counter();
  return err;
}

// ------------------------------------------------------------- unpack
// Bit-exact dense reconstruction (unpack, packed.cpp:197-209).
__device__ __forceinline__ void set_mask(uint8_t* mask, uint32_t cols, uint32_t r, uint32_t c) {
  if (!mask) return;
  const uint64_t i = static_cast<uint64_t>(r) * cols + c;
  atomicOr(reinterpret_cast<unsigned int*>(mask) + (i >> 5), 1u << (i & 31));
}

__global__ void dequant_general_kernel(const GeneralArgs a, float* w, uint8_t* mask) {
  const uint64_t row_nnz = a.kind == 2 ? a.cols : static_cast<uint64_t>(a.cols) * a.n / 4;
  const uint64_t total = static_cast<uint64_t>(a.rows) * row_nnz;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(i / row_nnz);
    const uint64_t j = i % row_nnz;
    const uint64_t R = a.raw.row_begin + r;
    const uint64_t k = R * row_nnz + j;
    uint32_t col;
    float v;
    if (a.kind == 2) {
      col = static_cast<uint32_t>(j);
      const uint32_t gi = a.raw.group_offsets[R] + col / a.raw.group_sizes[R];
      v = decode(a.raw.dense_codes[k], a.raw.zps[gi], a.raw.scales[gi]);
    } else {
      col = static_cast<uint32_t>(j / a.n) * 4 + offset_at(a.raw.words, k);
      if (a.kind == 0) {
        const uint32_t gi = a.raw.group_offsets[R] + col / a.raw.group_sizes[R];
        v = decode(nibble_at(a.raw.codes, k), a.raw.zps[gi], a.raw.scales[gi]);
      } else {
        v = __half2float(a.raw.values[k]);
      }
    }
    w[static_cast<uint64_t>(r) * a.cols + col] = v;
    set_mask(mask, a.cols, r, col);
  }
}

struct DequantTiledArgs {
  TiledStream ts;
  int format;
  uint32_t rows, cols;
  float* w;
  uint8_t* mask;
};

__global__ void dequant_tiled_kernel(const DequantTiledArgs a) {
  const uint64_t total = static_cast<uint64_t>(a.ts.RT) * a.ts.KQ * 32;
  const uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (idx >= total) return;
  const int lane = static_cast<int>(idx & 31);
  const uint64_t lblk = idx >> 5;  // block index within this handle
  const int kq = static_cast<int>(lblk % a.ts.KQ);
  const int rt = static_cast<int>(lblk / a.ts.KQ);
  const uint64_t blk = static_cast<uint64_t>(a.ts.rt_begin + rt) * a.ts.KQ + kq;
  const int g = lane >> 2, t = lane & 3;
  const int f = a.format;
  const int VB = val_lane_bytes(f), MB = meta_lane_bytes(f);
  const uint32_t* v = reinterpret_cast<const uint32_t*>(a.ts.vals + blk * 32 * VB + lane * VB);
  const uint32_t* mb = reinterpret_cast<const uint32_t*>(a.ts.meta + blk * 32 * MB);
  auto scale_of = [&](int j, int q, int h, float* s, uint32_t* z) {  // k-tile j, 16-column half q
    const int e = a.ts.SS ? j / a.ts.SS : 2 * j + q;
    const uint64_t si = (blk * a.ts.E + e) * 16 + 2 * g + h;
    *s = a.ts.scales[si];
    *z = a.ts.zps[si];
  };
  if (f == I4_DENSE) {
    for (int w16 = 0; w16 < 8; ++w16)
      for (int h = 0; h < 2; ++h)
        for (int q = 0; q < 2; ++q)
          for (int i = 0; i < 2; ++i) {
            const uint32_t r = rt * 16 + g + 8 * h;
            const uint32_t c = kq * 128 + 16 * w16 + 2 * t + 8 * q + i;
            if (r >= a.rows || c >= a.cols) continue;
            const int p = h + 2 * q;
            const uint32_t code = (v[w16] >> (4 * p + 16 * i)) & 0xFu;
            float s;
            uint32_t z;
            scale_of((16 * w16) / 32, w16 & 1, h, &s, &z);
            a.w[static_cast<uint64_t>(r) * a.cols + c] = decode(code, z, s);
            set_mask(a.mask, a.cols, r, c);
          }
    return;
  }
  const bool two = (f == I4_SP24 || f == F16_SP24);
  for (int j = 0; j < 4; ++j)
    for (int h = 0; h < 2; ++h)
      for (int q = 0; q < 2; ++q) {
        const uint32_t r = rt * 16 + g + 8 * h;
        const uint32_t G = (kq * 4 + j) * 8 + t + 4 * q;
        if (r >= a.rows || G * 4 >= a.cols) continue;
        // metadata of (row g+8h, group t+4q of k-tile j) lives in lane
        // 4g + 2(j&1) + q, nibble 4h + t (see relayout_kernel)
        const int holder = 4 * g + 2 * (j & 1) + q;
        if (two) {
          const uint32_t word = mb[holder * 2 + (j >> 1)];
          const uint32_t nib = (word >> (16 * h + 4 * t)) & 0xFu;
          const uint32_t off[2] = {nib & 3u, (nib >> 2) & 3u};
          // pad14: only the kept entry of the pair (the second one iff (1, 3))
          const int only = a.ts.pad14 ? ((off[0] == 1u && off[1] == 3u) ? 1 : 0) : -1;
          for (int i = 0; i < 2; ++i) {
            if (only >= 0 && i != only) continue;
            const uint32_t c = G * 4 + off[i];
            float val;
            if (f == I4_SP24) {
              const int p = h + 2 * q;
              const uint32_t code = (v[j] >> (4 * p + 16 * i)) & 0xFu;
              float s;
              uint32_t z;
              scale_of(j, q, h, &s, &z);
              val = decode(code, z, s);
            } else {
              const uint32_t pair = v[4 * j + h + 2 * q];
              val = __half2float(__ushort_as_half(static_cast<unsigned short>(pair >> (16 * i))));
            }
            a.w[static_cast<uint64_t>(r) * a.cols + c] = val;
            set_mask(a.mask, a.cols, r, c);
          }
        } else {
          const uint32_t own = mb[lane];
          const uint32_t slot = (own >> (4 * j + h + 2 * q)) & 1u;
          const uint32_t hword = mb[holder];
          const uint32_t hi = (hword >> (16 + 8 * (j >> 1) + 4 * h + t)) & 1u;
          const uint32_t c = G * 4 + (hi << 1 | slot);
          float val;
          if (f == I4_SP14) {
            const uint32_t code = (v[j >> 1] >> (4 * (2 * (j & 1) + q) + 16 * h)) & 0xFu;
            float s;
            uint32_t z;
            scale_of(j, q, h, &s, &z);
            val = decode(code, z, s);
          } else {
            val = __half2float(__ushort_as_half(static_cast<unsigned short>(v[2 * j + q] >> (16 * h))));
          }
          a.w[static_cast<uint64_t>(r) * a.cols + c] = val;
          set_mask(a.mask, a.cols, r, c);
        }
      }
}

cudaError_t launch_dequant(const egt_dev_packed* h, float* w, uint8_t* mask, cudaStream_t s) {
  if (h->path == 0) {
    DequantTiledArgs a;
    a.ts = h->tiled;
    a.format = h->format;
    a.rows = h->rows;
    a.cols = h->cols;
    a.w = w;
    a.mask = mask;
    const uint64_t total = static_cast<uint64_t>(h->tiled.RT) * h->tiled.KQ * 32;
    if (total == 0) return cudaSuccess;
    dequant_tiled_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(a);
  } else {
    GeneralArgs a;
    a.raw = h->raw;
    a.kind = h->format == I4_DENSE ? 2 : (h->kind == 0 ? 1 : 0);
    a.rows = h->rows;
    a.cols = h->cols;
    a.n = h->n;
    dequant_general_kernel<<<1184, 256, 0, s>>>(a, w, mask);
  }
  ++launch_counter();
  return cudaGetLastError();
}

}  // namespace egt_impl

namespace egt_impl {
// Sparse-FP upload: the reference keeps f32 values (packed.hpp:33
// kFloat32); the device stores fp16.  Values that fp16 cannot hold exactly
// (precision or range) set err bit 8 unless rounding was requested.
__global__ void f32_to_f16_kernel(const float* src, __half* dst, uint64_t n, int check, uint32_t* err) {
  bool bad = false;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float v = src[i];
    const __half h = __float2half_rn(v);
    dst[i] = h;
    if (check && __half2float(h) != v && v == v) bad = true;  // NaN stays NaN
  }
  if (check && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 8u);
}

cudaError_t launch_f32_to_f16(const float* src, __half* dst, uint64_t n, bool check, uint32_t* err,
                              cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  f32_to_f16_kernel<<<1184, 256, 0, s>>>(src, dst, n, check ? 1 : 0, err);
  ++launch_counter();
  return cudaGetLastError();
}
}  // namespace egt_impl

// ------------------------------------------------------------- dense FP32
// y = W x for a dense row-major f32 W: the mixed dispatch's (dense, !quant)
// baseline arm (compress.cpp:395-414 materialises it) and bench_spmv's
// "dense-fp" variant (packed.cpp:337-347).  Warp per row, float4 loads,
// HBM-bound (4 B per weight).
namespace egt_impl {
namespace {
__global__ void __launch_bounds__(256) gemv_f32_kernel(const float* __restrict__ w, const float* __restrict__ x,
                                                       float* __restrict__ y, uint32_t rows, uint32_t cols) {
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* wr = w + static_cast<size_t>(r) * cols;
  float acc = 0.f;
  if ((cols & 3u) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const float4* w4 = reinterpret_cast<const float4*>(wr);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (uint32_t c = lane; c < cols / 4; c += 32) {
      const float4 a = __ldcs(w4 + c), b = x4[c];
      acc = fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, acc))));
    }
  } else {
    for (uint32_t c = lane; c < cols; c += 32) acc = fmaf(wr[c], x[c], acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) y[r] = acc;
}
}  // namespace

cudaError_t launch_gemv_f32(const float* w, const float* x, float* y, uint32_t rows, uint32_t cols, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  gemv_f32_kernel<<<(rows + 7) / 8, 256, 0, s>>>(w, x, y, rows, cols);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++launch_counter();
  return e;
}
}  // namespace egt_impl
