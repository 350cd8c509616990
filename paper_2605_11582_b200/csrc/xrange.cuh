// Full f32 range for the fp16 hi/lo activation split (every tensor-core
// product kernel).
//
// The reference's spmv (packed.cpp:211-220) is f32 for any x.  The product
// kernels feed x to the tensor cores as fp16 hi + fp16 lo (x - hi), which on
// its own overflows for |x| >= 65520 and loses relative precision below the
// fp16 normal range (2^-14).  So every staging window (the x slice one CTA
// multiplies, per token) is first scaled by a power of two 2^e that maps its
// largest finite |x| into [2^14, 2^15): the split is then exact to ~22 bits
// for every value within 2^17 of the window maximum, never overflows, and
// the f32 partial sum is multiplied by 2^-e exactly.
//
// Non-finite x (inf / NaN) enter the tensor-core sum as 0 and are added back
// per output row in the epilogue, in f32, for exactly the kept entries of
// that row (v * x, the reference's term): rows reach inf / NaN exactly where
// the reference's left-to-right sum does (a kept zero-valued entry times inf
// is NaN, opposite infinities are NaN, unkept columns contribute nothing).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "tiled_format.h"

namespace egt_dev {

// running finite max |x| (as ordered u32 bits) and a non-finite flag
__device__ __forceinline__ void xr_note(uint32_t& mx, uint32_t& nf, float v) {
  const uint32_t b = __float_as_uint(v) & 0x7fffffffu;
  if (b >= 0x7f800000u)
    nf = 1u;
  else
    mx = max(mx, b);
}

// warp-reduce, then one shared atomic per warp (s_mx / s_nf zeroed before)
__device__ __forceinline__ void xr_commit(uint32_t mx, uint32_t nf, uint32_t* s_mx, uint32_t* s_nf) {
  mx = __reduce_max_sync(0xffffffffu, mx);
  nf = __reduce_or_sync(0xffffffffu, nf);
  if ((threadIdx.x & 31) == 0) {
    if (mx) atomicMax(s_mx, mx);
    if (nf) atomicOr(s_nf, 1u);
  }
}

// e such that max|x| * 2^e lies in [2^14, 2^15) (0 for an all-zero window)
__device__ __forceinline__ int xr_exp(uint32_t mx_bits) {
  if (mx_bits == 0u) return 0;
  int E = static_cast<int>(mx_bits >> 23) - 127;               // floor(log2) of a normal
  if (mx_bits < 0x00800000u) E = (31 - __clz(mx_bits)) - 149;  // subnormal
  return min(126, max(-126, 14 - E));
}

// 2^e for -126 <= e <= 127, exactly
__device__ __forceinline__ float xr_pow2(int e) { return __uint_as_float(static_cast<uint32_t>(e + 127) << 23); }

// x * 2^e with non-finite values replaced by 0 (they are added back exactly
// by the epilogue fix-up)
__device__ __forceinline__ float xr_scaled(float v, float s) {
  const float r = v * s;
  return (__float_as_uint(v) & 0x7fffffffu) >= 0x7f800000u ? 0.f : r;
}

__device__ __forceinline__ float xr_decode(uint32_t code, uint32_t zp, float scale) {
  return __fmul_rn(__fsub_rn(static_cast<float>(code), static_cast<float>(zp)), scale);
}

// One fragment-tiled matrix (tiled_format.h) for the element lookup below.
struct TiledRef {
  const uint8_t* vals;
  const uint8_t* meta;
  const float* scales;
  const uint8_t* zps;
  int KQ, rt_begin, SS, pad14;
};

// Is W[r][c] kept, and its value (bit-exact with unpack, packed.cpp:197-209).
// Mirrors the fragment layout dequant_tiled_kernel walks lane by lane.
template <int FMT>
__device__ bool tiled_value(const TiledRef& m, int r, int c, float* out) {
  using namespace egt_fmt;
  constexpr int VB = val_lane_bytes(FMT), MB = meta_lane_bytes(FMT);
  const int r16 = r & 15, g = r16 & 7, h = r16 >> 3;
  const int cin = c & 127, j = cin >> 5, gi = (cin & 31) >> 2, t = gi & 3, q = gi >> 2;
  const size_t blk = static_cast<size_t>(m.rt_begin + (r >> 4)) * m.KQ + (c >> 7);
  const int E = ss_entries(m.SS);
  auto vword = [&](int lane, int idx) {
    return reinterpret_cast<const uint32_t*>(m.vals + blk * 32 * VB + lane * VB)[idx];
  };
  auto scaled = [&](uint32_t code, int jj) {  // jj: the k-tile (32 columns) of c within the quad
    const size_t si = (blk * E + (m.SS ? jj / m.SS : ss_entry(0, cin))) * 16 + 2 * g + h;
    return xr_decode(code, m.zps[si], m.scales[si]);
  };
  if constexpr (FMT == I4_DENSE) {
    const int w16 = cin >> 4, rem = cin & 15, qq = rem >> 3, tt = (rem & 7) >> 1, i = rem & 1;
    const uint32_t code = (vword(4 * g + tt, w16) >> (4 * (h + 2 * qq) + 16 * i)) & 0xFu;
    *out = scaled(code, w16 >> 1);
    return true;
  } else {
    const uint32_t* mb = reinterpret_cast<const uint32_t*>(m.meta + blk * 32 * MB);
    const int holder = 4 * g + 2 * (j & 1) + q, lane = 4 * g + t;
    const int o = c & 3;
    if constexpr (FMT == I4_SP24 || FMT == F16_SP24) {
      const uint32_t nib = (mb[holder * 2 + (j >> 1)] >> (16 * h + 4 * t)) & 0xFu;
      const int o0 = static_cast<int>(nib & 3u), o1 = static_cast<int>((nib >> 2) & 3u);
      const int i = o == o0 ? 0 : (o == o1 ? 1 : -1);
      if (i < 0) return false;
      if (m.pad14 && i != ((o0 == 1 && o1 == 3) ? 1 : 0)) return false;  // the zero-valued 1:4 partner
      if constexpr (FMT == I4_SP24) {
        *out = scaled((vword(lane, j) >> (4 * (h + 2 * q) + 16 * i)) & 0xFu, j);
      } else {
        const uint32_t pair = vword(lane, 4 * j + h + 2 * q);
        *out = __half2float(__ushort_as_half(static_cast<unsigned short>(pair >> (16 * i))));
      }
      return true;
    } else {  // native 1:4 (I4_SP14 / F16_SP14)
      const uint32_t slot = (mb[lane] >> (4 * j + h + 2 * q)) & 1u;
      const uint32_t hi = (mb[holder] >> (16 + 8 * (j >> 1) + 4 * h + t)) & 1u;
      if (static_cast<int>(hi << 1 | slot) != o) return false;
      if constexpr (FMT == I4_SP14) {
        *out = scaled((vword(lane, j >> 1) >> (4 * (2 * (j & 1) + q) + 16 * h)) & 0xFu, j);
      } else {
        *out = __half2float(__ushort_as_half(static_cast<unsigned short>(vword(lane, 2 * j + q) >> (16 * h))));
      }
      return true;
    }
  }
}

}  // namespace egt_dev
