// Per-unit compute of the tensor-core SparseGemv over the fragment-tiled
// stream (tiled_format.h), shared by the per-launch kernel (spmm_tiled.cu)
// and the persistent multi-GEMV program kernel (program.cu).  A "unit" is one
// k-quad block (16 rows x 128 columns) as one warp consumes it from a
// shared-memory stage.
#pragma once
#include "device_common.cuh"
#include "tiled_format.h"

namespace egt_impl {
using namespace egt_dev;
using namespace egt_fmt;

template <int FMT, int E>
struct Unit {
  static constexpr int NV = val_lane_bytes(FMT) / 4;
  static constexpr int NM = meta_lane_bytes(FMT) > 0 ? meta_lane_bytes(FMT) / 4 : 1;
  // 16-column groups (E = 8): the scales / zero points stay in shared memory
  // and are read per k-tile (24 more registers per unit would spill)
  static constexpr int NS = has_scales(FMT) && E <= 4 ? E : 1;
  uint32_t v[NV];
  uint32_t m[NM];
  uint32_t s[2 * NS];
  uint32_t z[NS];
  uint32_t sca, zpa;  // E = 8: shared-memory addresses of this lane's rows' entries
};

// A stage in shared memory holds one row tile's blocks for the CTA's KCs
// k-quads, copied verbatim from HBM by the bulk-copy engine:
//   [vals: KCs x 32 lanes x VB][meta: KCs x 32 x MB][scales: KCs x E x 16 f32][zps: KCs x E x 16 u8]
// Shared-memory read cursor over one stage: a lane's A-operand bits, its
// metadata, and its rows' scale / zero-point entries for the current unit,
// plus its B-fragment slot.  Advancing by n units is five additions.
struct Cursor {
  const uint8_t* v;
  const uint8_t* m;
  const uint8_t* sc;
  const uint8_t* zp;
  const uint32_t* b;
};

template <int FMT, int E>
__device__ __forceinline__ Cursor make_cursor(const uint8_t* st, int CHc, int kql, int lane,
                                              const uint32_t* sB, int kt0, int LS) {
  constexpr int VB = val_lane_bytes(FMT), MB = meta_lane_bytes(FMT);
  const int g = lane >> 2;
  Cursor c;
  c.v = st + (kql * 32 + lane) * VB;
  c.m = st + CHc * 32 * VB + (kql * 32 + lane) * MB;
  const uint8_t* sp = st + CHc * 32 * (VB + MB);
  c.sc = sp + kql * E * 64 + 8 * g;
  c.zp = sp + CHc * E * 64 + kql * E * 16 + 2 * g;
  c.b = sB + (kt0 * LS + (lane < LS ? lane : (lane & 7))) * 4;
  return c;
}

template <int FMT, int E>
__device__ __forceinline__ void advance(Cursor& c, int n, int LS) {
  c.v += n * 32 * val_lane_bytes(FMT);
  c.m += n * 32 * meta_lane_bytes(FMT);
  c.sc += n * E * 64;
  c.zp += n * E * 16;
  c.b += n * 4 * LS * 4;
}

template <int FMT, int E>
__device__ __forceinline__ void lds_unit(Unit<FMT, E>& u, const Cursor& c) {
  constexpr int VB = val_lane_bytes(FMT), MB = meta_lane_bytes(FMT);
  if constexpr (VB == 8) {
    const uint2 t = *reinterpret_cast<const uint2*>(c.v);
    u.v[0] = t.x;
    u.v[1] = t.y;
  } else {
#pragma unroll
    for (int i = 0; i < VB / 16; ++i) {
      const uint4 t = *reinterpret_cast<const uint4*>(c.v + 16 * i);
      u.v[4 * i + 0] = t.x;
      u.v[4 * i + 1] = t.y;
      u.v[4 * i + 2] = t.z;
      u.v[4 * i + 3] = t.w;
    }
  }
  if constexpr (MB == 8) {
    const uint2 t = *reinterpret_cast<const uint2*>(c.m);
    u.m[0] = t.x;
    u.m[1] = t.y;
  } else if constexpr (MB == 4) {
    u.m[0] = *reinterpret_cast<const uint32_t*>(c.m);
  } else {
    u.m[0] = 0;
  }
  if constexpr (has_scales(FMT) && E == 8) {
    u.sca = smem_u32(c.sc);
    u.zpa = smem_u32(c.zp);
  } else if constexpr (has_scales(FMT)) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint2 sc = *reinterpret_cast<const uint2*>(c.sc + e * 64);
      u.s[2 * e] = sc.x;
      u.s[2 * e + 1] = sc.y;
      u.z[e] = *reinterpret_cast<const uint16_t*>(c.zp + e * 16);
    }
  }
}

// Bit q of the 8-bit plane -> bit 4q.
__device__ __forceinline__ uint32_t spread4(uint32_t p) {
  uint32_t x = p & 0xFFu;
  x = (x | (x << 12)) & 0x000F000Fu;
  x = (x | (x << 6)) & 0x03030303u;
  x = (x | (x << 3)) & 0x11111111u;
  return x;
}

// 1:4 placement: the kept value (low or high half of r) goes to slot 0 or 1
// of the 2:4 pair whose metadata is (0,1) or (2,3); the partner is zero.
__device__ __forceinline__ uint32_t place_lo(uint32_t r, uint32_t slot) {
  return prmt(r, 0u, slot ? 0x1044u : 0x4410u);
}
__device__ __forceinline__ uint32_t place_hi(uint32_t r, uint32_t slot) {
  return prmt(r, 0u, slot ? 0x3244u : 0x4432u);
}

// B fragments of k-tile kt for every n-tile.  D column n only depends on B
// column n, so lanes whose column holds no token (lane >= LS) may read any
// valid slot: they load lane & 7's without predication and their output
// columns are never used.
template <int NT>
__device__ __forceinline__ void load_b(uint32_t (&b)[NT][4], const uint32_t* pb, int nt_stride) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const uint4 t = *reinterpret_cast<const uint4*>(pb + nt * nt_stride);
    b[nt][0] = t.x;
    b[nt][1] = t.y;
    b[nt][2] = t.z;
    b[nt][3] = t.w;
  }
}

// j is a compile-time constant after unrolling; the branch folds away.
template <int NT>
__device__ __forceinline__ void mma_sp_sel(int j, float (&d)[NT][4], const uint32_t (&a)[4],
                                           const uint32_t (&b)[NT][4], uint32_t ev) {
  if (j & 1) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) mma_sp_16832<1>(d[nt], a, b[nt], ev);
  } else {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) mma_sp_16832<0>(d[nt], a, b[nt], ev);
  }
}

// INT4 dequantisation on the tensor core.  The nibble c itself is the A
// operand: an fp16 subnormal c * 2^-24 is exact and needs a single LOP3 per
// pair (no exponent magic, no subtraction).  Row g+8's nibbles sit 4 bits
// higher (16c * 2^-24), so one shift per k-tile feeds all four A registers;
// the x16 is folded into row g+8's scale.  The zero point is applied after
// the fact: a second mma with A = 1.0 under the same sparsity metadata yields
// the sum of the kept x, and per scale step
//   y_r += s_r * (2^24 * D_c - zp_r * D_1)      (2^20 for row g+8).
constexpr float kTwo24 = 16777216.f;
constexpr float kTwo20 = 1048576.f;
constexpr uint32_t kOnes = 0x3C003C00u;  // half2(1, 1)

// NR units of the same k-quad (NR row tiles) share every B fragment load.
template <int FMT, int SS, int NT, int NR, bool kLoadB = true, bool kOnesMma = true>
__device__ __forceinline__ void compute_units(const Unit<FMT, ss_entries(SS)> (&uu)[NR], const uint32_t* pb, int KTc,
                                              int LS, float (&acc)[NR][NT][2]) {
  if constexpr (SS == 0) {
    // 16-column groups (INT4 2:4): per k-tile two mma.sp, the first half's A
    // registers (a0, a1: logical columns 0-15) with its zero points and the
    // second half's (a2, a3: columns 16-31) with theirs, the other half zero
    // (the metadata stays valid); each half's sum times its own scale.
    static_assert(FMT == I4_SP24, "16-column groups: INT4 2:4 only");
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t b[NT][4];
      load_b<NT>(b, pb + j * LS * 4, KTc * LS * 4);
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const Unit<FMT, 8>& u = uu[r];
        float dA[NT][4], dB[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) dA[nt][i] = dB[nt][i] = 0.f;
        uint32_t z0, z1;  // zero points of rows g (low byte) and g + 8, entries 2j and 2j + 1
        asm volatile("ld.shared.u16 %0, [%1];\n" : "=r"(z0) : "r"(u.zpa + 32 * j));
        asm volatile("ld.shared.u16 %0, [%1];\n" : "=r"(z1) : "r"(u.zpa + 32 * j + 16));
        const uint32_t zA0 = (0x6400u | (z0 & 0xFFu)) * 0x10001u, zA80 = (0x6400u | ((z0 >> 4) & 0xF0u)) * 0x10001u;
        const uint32_t zA1 = (0x6400u | (z1 & 0xFFu)) * 0x10001u, zA81 = (0x6400u | ((z1 >> 4) & 0xF0u)) * 0x10001u;
        const uint32_t w = u.v[j], w8 = w >> 8;
        const uint32_t aA[4] = {hsub2_u32(nib2_magic(w), zA0), hsub2_u32(nib16_magic(w), zA80), 0u, 0u};
        const uint32_t aB[4] = {0u, 0u, hsub2_u32(nib2_magic(w8), zA1), hsub2_u32(nib16_magic(w8), zA81)};
        mma_sp_sel<NT>(j, dA, aA, b, u.m[j >> 1]);
        mma_sp_sel<NT>(j, dB, aB, b, u.m[j >> 1]);
        float s0, s08, s1, s18;  // scales of rows g, g + 8 for entries 2j, 2j + 1
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(s0), "=f"(s08) : "r"(u.sca + 128 * j));
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(s1), "=f"(s18) : "r"(u.sca + 128 * j + 64));
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[r][nt][0] = fmaf(s0, dA[nt][0] + dA[nt][1], fmaf(s1, dB[nt][0] + dB[nt][1], acc[r][nt][0]));
          acc[r][nt][1] = fmaf(s08 * 0.0625f, dA[nt][2] + dA[nt][3],
                               fmaf(s18 * 0.0625f, dB[nt][2] + dB[nt][3], acc[r][nt][1]));
        }
      }
    }
  } else {
  // INT4 2:4 and dense: the zero point is subtracted in the A operand.  A
  // nibble under the fp16 exponent 0x64 is exactly 1024 + c (row g) or
  // 1024 + 16c (row g+8, 4 bits higher); HSUB2 with 1024 + z (1024 + 16z)
  // leaves c - z (16(c - z)), exact in fp16, so one mma per k-tile suffices.
  // (kOnesMma = false falls back to the subnormal-nibble path whose zero point
  // comes from a second mma over A = 1.0.)
  constexpr bool kZpInA = (FMT == I4_SP24 || FMT == I4_DENSE) && kOnesMma;
  constexpr bool kOnesTrick = (FMT == I4_SP24 || FMT == I4_DENSE) && !kZpInA;
  // B fragments: lanes whose column holds no token (lane >= LS) read lane&7's
  // slot unpredicated -- D column n only depends on B column n, and the
  // columns of absent tokens are never used (make_cursor).
  float dd[NR][NT][4];
  float dd1[NR][NT][4];
  uint32_t zpairs[NR], zAs[NR], zA8s[NR];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int e = j / SS;
    if (j % SS == 0) {
#pragma unroll
      for (int r = 0; r < NR; ++r) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dd[r][nt][0] = dd[r][nt][1] = dd[r][nt][2] = dd[r][nt][3] = 0.f;
          dd1[r][nt][0] = dd1[r][nt][1] = dd1[r][nt][2] = dd1[r][nt][3] = 0.f;
        }
        if constexpr (FMT == I4_SP14) {
          const uint32_t z0 = uu[r].z[e] & 0xFFu, z1 = (uu[r].z[e] >> 8) & 0xFFu;
          zpairs[r] = zp_magic(z0, z1);
        }
        if constexpr (kZpInA) {
          zAs[r] = (0x6400u | (uu[r].z[e] & 0xFFu)) * 0x10001u;
          zA8s[r] = (0x6400u | ((uu[r].z[e] >> 4) & 0xF0u)) * 0x10001u;
        }
      }
    }
    uint32_t b[NT][4];
    if constexpr (kLoadB) {
      load_b<NT>(b, pb + j * LS * 4, KTc * LS * 4);
    } else {  // tuning experiment: B from registers (results are garbage)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt][0] = b[nt][1] = b[nt][2] = b[nt][3] = uu[0].m[0] ^ j;
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
    const Unit<FMT, ss_entries(SS)>& u = uu[r];
    float (&d)[NT][4] = dd[r];
    float (&d1)[NT][4] = dd1[r];
    const uint32_t zpair = zpairs[r], zA = zAs[r], zA8 = zA8s[r];
    (void)zpair;
    (void)zA;
    (void)zA8;
    (void)d1;
    if constexpr (FMT == I4_SP24 && kZpInA) {
      const uint32_t w = u.v[j], w8 = w >> 8;
      const uint32_t a[4] = {hsub2_u32(nib2_magic(w), zA), hsub2_u32(nib16_magic(w), zA8),
                             hsub2_u32(nib2_magic(w8), zA), hsub2_u32(nib16_magic(w8), zA8)};
      mma_sp_sel<NT>(j, d, a, b, u.m[j >> 1]);
    } else if constexpr (FMT == I4_SP24) {
      const uint32_t w = u.v[j], w8 = w >> 8;
      const uint32_t a[4] = {w & 0x000F000Fu, w & 0x00F000F0u, w8 & 0x000F000Fu, w8 & 0x00F000F0u};
      const uint32_t ones[4] = {kOnes, kOnes, kOnes, kOnes};
      mma_sp_sel<NT>(j, d, a, b, u.m[j >> 1]);
      if constexpr (kOnesMma) mma_sp_sel<NT>(j, d1, ones, b, u.m[j >> 1]);
    } else if constexpr (FMT == F16_SP24) {
      const uint32_t a[4] = {u.v[4 * j + 0], u.v[4 * j + 1], u.v[4 * j + 2], u.v[4 * j + 3]};
      mma_sp_sel<NT>(j, d, a, b, u.m[j >> 1]);
    } else if constexpr (FMT == I4_SP14 || FMT == F16_SP14) {
      uint32_t r0, r1;
      if constexpr (FMT == I4_SP14) {
        const uint32_t w = u.v[j >> 1] >> (8 * (j & 1));
        r0 = hsub2_u32(nib2_magic(w), zpair);
        r1 = hsub2_u32(nib2_magic(w >> 4), zpair);
      } else {
        r0 = u.v[2 * j];
        r1 = u.v[2 * j + 1];
      }
      const uint32_t sl = (u.m[0] >> (4 * j)) & 0xFu;
      uint32_t a[4];
      a[0] = place_lo(r0, sl & 1u);
      a[1] = place_hi(r0, sl & 2u);
      a[2] = place_lo(r1, sl & 4u);
      a[3] = place_hi(r1, sl & 8u);
      const uint32_t plane = (u.m[0] >> (16 + 8 * (j >> 1))) & 0xFFu;
      mma_sp_sel<NT>(j, d, a, b, 0x44444444u | (spread4(plane) * 0xAu));
    } else if constexpr (kZpInA) {  // I4_DENSE: two m16n8k16 per 32-column k-tile
      const uint32_t w0 = u.v[2 * j], w1 = u.v[2 * j + 1], w08 = w0 >> 8, w18 = w1 >> 8;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        mma_16816(d[nt], hsub2_u32(nib2_magic(w0), zA), hsub2_u32(nib16_magic(w0), zA8),
                  hsub2_u32(nib2_magic(w08), zA), hsub2_u32(nib16_magic(w08), zA8), b[nt][0], b[nt][1]);
        mma_16816(d[nt], hsub2_u32(nib2_magic(w1), zA), hsub2_u32(nib16_magic(w1), zA8),
                  hsub2_u32(nib2_magic(w18), zA), hsub2_u32(nib16_magic(w18), zA8), b[nt][2], b[nt][3]);
      }
    } else {  // I4_DENSE: two m16n8k16 per 32-column k-tile
      const uint32_t w0 = u.v[2 * j], w1 = u.v[2 * j + 1], w08 = w0 >> 8, w18 = w1 >> 8;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        mma_16816(d[nt], w0 & 0x000F000Fu, w0 & 0x00F000F0u, w08 & 0x000F000Fu, w08 & 0x00F000F0u, b[nt][0],
                  b[nt][1]);
        mma_16816(d[nt], w1 & 0x000F000Fu, w1 & 0x00F000F0u, w18 & 0x000F000Fu, w18 & 0x00F000F0u, b[nt][2],
                  b[nt][3]);
        mma_16816(d1[nt], kOnes, kOnes, kOnes, kOnes, b[nt][0], b[nt][1]);
        mma_16816(d1[nt], kOnes, kOnes, kOnes, kOnes, b[nt][2], b[nt][3]);
      }
    }
    }  // r (mma)
    if (j % SS == SS - 1) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
    const Unit<FMT, ss_entries(SS)>& u = uu[r];
    float (&d)[NT][4] = dd[r];
    float (&d1)[NT][4] = dd1[r];
    (void)d1;
      if constexpr (kZpInA) {
        const float sg = __uint_as_float(u.s[2 * e]), sg8 = __uint_as_float(u.s[2 * e + 1]) * 0.0625f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[r][nt][0] = fmaf(sg, d[nt][0] + d[nt][1], acc[r][nt][0]);
          acc[r][nt][1] = fmaf(sg8, d[nt][2] + d[nt][3], acc[r][nt][1]);
        }
      } else if constexpr (kOnesTrick) {
        const float sg = __uint_as_float(u.s[2 * e]), sg8 = __uint_as_float(u.s[2 * e + 1]);
        const float cg = sg * kTwo24, cg8 = sg8 * kTwo20;
        const float ng = -sg * static_cast<float>(u.z[e] & 0xFFu);
        const float ng8 = -sg8 * static_cast<float>((u.z[e] >> 8) & 0xFFu);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[r][nt][0] = fmaf(cg, d[nt][0] + d[nt][1], fmaf(ng, d1[nt][0] + d1[nt][1], acc[r][nt][0]));
          acc[r][nt][1] = fmaf(cg8, d[nt][2] + d[nt][3], fmaf(ng8, d1[nt][2] + d1[nt][3], acc[r][nt][1]));
        }
      } else if constexpr (has_scales(FMT)) {
        const float sg = __uint_as_float(u.s[2 * e]), sg8 = __uint_as_float(u.s[2 * e + 1]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[r][nt][0] = fmaf(sg, d[nt][0] + d[nt][1], acc[r][nt][0]);
          acc[r][nt][1] = fmaf(sg8, d[nt][2] + d[nt][3], acc[r][nt][1]);
        }
      } else {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[r][nt][0] += d[nt][0] + d[nt][1];
          acc[r][nt][1] += d[nt][2] + d[nt][3];
        }
      }
    }  // r (scale)
    }
  }
  }  // SS != 0
}

template <int FMT, int SS, int NT, bool kLoadB = true, bool kOnesMma = true>
__device__ __forceinline__ void compute_unit(const Unit<FMT, ss_entries(SS)>& u, const uint32_t* pb, int KTc,
                                             int LS, float (&acc)[NT][2]) {
  const Unit<FMT, ss_entries(SS)> uu[1] = {u};
  float (&a1)[1][NT][2] = *reinterpret_cast<float (*)[1][NT][2]>(&acc);
  compute_units<FMT, SS, NT, 1, kLoadB, kOnesMma>(uu, pb, KTc, LS, a1);
}

template <int FMT>
__host__ __device__ constexpr int stage_bytes(int KCs, int E) {
  return KCs * 32 * (val_lane_bytes(FMT) + meta_lane_bytes(FMT)) + (has_scales(FMT) ? KCs * E * 80 : 0);
}

}  // namespace egt_impl
