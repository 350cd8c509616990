// Tensor-core SparseGemv / skinny SpGEMM over the fragment-tiled stream.
//
// Y[M x rows] = X[M x cols] * W^T for W in INT4 2bit-CSR (2:4, 1:4), dense
// INT4, or sparse-FP16 2bit-CSR.  Replaces the reference's scalar
// spmv (packed.cpp:211-220 via for_each_nonzero :169-184 and packed_value
// :186-193) and quant_dense_gemv (packed.cpp:266-281).
//
// Why tensor cores at batch 1: the path is HBM-bound only if the per-nonzero
// work stays under ~4.6 issue slots (148 SMs x 4 schedulers x ~1.9 GHz vs
// 8.4 M nonzeros in ~1.07 us for a 4096^2 2:4 layer).  A CUDA-core gather
// (shift/mask the 2-bit offset, address, LDS x, dequant, FFMA) costs ~5-7.
// mma.sp consumes the 2-bit offsets natively as sparse metadata, so the
// gather is done by the tensor core; per 8 nonzeros a lane spends 3 SHF +
// 4 LOP3 (nibble -> fp16 via the 0x6400 exponent) + 4 HSUB2 (zero point) +
// 1 mma.sp.  x is split into fp16 hi + lo parts placed in B columns 2m and
// 2m+1, so products are exact and the sum keeps ~22 mantissa bits; the
// per-group f32 scale is applied to the f32 accumulator, as in
// y = sum_g s_g * sum_k (c_k - z_g) x_k.
#include "device_common.cuh"
#include "handle.h"

#include <algorithm>
#include <cmath>

namespace egt_impl {
using namespace egt_dev;
using namespace egt_fmt;

struct TiledArgs {
  const uint8_t* vals;
  const uint8_t* meta;
  const float* scales;
  const uint8_t* zps;
  int KQ, rt_begin, RT, rows, cols;
  const float* x;
  int ldx, M;
  float* y;
  int ldy;
  float* partial;
  uint32_t* counters;
  int RB, WK, KC, S;
};

template <int FMT, int E>
struct Unit {
  static constexpr int NV = val_lane_bytes(FMT) / 4;
  static constexpr int NM = meta_lane_bytes(FMT) > 0 ? meta_lane_bytes(FMT) / 4 : 1;
  static constexpr int NS = has_scales(FMT) ? E : 1;
  uint32_t v[NV];
  uint32_t m[NM];
  uint32_t s[2 * NS];
  uint32_t z[NS];
};

template <int FMT, int E>
__device__ __forceinline__ void load_unit(Unit<FMT, E>& u, const TiledArgs& a, int rt_abs, int kq,
                                          int lane, uint64_t pol) {
  constexpr int VB = val_lane_bytes(FMT), MB = meta_lane_bytes(FMT);
  const size_t blk = static_cast<size_t>(rt_abs) * a.KQ + kq;
  const uint8_t* vp = a.vals + blk * 32 * VB + lane * VB;
  if constexpr (VB == 8) {
    uint2 t = ldg_stream_v2(vp, pol);
    u.v[0] = t.x;
    u.v[1] = t.y;
  } else {
#pragma unroll
    for (int i = 0; i < VB / 16; ++i) {
      uint4 t = ldg_stream_v4(vp + 16 * i, pol);
      u.v[4 * i + 0] = t.x;
      u.v[4 * i + 1] = t.y;
      u.v[4 * i + 2] = t.z;
      u.v[4 * i + 3] = t.w;
    }
  }
  if constexpr (MB == 8) {
    uint2 t = ldg_stream_v2(a.meta + blk * 32 * MB + lane * MB, pol);
    u.m[0] = t.x;
    u.m[1] = t.y;
  } else if constexpr (MB == 4) {
    u.m[0] = ldg_stream_u32(a.meta + blk * 32 * MB + lane * MB, pol);
  } else {
    u.m[0] = 0;
  }
  if constexpr (has_scales(FMT)) {
    const int g = lane >> 2;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const size_t idx = (blk * E + e) * 16 + 2 * g;
      uint2 sc = ldg_stream_v2(a.scales + idx, pol);
      u.s[2 * e] = sc.x;
      u.s[2 * e + 1] = sc.y;
      u.z[e] = ldg_stream_u16(a.zps + idx, pol);
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

template <int NT>
__device__ __forceinline__ void load_b(uint32_t (&b)[NT][4], const uint32_t* sB, int KTc, int kt,
                                       int lane, int valid_cols_nt0, int M_left) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int col = lane >> 2;  // B column held by this lane
    const int cols_here = min(8, 2 * (M_left - 4 * nt));
    if (col < cols_here) {
      const uint4 t = *reinterpret_cast<const uint4*>(sB + ((nt * KTc + kt) * 32 + lane) * 4);
      b[nt][0] = t.x;
      b[nt][1] = t.y;
      b[nt][2] = t.z;
      b[nt][3] = t.w;
    } else {
      b[nt][0] = b[nt][1] = b[nt][2] = b[nt][3] = 0u;
    }
  }
  (void)valid_cols_nt0;
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

template <int FMT, int SS, int NT>
__device__ __forceinline__ void compute_unit(const Unit<FMT, 4 / SS>& u, const uint32_t* sB, int KTc,
                                             int kt_base, int lane, int M_left,
                                             float (&acc)[NT][2]) {
  float d[NT][4];
  uint32_t zg = 0, zg8 = 0, zpair = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int e = j / SS;
    if (j % SS == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
      if constexpr (has_scales(FMT)) {
        const uint32_t z0 = u.z[e] & 0xFFu, z1 = (u.z[e] >> 8) & 0xFFu;
        zg = zp_magic(z0, z0);
        zg8 = zp_magic(z1, z1);
        zpair = zp_magic(z0, z1);
      }
    }
    uint32_t b[NT][4];
    load_b<NT>(b, sB, KTc, kt_base + j, lane, 0, M_left);
    if constexpr (FMT == I4_SP24 || FMT == F16_SP24) {
      uint32_t a[4];
      if constexpr (FMT == I4_SP24) {
        const uint32_t w = u.v[j];
        a[0] = hsub2_u32(nib2_magic(w), zg);
        a[1] = hsub2_u32(nib2_magic(w >> 4), zg8);
        a[2] = hsub2_u32(nib2_magic(w >> 8), zg);
        a[3] = hsub2_u32(nib2_magic(w >> 12), zg8);
      } else {
        a[0] = u.v[4 * j + 0];
        a[1] = u.v[4 * j + 1];
        a[2] = u.v[4 * j + 2];
        a[3] = u.v[4 * j + 3];
      }
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
    } else {  // I4_DENSE: two m16n8k16 per 32-column k-tile
      const uint32_t w0 = u.v[2 * j], w1 = u.v[2 * j + 1];
      const uint32_t a0 = hsub2_u32(nib2_magic(w0), zg), a1 = hsub2_u32(nib2_magic(w0 >> 4), zg8);
      const uint32_t a2 = hsub2_u32(nib2_magic(w0 >> 8), zg), a3 = hsub2_u32(nib2_magic(w0 >> 12), zg8);
      const uint32_t c0 = hsub2_u32(nib2_magic(w1), zg), c1 = hsub2_u32(nib2_magic(w1 >> 4), zg8);
      const uint32_t c2 = hsub2_u32(nib2_magic(w1 >> 8), zg), c3 = hsub2_u32(nib2_magic(w1 >> 12), zg8);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        mma_16816(d[nt], a0, a1, a2, a3, b[nt][0], b[nt][1]);
        mma_16816(d[nt], c0, c1, c2, c3, b[nt][2], b[nt][3]);
      }
    }
    if (j % SS == SS - 1) {
      if constexpr (has_scales(FMT)) {
        const float sg = __uint_as_float(u.s[2 * e]), sg8 = __uint_as_float(u.s[2 * e + 1]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[nt][0] = fmaf(sg, d[nt][0] + d[nt][1], acc[nt][0]);
          acc[nt][1] = fmaf(sg8, d[nt][2] + d[nt][3], acc[nt][1]);
        }
      } else {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[nt][0] += d[nt][0] + d[nt][1];
          acc[nt][1] += d[nt][2] + d[nt][3];
        }
      }
    }
  }
}

// One CTA = RB row tiles x KC k-quads x 4*NT tokens, nw = blockDim/32 warps
// arranged as RBw = nw/WK warp rows x WK warp columns.  Warp (wi, wj) owns
// row tiles wi, wi+RBw, ... over the wj-th part of the CTA's k-quads and
// streams its units (row tile, k-quad) through a D-deep register pipeline;
// the first D units are requested before the PDL wait (weights do not depend
// on the previous kernel).  Split-K partial sums (S > 1) are reduced by the
// last-arriving CTA of each row block, in slice order: deterministic.
template <int FMT, int SS, int NT, int D>
__global__ void __launch_bounds__(256, 2) tiled_spmm_kernel(const TiledArgs a) {
  constexpr int E = 4 / SS;
  constexpr int TOK = 4 * NT;                       // tokens per CTA (power of two)
  constexpr int TOK_SHIFT = NT == 1 ? 2 : (NT == 2 ? 3 : 4);
  extern __shared__ __align__(16) uint32_t smem[];
  pdl_launch_dependents();

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = blockDim.x >> 5;
  const int RBw = nw / a.WK;
  const int wi = warp / a.WK, wj = warp % a.WK;
  const int rt0 = blockIdx.x * a.RB;
  const int RBc = min(a.RB, a.RT - rt0);
  const int kq0 = blockIdx.y * a.KC;
  const int kq1 = min(a.KQ, kq0 + a.KC);
  const int KTc = (kq1 - kq0) * 4;
  const int per = (kq1 - kq0 + a.WK - 1) / a.WK;
  const int k0 = min(kq1, kq0 + wj * per);
  const int nK = max(0, min(kq1, k0 + per) - k0);
  const int nR = wi < RBc ? (RBc - wi + RBw - 1) / RBw : 0;
  const int nU = nR * nK;
  const int m0 = blockIdx.z * TOK;
  const int M_left = a.M - m0;
  const int rt_base = a.rt_begin + rt0 + wi;  // storage row tile of the warp's first unit

  const uint64_t pol = evict_first_policy();
  Unit<FMT, E> buf[D];
  int lr = 0, lk = 0;  // (row iteration, k-quad) of the next unit to load
#pragma unroll
  for (int s = 0; s < D; ++s) {
    if (s < nU) {
      load_unit<FMT, E>(buf[s], a, rt_base + lr * RBw, k0 + lk, lane, pol);
      if (++lk == nK) { lk = 0; ++lr; }
    }
  }

  pdl_wait();  // x and the split-K workspace belong to earlier kernels

  // x slice -> fp16 hi/lo B fragments sB[nt][kt][lane][4]: token m's hi part
  // is B column 2m (lanes 8m..8m+3), its lo part (the rounding residual)
  // column 2m+1.  Only the lanes of present tokens are written (load_b skips
  // the others).
  uint32_t* sB = smem;
  const int nB = NT * KTc * 128;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int items = KTc * 64;
    for (int i = tid; i < items; i += blockDim.x) {
      const int reg = i & 3, t = (i >> 2) & 3, m = (i >> 4) & 3, kt = i >> 6;
      const int tok = m0 + 4 * nt + m;
      if (tok >= a.M) continue;
      const int k = (kq0 * 4 + kt) * 32 + 2 * t + 8 * reg;
      float v0 = 0.f, v1 = 0.f;
      if (k < a.cols) {
        const float* xp = a.x + static_cast<size_t>(tok) * a.ldx + k;
        v0 = xp[0];
        v1 = xp[1];
      }
      const __half h0 = __float2half_rn(v0), h1 = __float2half_rn(v1);
      const __half l0 = __float2half_rn(v0 - __half2float(h0));
      const __half l1 = __float2half_rn(v1 - __half2float(h1));
      uint32_t* row = sB + static_cast<size_t>(nt * KTc + kt) * 128;
      row[(8 * m + t) * 4 + reg] = static_cast<uint32_t>(__half_as_ushort(h0)) |
                                   (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
      row[(8 * m + 4 + t) * 4 + reg] = static_cast<uint32_t>(__half_as_ushort(l0)) |
                                       (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
    }
  }
  float* red = reinterpret_cast<float*>(smem + nB);  // [RB][WK][TOK][16]
  const int nRed = a.RB * a.WK * TOK * 16;
  for (int i = tid; i < nRed; i += blockDim.x) red[i] = 0.f;
  __syncthreads();

  float acc[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.f;
  int cr = 0, ck = 0;  // (row iteration, k-quad) of the unit being computed
  const int g = lane >> 2, t = lane & 3;
  for (int base = 0; base < nU; base += D) {
#pragma unroll
    for (int s = 0; s < D; ++s) {
      if (base + s < nU) {
        compute_unit<FMT, SS, NT>(buf[s], sB, KTc, (k0 + ck - kq0) * 4, lane, M_left, acc);
        if (base + s + D < nU) {
          load_unit<FMT, E>(buf[s], a, rt_base + lr * RBw, k0 + lk, lane, pol);
          if (++lk == nK) { lk = 0; ++lr; }
        }
        if (++ck == nK) {  // row tile done: park its partial sums in smem
          float* r = red + ((static_cast<size_t>(wi + cr * RBw) * a.WK + wj) * TOK) * 16;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            r[(4 * nt + t) * 16 + g] = acc[nt][0];
            r[(4 * nt + t) * 16 + g + 8] = acc[nt][1];
            acc[nt][0] = acc[nt][1] = 0.f;
          }
          ck = 0;
          ++cr;
        }
      }
    }
  }
  __syncthreads();

  const int rows_pad = a.RT * 16;
  const int nOut = RBc * TOK * 16;
  for (int idx = tid; idx < nOut; idx += blockDim.x) {
    const int row16 = idx & 15, tl = (idx >> 4) & (TOK - 1), i = idx >> (4 + TOK_SHIFT);
    float v = 0.f;
    for (int j = 0; j < a.WK; ++j) v += red[((static_cast<size_t>(i) * a.WK + j) * TOK + tl) * 16 + row16];
    const int row = (rt0 + i) * 16 + row16;
    const int tok = m0 + tl;
    if (row < a.rows && tok < a.M) {
      if (a.S == 1)
        a.y[static_cast<size_t>(tok) * a.ldy + row] = v;
      else
        a.partial[(static_cast<size_t>(blockIdx.y) * a.M + tok) * rows_pad + row] = v;
    }
  }
  if (a.S == 1) return;

  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  const int cidx = blockIdx.x + gridDim.x * blockIdx.z;
  if (tid == 0) s_last = (atomicAdd(a.counters + cidx, 1u) == static_cast<uint32_t>(a.S - 1));
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int idx = tid; idx < nOut; idx += blockDim.x) {
    const int row16 = idx & 15, tl = (idx >> 4) & (TOK - 1), i = idx >> (4 + TOK_SHIFT);
    const int row = (rt0 + i) * 16 + row16;
    const int tok = m0 + tl;
    if (row < a.rows && tok < a.M) {
      float v = 0.f;
      for (int sidx = 0; sidx < a.S; ++sidx)
        v += __ldcg(a.partial + (static_cast<size_t>(sidx) * a.M + tok) * rows_pad + row);
      a.y[static_cast<size_t>(tok) * a.ldy + row] = v;
    }
  }
  if (tid == 0) a.counters[cidx] = 0u;  // ready for the next launch / graph replay
}

// ---------------------------------------------------------------- planning

namespace {
constexpr int kDepth = 4;

template <int FMT, int SS, int NT>
void* kernel_ptr() {
  return reinterpret_cast<void*>(&tiled_spmm_kernel<FMT, SS, NT, kDepth>);
}

template <int FMT, int SS>
void* pick_nt(int NT) {
  switch (NT) {
    case 1: return kernel_ptr<FMT, SS, 1>();
    case 2: return kernel_ptr<FMT, SS, 2>();
    default: return kernel_ptr<FMT, SS, 4>();
  }
}

template <int FMT>
void* pick_ss(int SS, int NT) {
  switch (SS) {
    case 1: return pick_nt<FMT, 1>(NT);
    case 2: return pick_nt<FMT, 2>(NT);
    default: return pick_nt<FMT, 4>(NT);
  }
}

void* pick_kernel(int fmt, int SS, int NT) {
  switch (fmt) {
    case I4_SP24: return pick_ss<I4_SP24>(SS, NT);
    case I4_SP14: return pick_ss<I4_SP14>(SS, NT);
    case I4_DENSE: return pick_ss<I4_DENSE>(SS, NT);
    case F16_SP24: return pick_nt<F16_SP24, 4>(NT);
    default: return pick_nt<F16_SP14, 4>(NT);
  }
}

size_t block_bytes(const egt_dev_packed* h) {
  const int f = h->format;
  size_t b = 32u * (val_lane_bytes(f) + meta_lane_bytes(f));
  if (has_scales(f)) b += 16u * 5u * h->tiled.E;
  return b;
}

size_t smem_bytes(int NT, int KC, int RB, int WK) {
  return static_cast<size_t>(NT) * KC * 4 * 512 + static_cast<size_t>(RB) * WK * 4 * NT * 16 * 4;
}
}  // namespace

// Picks the CTA tile (RB row tiles x KC k-quads, nw warps as RBw x WK) and the
// split-K factor S with a small model of one launch: the busiest SM's HBM
// bytes at its 1/148 share of bandwidth, the per-scheduler issue time of the
// dequant + mma.sp stream, the number of waves, and a fixed tail for the
// split-K reduction.  Everything is resident in one wave whenever possible
// (2 CTAs/SM leave room for the next kernel's CTAs under PDL).
TiledSchedule plan_tiled(const egt_dev_packed* h, int M, int num_sms) {
  TiledSchedule best;
  const int RT = h->tiled.RT, KQ = h->tiled.KQ;
  const int NT = M <= 4 ? 1 : (M <= 8 ? 2 : 4);
  const int NB = (M + 4 * NT - 1) / (4 * NT);
  const int tok = std::min(M, 4 * NT);
  const double unit_b = static_cast<double>(block_bytes(h));
  const double sm_bw = 44.0;          // B/ns per SM (6.5 TB/s / 148)
  const double unit_cycles = 60.0 * NT;  // issue slots per (warp, unit)
  void* fn = pick_kernel(h->format, h->tiled.SS, NT);
  double best_cost = 1e300;
  for (int S = 1; S <= std::min(KQ, 8); ++S) {
    const int KC = (KQ + S - 1) / S;
    if (S > 1 && (S - 1) * KC >= KQ) continue;
    for (int nw : {4, 8}) {
      for (int WK : {1, 2, 4, 8}) {
        if (WK > nw || WK > KC) continue;
        const int RBw = nw / WK;
        for (int RB = 1; RB <= 64; ++RB) {
          const size_t smem = smem_bytes(NT, KC, RB, WK);
          if (smem > 200 * 1024) continue;
          int occ = 0;
          if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * nw, smem) != cudaSuccess ||
              occ < 1)
            continue;
          const long grid = static_cast<long>((RT + RB - 1) / RB) * S * NB;
          const double ctas_per_sm = std::ceil(static_cast<double>(grid) / num_sms);
          const double waves = std::ceil(static_cast<double>(grid) / (static_cast<double>(num_sms) * occ));
          const double units_per_warp = std::ceil(static_cast<double>(RB) / RBw) *
                                        std::ceil(static_cast<double>(KC) / WK);
          const double bytes_cta = RB * KC * unit_b + KC * 512.0 * tok + (S > 1 ? 2.0 * RB * 64 * tok : 0.0);
          const double t_mem = ctas_per_sm * bytes_cta / sm_bw;
          const double warps_per_sched = std::max(1.0, nw * std::min<double>(occ, ctas_per_sm) / 4.0);
          const double t_issue = waves * units_per_warp * unit_cycles * warps_per_sched / 1.9;
          const double t_tail = waves * 700.0 + (S > 1 ? 700.0 : 0.0);
          const double cost = std::max(t_mem, t_issue) + t_tail;
          if (cost < best_cost * 0.999) {
            best_cost = cost;
            best.RB = RB;
            best.WK = WK;
            best.KC = KC;
            best.S = S;
            best.NT = NT;
            best.NB = NB;
            best.grid_x = (RT + RB - 1) / RB;
            best.grid_y = S;
            best.grid_z = NB;
            best.nw = nw;
            best.smem = smem;
          }
        }
      }
    }
  }
  return best;
}

size_t tiled_workspace_floats(const egt_dev_packed* h, const TiledSchedule& sc, int M) {
  if (sc.S <= 1) return 0;
  return static_cast<size_t>(sc.S) * M * h->tiled.RT * 16;
}

cudaError_t launch_tiled(const egt_dev_packed* h, const TiledSchedule& sc, const float* x, int ldx,
                         int M, float* y, int ldy, const LaunchCtx& ctx) {
  TiledArgs a;
  a.vals = h->tiled.vals;
  a.meta = h->tiled.meta;
  a.scales = h->tiled.scales;
  a.zps = h->tiled.zps;
  a.KQ = h->tiled.KQ;
  a.rt_begin = h->tiled.rt_begin;
  a.RT = h->tiled.RT;
  a.rows = static_cast<int>(h->rows);
  a.cols = static_cast<int>(h->cols);
  a.x = x;
  a.ldx = ldx;
  a.M = M;
  a.y = y;
  a.ldy = ldy;
  a.partial = ctx.partial;
  a.counters = ctx.counters;
  a.RB = sc.RB;
  a.WK = sc.WK;
  a.KC = sc.KC;
  a.S = sc.S;
  void* fn = pick_kernel(h->format, h->tiled.SS, sc.NT);
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sc.smem));
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sc.grid_x, sc.grid_y, sc.grid_z);
  cfg.blockDim = dim3(32 * sc.nw);
  cfg.dynamicSmemBytes = sc.smem;
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

}  // namespace egt_impl
