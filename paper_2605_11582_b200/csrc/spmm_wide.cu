// Many-token SparseGemv (M >= 17): the X * W^T products of the prefix-tree
// verification pass (forward_impl, model.cpp:156-195, M = committed prefix +
// tree nodes, 64-272 rows in the BASELINE configs).
//
// The one-wave M <= 16 kernel (spmm_tiled.cu) keeps the CTA's whole K range
// of x fragments in shared memory; at M = 80 that no longer fits and it falls
// back to dozens of K slices whose partial sums outweigh the weights.  Here:
//   1. xfrag_kernel splits X once into fp16 hi/lo B fragments in global
//      memory, [token block of 16][n-tile][k-tile][32 lanes][4 u32] (the
//      layout compute_unit reads with LS = 32), zero-padded (L2 resident).
//   2. wide_spmm_kernel: one CTA = RB row tiles x one 16-token block over the
//      full K.  A producer warp streams, per chunk of CH k-quads, the x chunk
//      (4 bulk copies, one per n-tile) into a 2-deep ring and each row tile's
//      weight blocks into a weight ring; consumer warp w owns row tiles
//      w, w + nw, ... so every row is reduced inside one warp (no cross-warp
//      reduction) and stored directly.  Weights are read ceil(M / 16) times,
//      x fragments once per CTA: at these M the kernel is tensor-pipe bound.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "device_common.cuh"

#include <cmath>
#include "handle.h"
#include "tiled_compute.cuh"
#include "xrange.cuh"

namespace egt_impl {

constexpr int kWideTok = 16;    // tokens per CTA (4 n-tiles of 4)
constexpr int kWideMaxRT = 2;   // row tiles per consumer warp

struct WideArgs {
  const uint8_t* vals;
  const uint8_t* meta;
  const float* scales;
  const uint8_t* zps;
  const uint32_t* xf;  // x fragments
  float* y;
  int KQ, rt_begin, RT, rows, M, ldy, RB, CH, NSTW, wstage_bytes, xstage_bytes, KTtot;
  int XS;  // x chunk stages
  const float* res;  // y = res + product (may alias y; row stride ldr), model.cpp:186/190
  int ldr;
  int out_silu;      // y = silu(...), model.cpp:80-84 (the next product's input)
  // x range (xrange.cuh): per token 2^-e rescale and non-finite flag
  // (written by xfrag_kernel), and x itself for the non-finite fix-up
  const float* unsc;
  const uint32_t* nonfin;
  const float* x;
  int ldx, cols, SS, pad14;
};

// X [M x cols] (row stride ldx) -> fragments, one CTA per (padded) token:
// the token's row range first (xrange.cuh: finite max |x| -> 2^e, non-finite
// flag), then one thread per (k-tile, part, t): 4 u32 = lane (g, t)'s B
// fragment (k = kt*32 + 2t + 8r, pair (k, k+1); g = 2 (tok % 4) + part,
// part 0 = fp16 hi, 1 = residual lo), at [token block][n-tile][k-tile][lane].
__global__ void __launch_bounds__(256) xfrag_kernel(const float* __restrict__ x, int ldx, int M, int cols,
                                                    int KTtot, uint32_t* __restrict__ xf, float* __restrict__ unsc,
                                                    uint32_t* __restrict__ nonfin) {
  // launched programmatically: x (and the fragment workspace the previous
  // product reads) belong to the preceding kernel
  pdl_wait();
  pdl_launch_dependents();
  __shared__ uint32_t s_mx, s_nf;
  const int tok = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) {
    s_mx = 0u;
    s_nf = 0u;
  }
  __syncthreads();
  const float* xr = x + static_cast<size_t>(tok) * ldx;
  if (tok < M) {
    uint32_t mx = 0u, nf = 0u;
    for (int k = tid; k < cols; k += blockDim.x) xr_note(mx, nf, __ldg(xr + k));
    xr_commit(mx, nf, &s_mx, &s_nf);
  }
  __syncthreads();
  const int e = xr_exp(s_mx);
  const float sc = xr_pow2(e);
  if (tid == 0) {
    unsc[tok] = xr_pow2(-e);
    nonfin[tok] = s_nf;
  }
  const int tb = tok / kWideTok, nt = (tok % kWideTok) / 4, m4 = tok % 4;
  for (int idx = tid; idx < KTtot * 8; idx += blockDim.x) {
    const int kt = idx >> 3, part = (idx >> 2) & 1, t = idx & 3;
    const int lane = 4 * (2 * m4 + part) + t;
    uint4 o;
    uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int reg = 0; reg < 4; ++reg) {
      const int k = kt * 32 + 2 * t + 8 * reg;
      float a = 0.f, b = 0.f;
      if (tok < M) {
        if (k < cols) a = xr_scaled(__ldg(xr + k), sc);
        if (k + 1 < cols) b = xr_scaled(__ldg(xr + k + 1), sc);
      }
      __half ha = __float2half_rn(a), hb = __float2half_rn(b);
      if (part) {
        ha = __float2half_rn(a - __half2float(ha));
        hb = __float2half_rn(b - __half2float(hb));
      }
      op[reg] = static_cast<uint32_t>(__half_as_ushort(ha)) | (static_cast<uint32_t>(__half_as_ushort(hb)) << 16);
    }
    reinterpret_cast<uint4*>(xf)[((static_cast<size_t>(tb) * 4 + nt) * KTtot + kt) * 32 + lane] = o;
  }
}

// sum of W[row][c] * x[c] over the kept entries of row with non-finite x[c]
template <int FMT>
__device__ __noinline__ float wide_nonfinite_terms(const WideArgs& a, int row, int tok) {
  const TiledRef m{a.vals, a.meta, a.scales, a.zps, a.KQ, a.rt_begin, a.SS, a.pad14};
  const float* xr = a.x + static_cast<size_t>(tok) * a.ldx;
  float add = 0.f;
  for (int c = 0; c < a.cols; ++c) {
    const float xv = xr[c];
    if ((__float_as_uint(xv) & 0x7fffffffu) < 0x7f800000u) continue;
    float w;
    if (tiled_value<FMT>(m, row, c, &w)) add += w * xv;
  }
  return add;
}

template <int FMT, int SS, int NW>
__global__ void __launch_bounds__(32 * (NW + 1), 1) wide_spmm_kernel(const __grid_constant__ WideArgs a) {
  constexpr int E = 4 / SS;
  constexpr int VB = val_lane_bytes(FMT), MB = meta_lane_bytes(FMT);
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int nw = NW;
  const int rt0 = blockIdx.x * a.RB;
  const int RBc = min(a.RB, a.RT - rt0);
  const int tb = blockIdx.y;
  const int NCH = (a.KQ + a.CH - 1) / a.CH;
  uint64_t* xfull = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* xempty = xfull + a.XS;
  uint64_t* wfull = xempty + a.XS;
  uint64_t* wempty = wfull + a.NSTW;
  uint8_t* xst = smem_raw + ((16 * (2 * a.XS + 2 * a.NSTW) + 127) / 128) * 128;
  uint8_t* wst = xst + static_cast<size_t>(a.XS) * a.xstage_bytes;
  if (tid == 0) {
    for (int s = 0; s < a.XS; ++s) {
      mbar_init(xfull + s, 1);
      mbar_init(xempty + s, nw);
    }
    for (int s = 0; s < a.NSTW; ++s) {
      mbar_init(wfull + s, 1);
      mbar_init(wempty + s, 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // x fragments come from the preceding xfrag_kernel

  if (warp == nw) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int ws = 0;
      uint32_t wph = 0;
      long long wq = 0;
      for (int c = 0; c < NCH; ++c) {
        const int kq0 = c * a.CH, n = min(a.CH, a.KQ - kq0);
        const int xs = c % a.XS;
        if (c >= a.XS) mbar_wait(xempty + xs, ((c / a.XS) - 1) & 1);
        const uint32_t xb = static_cast<uint32_t>(n) * 4 * 512;  // bytes per n-tile
        mbar_expect_tx(xfull + xs, 4 * xb);
        for (int nt = 0; nt < 4; ++nt) {
          const uint32_t* src = a.xf + ((static_cast<size_t>(tb) * 4 + nt) * a.KTtot + kq0 * 4) * 128;
          bulk_g2s(xst + xs * a.xstage_bytes + nt * (a.CH * 4 * 512), src, xb, xfull + xs, pol);
        }
        for (int i = 0; i < RBc; ++i) {
          if (wq >= a.NSTW) mbar_wait(wempty + ws, wph ^ 1u);
          uint8_t* st = wst + static_cast<size_t>(ws) * a.wstage_bytes;
          const size_t blk = static_cast<size_t>(a.rt_begin + rt0 + i) * a.KQ + kq0;
          mbar_expect_tx(wfull + ws, stage_bytes<FMT>(n, E));
          bulk_g2s(st, a.vals + blk * 32 * VB, n * 32 * VB, wfull + ws, pol);
          if constexpr (MB > 0) bulk_g2s(st + n * 32 * VB, a.meta + blk * 32 * MB, n * 32 * MB, wfull + ws, pol);
          if constexpr (has_scales(FMT)) {
            uint8_t* sp = st + n * 32 * (VB + MB);
            bulk_g2s(sp, a.scales + blk * E * 16, n * E * 64, wfull + ws, pol);
            bulk_g2s(sp + n * E * 64, a.zps + blk * E * 16, n * E * 16, wfull + ws, pol);
          }
          ++wq;
          if (++ws == a.NSTW) {
            ws = 0;
            wph ^= 1u;
          }
        }
      }
    }
    return;
  }

  // consumer warp: row tiles warp, warp + nw, ... (at most kWideMaxRT)
  float acc[kWideMaxRT][4][2];
#pragma unroll
  for (int r = 0; r < kWideMaxRT; ++r)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[r][nt][0] = acc[r][nt][1] = 0.f;
  // own row tiles: warp + r * nw (r < nr); both are consumed in lockstep so
  // that every B fragment load from shared memory feeds nr row tiles
  const int nr = warp < RBc ? (warp + nw < RBc ? 2 : 1) : 0;
  static_assert(kWideMaxRT == 2, "lockstep over two row tiles");
  for (int c = 0; c < NCH; ++c) {
    const int n = min(a.CH, a.KQ - c * a.CH);
    const int xs = c % a.XS;
    mbar_wait(xfull + xs, (c / a.XS) & 1);
    const uint32_t* sx = reinterpret_cast<const uint32_t*>(xst + xs * a.xstage_bytes);
    const uint8_t* st[kWideMaxRT] = {nullptr, nullptr};
    int wsi[kWideMaxRT] = {0, 0};
    for (int r = 0; r < nr; ++r) {
      const long long q = static_cast<long long>(c) * RBc + warp + r * nw;  // weight stage index
      wsi[r] = static_cast<int>(q % a.NSTW);
      mbar_wait(wfull + wsi[r], static_cast<uint32_t>((q / a.NSTW) & 1));
      st[r] = wst + static_cast<size_t>(wsi[r]) * a.wstage_bytes;
    }
    const int KTc = a.CH * 4;
    if (nr == 2) {
      for (int u = 0; u < n; ++u) {
        Unit<FMT, E> un[2];
        const Cursor c0 = make_cursor<FMT, E>(st[0], n, u, lane, sx, u * 4, 32);
        const Cursor c1 = make_cursor<FMT, E>(st[1], n, u, lane, sx, u * 4, 32);
        lds_unit<FMT, E>(un[0], c0);
        lds_unit<FMT, E>(un[1], c1);
        compute_units<FMT, SS, 4, 2>(un, sx + (u * 4 * 32 + lane) * 4, KTc, 32, acc);
      }
    } else if (nr == 1) {
      float (&a1)[1][4][2] = *reinterpret_cast<float (*)[1][4][2]>(&acc[0]);
      for (int u = 0; u < n; ++u) {
        Unit<FMT, E> un[1];
        lds_unit<FMT, E>(un[0], make_cursor<FMT, E>(st[0], n, u, lane, sx, u * 4, 32));
        compute_units<FMT, SS, 4, 1>(un, sx + (u * 4 * 32 + lane) * 4, KTc, 32, a1);
      }
    }
    __syncwarp();
    if (lane == 0) {
      for (int r = 0; r < nr; ++r) mbar_arrive(wempty + wsi[r]);
      mbar_arrive(xempty + xs);
    }
  }
  // lane (g, t): n-tile nt's token 4nt + t, rows g (acc[.][0]) and g + 8 (acc[.][1])
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int r = 0; r < kWideMaxRT; ++r) {
    const int i = warp + r * nw;
    if (i < RBc) {
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int tok = tb * kWideTok + 4 * nt + t;
        if (tok < a.M) {
          const int row = (rt0 + i) * 16 + g;
          float* yr = a.y + static_cast<size_t>(tok) * a.ldy;
          const float* rr = a.res ? a.res + static_cast<size_t>(tok) * a.ldr : nullptr;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int rw = row + 8 * hh;
            if (rw < a.rows) {
              float p = acc[r][nt][hh] * a.unsc[tok];  // undo the token's 2^e (xrange.cuh)
              if (a.nonfin[tok]) p += wide_nonfinite_terms<FMT>(a, rw, tok);
              float val = (rr ? rr[rw] : 0.f) + p;
              if (a.out_silu) val = val * (1.0f / (1.0f + expf(-val)));
              yr[rw] = val;
            }
          }
        }
      }
    }
  }
}

namespace {
template <int FMT, int SS>
void* wide_ptr(int nw) {
  return nw == 12 ? reinterpret_cast<void*>(&wide_spmm_kernel<FMT, SS, 12>)
                  : reinterpret_cast<void*>(&wide_spmm_kernel<FMT, SS, 8>);
}
void* pick_wide(int fmt, int SS, int nw) {
  switch (fmt * 8 + SS) {
    case I4_SP24 * 8 + 4: return wide_ptr<I4_SP24, 4>(nw);
    case I4_SP24 * 8 + 2: return wide_ptr<I4_SP24, 2>(nw);
    case I4_SP24 * 8 + 1: return wide_ptr<I4_SP24, 1>(nw);
    case I4_SP14 * 8 + 4: return wide_ptr<I4_SP14, 4>(nw);
    case I4_SP14 * 8 + 2: return wide_ptr<I4_SP14, 2>(nw);
    case I4_SP14 * 8 + 1: return wide_ptr<I4_SP14, 1>(nw);
    case I4_DENSE * 8 + 4: return wide_ptr<I4_DENSE, 4>(nw);
    case I4_DENSE * 8 + 2: return wide_ptr<I4_DENSE, 2>(nw);
    case I4_DENSE * 8 + 1: return wide_ptr<I4_DENSE, 1>(nw);
    case F16_SP24 * 8 + 4: return wide_ptr<F16_SP24, 4>(nw);
    default: return wide_ptr<F16_SP14, 4>(nw);
  }
}
}  // namespace

size_t wide_workspace_bytes(const egt_dev_packed* h, int M) {
  const int TB = (M + kWideTok - 1) / kWideTok;
  // fragments, then per padded token the rescale and the non-finite flag
  return static_cast<size_t>(TB) * 4 * h->tiled.KQ * 4 * 512 + static_cast<size_t>(TB) * kWideTok * 8;
}

cudaError_t launch_wide(const egt_dev_packed* h, const float* x, int ldx, int M, float* y, int ldy,
                        uint32_t* xf_ws, const LaunchCtx& ctx, int num_sms) {
  const int KQ = h->tiled.KQ, RT = h->tiled.RT, E = h->tiled.E, fmt = h->format;
  const int KTtot = KQ * 4;
  const int TB = (M + kWideTok - 1) / kWideTok;
  float* unsc = reinterpret_cast<float*>(xf_ws + static_cast<size_t>(TB) * 4 * KTtot * 128);
  uint32_t* nonfin = reinterpret_cast<uint32_t*>(unsc + TB * kWideTok);
  {
    cudaLaunchConfig_t xc = {};
    xc.gridDim = dim3(TB * kWideTok);
    xc.blockDim = dim3(256);
    xc.stream = ctx.stream;
    cudaLaunchAttribute xa[1];
    xa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    xa[0].val.programmaticStreamSerializationAllowed = 1;
    xc.attrs = xa;
    xc.numAttrs = ctx.pdl ? 1 : 0;
    const int cols_ = static_cast<int>(h->cols);
    void* xargs[] = {const_cast<float**>(&x), &ldx, &M, const_cast<int*>(&cols_), const_cast<int*>(&KTtot),
                     &xf_ws, &unsc, &nonfin};
    cudaError_t xe = cudaLaunchKernelExC(&xc, reinterpret_cast<void*>(&xfrag_kernel), xargs);
    if (xe != cudaSuccess) return xe;
    ++launch_counter();
  }
  WideArgs a;
  a.vals = h->tiled.vals;
  a.meta = h->tiled.meta;
  a.scales = h->tiled.scales;
  a.zps = h->tiled.zps;
  a.xf = xf_ws;
  a.y = y;
  a.KQ = KQ;
  a.rt_begin = h->tiled.rt_begin;
  a.RT = RT;
  a.rows = static_cast<int>(h->rows);
  a.M = M;
  a.ldy = ldy;
  a.KTtot = KTtot;
  a.res = ctx.res;
  a.ldr = ctx.ldr;
  a.out_silu = ctx.out_silu;
  a.unsc = unsc;
  a.nonfin = nonfin;
  a.x = x;
  a.ldx = ldx;
  a.cols = static_cast<int>(h->cols);
  a.SS = h->tiled.SS;
  a.pad14 = h->tiled.pad14;
  // RB: up to nw * kWideMaxRT row tiles; fewer when the token blocks alone
  // leave SMs idle (one wave of CTAs at one per SM)
  // RB: the critical path of the busiest SM is waves x (consumer warps per
  // scheduler) x (row tiles per warp, lockstep pairs cost ~2 singles); ties
  // go to the larger RB (x fragments re-read by fewer CTAs).
  // Consumer warps: 12 when the token blocks are few (M <= 128: one wave of
  // 12-row-tile CTAs), else 8 (measured, tools/wide_probe.py / verify_probe.py:
  // M = 80 products 16-21 % faster with 12, M = 272 8 % slower).
  static const int nw_env = getenv("EGT_WIDE_NW") ? atoi(getenv("EGT_WIDE_NW")) : 0;
  const int NW = nw_env == 8 || nw_env == 12 ? nw_env : (TB <= 8 ? 12 : 8);
  // Consumer warps hold up to two row tiles' stages of one chunk at once, so
  // the weight ring must cover a whole chunk (NSTW >= RB): then issuing chunk
  // c only ever waits for stages of chunk c - 1, which complete unconditionally.
  const int blk = 32 * (val_lane_bytes(fmt) + meta_lane_bytes(fmt)) + (has_scales(fmt) ? E * 80 : 0);
  static const int ch0 = getenv("EGT_WIDE_CH") ? atoi(getenv("EGT_WIDE_CH")) : 8;
  static const int cap = getenv("EGT_WIDE_NSTW") ? atoi(getenv("EGT_WIDE_NSTW")) : 32;
  static const int xs_env = getenv("EGT_WIDE_XS") ? atoi(getenv("EGT_WIDE_XS")) : 2;
  a.XS = std::max(2, std::min(8, xs_env));
  // k-quads per stage for rb row tiles: the largest CH <= ch0 whose ring
  // still holds a whole chunk
  auto chunk_for = [&](int rb) {
    int ch = std::max(1, ch0);
    for (;; ch /= 2) {
      const int wsb = (ch * blk + 127) / 128 * 128;
      const int budget = 200 * 1024 - a.XS * 4 * ch * 4 * 512 - 1024;
      if ((budget > 0 && std::min(std::max(cap, rb), budget / wsb) >= rb) || ch == 1) return ch;
    }
  };
  // RB: critical path of the busiest SM = waves x (consumer warps per
  // scheduler) x (row tiles per warp), x1.35 when the ring only fits weight
  // stages under 6 KB (the single producer thread's TMA issue rate then
  // bounds the kernel: measured, tools/wide_probe.py); ties -> the larger RB.
  int RB = 1;
  double best = 1e300;
  for (int rb = 1; rb <= NW * kWideMaxRT; ++rb) {
    const long long grid = static_cast<long long>((RT + rb - 1) / rb) * TB;
    const double waves = std::ceil(static_cast<double>(grid) / num_sms);
    const int busy = std::min(rb, NW);
    const double cost = waves * ((busy + 3) / 4) * ((rb + NW - 1) / NW) * (chunk_for(rb) * blk >= 6144 ? 1.0 : 1.35);
    if (cost <= best) {
      best = cost;
      RB = rb;
    }
  }
  static const int rb_force = getenv("EGT_WIDE_RB") ? atoi(getenv("EGT_WIDE_RB")) : 0;
  if (rb_force > 0) RB = std::min(rb_force, NW * kWideMaxRT);
  a.RB = RB;
  for (a.CH = std::max(1, ch0);; a.CH /= 2) {
    a.wstage_bytes = (a.CH * blk + 127) / 128 * 128;
    a.xstage_bytes = 4 * a.CH * 4 * 512;
    const int budget = 200 * 1024 - a.XS * a.xstage_bytes - 1024;
    a.NSTW = std::min(std::max(cap, RB), budget / a.wstage_bytes);
    if (a.NSTW >= RB || a.CH == 1) break;
  }
  if (a.NSTW < RB) return cudaErrorInvalidConfiguration;
  const size_t smem = (16 * (2 * a.XS + 2 * a.NSTW) + 127) / 128 * 128 + static_cast<size_t>(a.XS) * a.xstage_bytes +
                      static_cast<size_t>(a.NSTW) * a.wstage_bytes;
  void* fn = pick_wide(fmt, h->tiled.SS, NW);
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((RT + RB - 1) / RB, TB, 1);
  cfg.blockDim = dim3(32 * (NW + 1));
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

}  // namespace egt_impl
