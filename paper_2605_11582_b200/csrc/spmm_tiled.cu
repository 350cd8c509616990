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
#include "tiled_compute.cuh"
#include "xrange.cuh"
#ifndef EGT_X4
#define EGT_X4 4
#endif
#ifndef EGT_XU
#define EGT_XU 8
#endif
#include "egt_b200.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

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
  int RB, WK, KC, S, NST, CH;
  int dbg;    // tuning experiments: 1 = empty kernel, 2 = weight stream only
  int indep;  // x is not produced by the previous kernel in the stream
  // fused forward_impl glue (model.cpp:155-190): input transform of x
  // (EGT_INPUT_RMSNORM per token, EGT_INPUT_SILU) and y = res + product
  int xform;
  float eps;
  const float* res;
  int ldr;
  int out_silu;  // y = silu(res + product): the producer applies the next product's input transform
  // L2 prefetch of the NEXT product's weights (decode chains): each CTA
  // requests its share of the four storage arrays while this product runs
  const uint8_t* pf_ptr[4];
  uint32_t pf_bytes[4];
  // tuning (EGT_TILED_TRACE): globaltimer stamps per launch slot:
  // [0] CTA 0 start, [1] CTA 0 past the PDL wait, [2] CTA 0 x staged,
  // [3] CTA 0 compute done, [4] last CTA exit (max), [5] ~first CTA start
  unsigned long long* trace;
  int trace_slot;
  // several matrices of one shape over the same x (decode Q/K/V): a virtual
  // matrix of nseg * RTs row tiles; segment s reads seg_* and writes seg_y[s]
  int nseg, RTs, rows_s;
  const uint8_t* seg_vals[3];
  const uint8_t* seg_meta[3];
  const float* seg_scales[3];
  const uint8_t* seg_zps[3];
  float* seg_y[3];
  int seg_rtb[3];
  // row shard with a fused all-gather: y rows go to every
  // peer's buffer (NVLink P2P stores) at peer_row0 + row; the last CTA to
  // finish signals each peer and (peer_wait) waits for every peer's slice
  int npeer, peer_rank, peer_row0, peer_wait;
  float* peer_y[kMaxPeers];
  uint32_t* peer_flag[kMaxPeers];
  uint32_t* peer_ctrl;  // this rank's [expected, done, error]
  // INT4 1:4 stored as 2:4 with zero-valued partners (the non-finite x
  // fix-up must skip the partners: they are not kept entries)
  int pad14;
  int seg_pad14[3];
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}


// silu (model.cpp:80-84) out of line: inlined 24x into the unrolled x
// staging it bloats the kernel past the instruction cache.
__device__ __noinline__ float2 silu2(float2 v) {
  return make_float2(v.x * (1.0f / (1.0f + expf(-v.x))), v.y * (1.0f / (1.0f + expf(-v.y))));
}

// One CTA = RB row tiles x KC k-quads (one of S K-slices) x 4*NT tokens.
// Warp specialised: warp nw (the producer) streams chunks of row tiles -- CH
// k-quads of one row tile, 2-4 contiguous bulk copies -- into an NST-deep
// ring of shared-memory stages (cp.async.bulk + mbarrier complete_tx); the
// first NST chunks are requested before the PDL wait, since weights do not
// depend on the previous kernel.  The nw consumer warps split each chunk's
// k-quads (two units in flight per warp), dequantise in registers and issue
// mma.sp.  Per-warp partial sums are reduced in a fixed order; split-K
// (S > 1) partial rows are summed by the last-arriving CTA of the row block,
// in slice order, so results are deterministic.
template <bool FUSED>
__device__ __forceinline__ void store_out(const TiledArgs& a, int tok, int row, float o) {
  if (FUSED && a.npeer > 0) {
    const size_t off = static_cast<size_t>(tok) * a.ldy + a.peer_row0 + row;
    for (int p = 0; p < a.npeer; ++p) a.peer_y[p][off] = o;
  } else if (FUSED && a.nseg > 1) {
    const int sg = row / a.rows_s;
    a.seg_y[sg][static_cast<size_t>(tok) * a.ldy + (row - sg * a.rows_s)] = o;
  } else {
    a.y[static_cast<size_t>(tok) * a.ldy + row] = o;
  }
}

// Fused all-gather completion: every storing CTA orders its stores before
// its done count (gpu scope: the counter is local); the last one, after a
// system-scope acq_rel fence (cumulative over everything the counter
// observed), bumps this rank's arrival counter in every peer's flag array
// and (peer_wait) waits until every rank's counter here reached this call's
// sequence number.  The wait is bounded (2 s of globaltimer): a missing peer
// sets the error word instead of hanging.  One rank: kernel completion
// already orders the (local) stores, so there is nothing to exchange.
__device__ __forceinline__ void peer_complete(const TiledArgs& a, unsigned expect) {
  if (a.npeer == 1 && a.dbg != 14) return;
  __syncthreads();  // the CTA's stores happen-before thread 0's fence
  if (threadIdx.x != 0) return;
  __threadfence();
  if (atomicAdd(a.peer_ctrl + 1, 1u) != expect - 1) return;
  a.peer_ctrl[1] = 0u;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int p = 0; p < a.npeer; ++p)
    asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(a.peer_flag[p] + a.peer_rank) : "memory");
  if (a.peer_wait) peer_wait_all(a.peer_flag[a.peer_rank], a.npeer, a.peer_ctrl);
}

// Non-finite x (xrange.cuh): sum of W[row][c] * x'[c] over the kept entries
// of row whose transformed input x'[c] is inf / NaN, c in [c0, c1).
template <int FMT, int SS, bool FUSED>
__device__ __noinline__ float nonfinite_terms(const TiledArgs& a, int row, int tok, int c0, int c1, float inv) {
  TiledRef m{a.vals, a.meta, a.scales, a.zps, a.KQ, a.rt_begin, SS, a.pad14};
  int r = row;
  if (FUSED && a.nseg > 1) {
    const int sg = row / a.rows_s;
    m = TiledRef{a.seg_vals[sg], a.seg_meta[sg], a.seg_scales[sg], a.seg_zps[sg], a.KQ, a.seg_rtb[sg], SS,
                 a.seg_pad14[sg]};
    r = row - sg * a.rows_s;
  }
  const float* xr = a.x + static_cast<size_t>(tok) * a.ldx;
  float add = 0.f;
  for (int c = c0; c < c1; ++c) {
    float xv = xr[c];
    if (FUSED && a.xform == EGT_INPUT_RMSNORM) xv *= inv;
    else if (FUSED && a.xform == EGT_INPUT_SILU) xv = xv * (1.0f / (1.0f + expf(-xv)));
    if ((__float_as_uint(xv) & 0x7fffffffu) < 0x7f800000u) continue;
    float w;
    if (tiled_value<FMT>(m, r, c, &w)) add += w * xv;
  }
  return add;
}

// One token's window staged again with its window scale 2^e (the optimistic
// unscaled staging found the range unsuitable): the window's finite max and
// non-finite flag into s_mx / s_nf (zero on entry), 2^-e into s_unsc, and
// the B fragments of token slot (nt, m): pair (k, k+1) at window offset
// 32 kt + 8 reg + 2 t.
template <bool FUSED>
__device__ __noinline__ void restage_token(const TiledArgs& a, uint32_t* sB, int tok, int nt, int m, int kq0,
                                           int KTc, int LS, float inv, uint32_t* s_mx, uint32_t* s_nf,
                                           float* s_unsc) {
  const float* xr = a.x + static_cast<size_t>(tok) * a.ldx;
  auto xform = [&](float2 q) {
    if (FUSED && a.xform == EGT_INPUT_RMSNORM) {
      q.x *= inv;
      q.y *= inv;
    } else if (FUSED && a.xform == EGT_INPUT_SILU) {
      q = silu2(q);
    }
    return q;
  };
  const int items = KTc * 16;
  uint32_t mx = 0u, nf = 0u;
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int k = kq0 * 128 + i * 2;
    if (k < a.cols) {
      const float2 q = xform(make_float2(xr[k], xr[k + 1]));
      xr_note(mx, nf, q.x);
      xr_note(mx, nf, q.y);
    }
  }
  xr_commit(mx, nf, s_mx, s_nf);
  __syncthreads();
  const int e = xr_exp(*s_mx);
  const float sc = xr_pow2(e);
  if (threadIdx.x == 0) *s_unsc = xr_pow2(-e);
  for (int i = threadIdx.x; i < items; i += blockDim.x) {
    const int reg = i & 3, t = (i >> 2) & 3, kt = i >> 4;
    const int k = (kq0 * 4 + kt) * 32 + 2 * t + 8 * reg;
    float2 q = make_float2(0.f, 0.f);
    if (k < a.cols) q = xform(make_float2(xr[k], xr[k + 1]));
    const float x0 = xr_scaled(q.x, sc), x1 = xr_scaled(q.y, sc);
    const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
    const __half l0 = __float2half_rn(x0 - __half2float(h0)), l1 = __float2half_rn(x1 - __half2float(h1));
    uint32_t* row = sB + static_cast<size_t>(nt * KTc + kt) * LS * 4;
    row[(8 * m + t) * 4 + reg] =
        static_cast<uint32_t>(__half_as_ushort(h0)) | (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
    row[(8 * m + 4 + t) * 4 + reg] =
        static_cast<uint32_t>(__half_as_ushort(l0)) | (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
  }
}

template <int FMT, int SS, int NT, bool SINGLE, bool FUSED>
__global__ void __launch_bounds__(NT == 1 ? 416 : 288, 2) tiled_spmm_kernel(const __grid_constant__ TiledArgs a) {
  constexpr int E = ss_entries(SS);
  constexpr int TOK = 4 * NT;
  constexpr int VB = val_lane_bytes(FMT), MB = meta_lane_bytes(FMT);
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // Programmatic dependent launch.  An independent product lets the next
  // kernel launch at once; a dependent one only after its own inputs are
  // complete (below), so that whenever any product starts, every kernel
  // before its immediate predecessor has finished -- which is what makes
  // EGT_SPMV_INDEPENDENT (inputs not written by the immediate predecessor)
  // safe in a chain of PDL launches.
  if (a.indep) pdl_launch_dependents();
  unsigned long long* tr = a.trace ? a.trace + static_cast<size_t>(a.trace_slot) * 8 : nullptr;
  const bool cta0 = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0;
  if (tr && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    if (cta0) tr[0] = t;
    atomicMax(tr + 5, ~t);
  }
  if (a.dbg == 1) {
    pdl_wait();
    return;
  }

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = (blockDim.x >> 5) - 1;  // consumer warps
  const int rt0 = blockIdx.x * a.RB;
  const int RBc = min(a.RB, a.RT - rt0);
  const int kq0 = blockIdx.y * a.KC;
  const int KCs = min(a.KQ, kq0 + a.KC) - kq0;
  const int KTc = KCs * 4;
  const int m0 = blockIdx.z * TOK;
  const int M_left = a.M - m0;
  const int Mc = min(TOK, M_left);  // tokens of this CTA
  const int sbytes = stage_bytes<FMT>(min(a.CH, KCs), E);
  const int NST = a.NST;

  // shared memory carve-up
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + NST;
  // sB lanes per (n-tile, k-tile): only present tokens (8 per token)
  const int LS = SINGLE ? 8 : 8 * min(4, Mc);
  uint32_t* sB = reinterpret_cast<uint32_t*>(smem_raw + 16 * NST + 128 - (16 * NST) % 128);
  uint8_t* stages = reinterpret_cast<uint8_t*>(sB + NT * KTc * LS * 4);
  float* red = reinterpret_cast<float*>(stages + static_cast<size_t>(NST) * sbytes);  // [RB][nw][Mc][16]
  // per token of the CTA: x window range (xrange.cuh) and the 2^-e rescale
  // (static shared memory is kept minimal: independent launches pack several
  // CTAs per SM, and 128 more bytes per CTA measured -23 % on the sweep)
  constexpr int kTokS = SINGLE ? 1 : TOK;
  __shared__ uint32_t s_xmx[kTokS], s_xnf[kTokS];
  __shared__ float s_unsc[kTokS];
  __shared__ uint32_t s_rng[2];  // several tokens: per-token masks of the optimistic range check

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, nw);
    }
    mbar_fence_init();
  }
  if (tid < 2) s_rng[tid] = 0u;
  if (tid < kTokS) {
    s_xmx[tid] = 0u;
    s_xnf[tid] = 0u;
    s_unsc[tid] = 1.f;
  }
  __syncthreads();

  const uint64_t pol = evict_first_policy();
  const size_t blk_stride = static_cast<size_t>(a.KQ);
  // Work is streamed in chunks q = (row tile i, k-quad chunk c) of CH k-quads:
  // chunk q lands in stage q % NST.
  const int CH = a.CH;
  const int NCH = (KCs + CH - 1) / CH;
  const int NQ = RBc * NCH;
  auto issue = [&](int s, int i, int c) {  // chunk (row tile i, k-quad chunk c) -> stage s
    const int CHc = min(CH, KCs - c * CH);
    uint8_t* st = stages + static_cast<size_t>(s) * sbytes;
    const uint8_t* vals = a.vals;
    const uint8_t* meta = a.meta;
    const float* scales = a.scales;
    const uint8_t* zps = a.zps;
    int rtg = a.rt_begin + rt0 + i;
    if (FUSED && a.nseg > 1) {
      const int g = rt0 + i, sg = g / a.RTs;
      vals = a.seg_vals[sg];
      meta = a.seg_meta[sg];
      scales = a.seg_scales[sg];
      zps = a.seg_zps[sg];
      rtg = a.seg_rtb[sg] + (g - sg * a.RTs);
    }
    const size_t blk = static_cast<size_t>(rtg) * blk_stride + kq0 + c * CH;
    mbar_expect_tx(full + s, stage_bytes<FMT>(CHc, E));
    bulk_g2s(st, vals + blk * 32 * VB, CHc * 32 * VB, full + s, pol);
    if constexpr (MB > 0) bulk_g2s(st + CHc * 32 * VB, meta + blk * 32 * MB, CHc * 32 * MB, full + s, pol);
    if constexpr (has_scales(FMT)) {
      uint8_t* sp = st + CHc * 32 * (VB + MB);
      bulk_g2s(sp, scales + blk * E * 16, CHc * E * 64, full + s, pol);
      bulk_g2s(sp + CHc * E * 64, zps + blk * E * 16, CHc * E * 16, full + s, pol);
    }
  };
  if (warp == nw && lane == 0) {
    int i = 0, c = 0;
    for (int q = 0; q < min(NST, NQ); ++q) {
      issue(q, i, c);
      if (++c == NCH) { c = 0; ++i; }
    }
  }

  // x and the split-K workspace belong to earlier kernels.  An independent
  // product (x not written by the previous kernel) skips the wait here and
  // waits before exiting instead, so stream order stays transitive.
  if (!a.indep) {
    pdl_wait();
    pdl_launch_dependents();
  }
  if (tr && a.dbg == 8) __syncthreads();  // tuning: all warps past the PDL wait before the stamp
  if (tr && cta0) tr[1] = gtimer();
  if (a.dbg == 7) {  // tuning: touch x once (timed into tr[6]) before the real staging
    float acc7 = 0.f;
    for (int k = tid * 4; k < a.cols; k += blockDim.x * 4)
      acc7 += __ldcg(reinterpret_cast<const float4*>(a.x + k)).x;
    if (acc7 == 12345.f) a.y[0] = acc7;
    __syncthreads();
    if (tr && cta0) tr[6] = gtimer();
  }

  const bool bulk_x = false;  // (a TMA bulk copy of x measured slower than these loads)
  constexpr int XU = EGT_XU;
  // rmsnorm (model.cpp:57-67): inv_m = 1 / sqrt(mean(x_m^2) + eps) over the
  // whole row of every token of this CTA, applied while converting
  __shared__ float s_inv[kTokS];
  __shared__ float s_red[FUSED ? 16 : 1];  // rmsnorm: one partial per warp (<= 13 warps)
  // residual rows of this CTA fetched now, not after the compute (decode:
  // the O / ff2 products); one output per thread when the CTA is small
  float res_pre = 0.f;
  if (FUSED && a.res != nullptr && a.S == 1 && tid < RBc * Mc * 16) {
    const int row16 = tid & 15, tl = (tid >> 4) % Mc, i = (tid >> 4) / Mc;
    const int row = (rt0 + i) * 16 + row16;
    if (row < a.rows) res_pre = a.res[static_cast<size_t>(m0 + tl) * a.ldr + row];
  }
  bool staged = false;
  // Optimistic range (xrange.cuh): every staging path converts x unscaled
  // right away and notes, per token slot, whether this thread saw a value
  // >= 2^15 (or inf / NaN) and one >= 2^-9; the barrier that ends staging
  // anyway combines them.  A token keeps scale 1 when its window has no
  // |x| >= 2^15 (no overflow) and some |x| >= 2^-9: every value then splits
  // to within 2^-25 absolute (lo's fp16 subnormal step), i.e. <= 2^-16 of the
  // window max -- below the reference's own f32 rounding vs float64 (~5e-5,
  // SURVEY 0.4).  Any other token is staged again with its 2^e
  // (restage_token).  A separate range pass (or a CTA-wide max) in front of
  // the conversion measured +0.2 us per call, and a 2^-3 threshold sent
  // decode activations (attention outputs ~0.05-0.3) through the restage:
  // x staging is on the critical path.
  uint32_t xbig = 0u, xmid = 0u;  // bit tl: this thread's share of token slot tl
  uint32_t xbits = 0u;            // max |x| bits of the current token's share
  auto note_token = [&](int tl) {
    xbig |= static_cast<uint32_t>(xbits >= 0x47000000u) << tl;
    xmid |= static_cast<uint32_t>(xbits >= 0x3b000000u) << tl;  // 2^-9
    xbits = 0u;
  };
  if constexpr (SINGLE) {
    // One token: each thread loads contiguous float4s of the CTA's x slice
    // (coalesced, trivial addressing) and scatters the two (k, k+1) pairs of
    // each into their B-fragment slots: pair at window offset w of k-tile kt
    // -> reg = w / 8, t = (w % 8) / 2.  rmsnorm's sum of squares comes from
    // the same registers when the slice is the whole row.
    const float* xb = a.x + static_cast<size_t>(m0) * a.ldx + kq0 * 128;
    const int nwin = min(KTc * 32, a.cols - kq0 * 128);  // floats of x in this CTA's window
    const int nf4 = KTc * 8;                             // float4s covering the window (zero past nwin)
    constexpr int X4 = EGT_X4;
    if (a.dbg != 3 && (reinterpret_cast<uintptr_t>(xb) & 15) == 0 && (nwin & 3) == 0 &&
        (!FUSED || a.xform != EGT_INPUT_RMSNORM || (kq0 == 0 && nwin == a.cols))) {
      const int per_pass = X4 * static_cast<int>(blockDim.x);
      float inv = 1.f;
      const bool one_pass = nf4 <= per_pass;
      float4 v[X4];
      if (one_pass) {  // every value in registers up front (rmsnorm reads them twice)
#pragma unroll
        for (int u = 0; u < X4; ++u) {
          const int j = tid + u * static_cast<int>(blockDim.x);
          v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (j < nf4 && 4 * j < nwin) v[u] = __ldg(reinterpret_cast<const float4*>(xb) + j);
        }
      }
      if (FUSED && a.xform == EGT_INPUT_RMSNORM) {
        // the whole row: from the registers when one pass holds it, else a
        // separate sum-of-squares pass
        float ss = 0.f;
        if (one_pass) {
#pragma unroll
          for (int u = 0; u < X4; ++u)
            ss = fmaf(v[u].x, v[u].x, fmaf(v[u].y, v[u].y, fmaf(v[u].z, v[u].z, fmaf(v[u].w, v[u].w, ss))));
        } else {
          for (int j = tid; j < nf4; j += blockDim.x) {
            if (4 * j < nwin) {
              const float4 q = __ldg(reinterpret_cast<const float4*>(xb) + j);
              ss = fmaf(q.x, q.x, fmaf(q.y, q.y, fmaf(q.z, q.z, fmaf(q.w, q.w, ss))));
            }
          }
        }
        ss = warp_sum(ss);
        if (lane == 0) s_red[warp] = ss;
        __syncthreads();
        float tot = 0.f;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += s_red[w];
        inv = 1.0f / sqrtf(tot / static_cast<float>(a.cols) + a.eps);
      }
      auto xform4 = [&](float4 q) {
        if (FUSED && a.xform == EGT_INPUT_RMSNORM) {
          q.x *= inv; q.y *= inv; q.z *= inv; q.w *= inv;
        } else if (FUSED && a.xform == EGT_INPUT_SILU) {
          const float2 q0 = silu2(make_float2(q.x, q.y)), q1 = silu2(make_float2(q.z, q.w));
          q = make_float4(q0.x, q0.y, q1.x, q1.y);
        }
        return q;
      };
      if (tid == 0) s_inv[0] = inv;
      auto pair = [&xbits](float p0, float p1) {
        xbits = max(xbits, max(__float_as_uint(p0) & 0x7fffffffu, __float_as_uint(p1) & 0x7fffffffu));
        const __half h0 = __float2half_rn(p0), h1 = __float2half_rn(p1);
        const __half l0 = __float2half_rn(p0 - __half2float(h0));
        const __half l1 = __float2half_rn(p1 - __half2float(h1));
        return make_uint2(static_cast<uint32_t>(__half_as_ushort(h0)) | (static_cast<uint32_t>(__half_as_ushort(h1)) << 16),
                          static_cast<uint32_t>(__half_as_ushort(l0)) | (static_cast<uint32_t>(__half_as_ushort(l1)) << 16));
      };
      for (int base = 0; base < nf4; base += per_pass) {
        if (!one_pass) {
#pragma unroll
          for (int u = 0; u < X4; ++u) {
            const int j = base + tid + u * static_cast<int>(blockDim.x);
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (j < nf4 && 4 * j < nwin) v[u] = __ldg(reinterpret_cast<const float4*>(xb) + j);
          }
        }
#pragma unroll
        for (int u = 0; u < X4; ++u) {
          const int j = base + tid + u * static_cast<int>(blockDim.x);
          if (j < nf4) {
            const float4 q = xform4(v[u]);
            const int kt = j >> 3, w = (j & 7) * 4, reg = w >> 3, t = (w & 7) >> 1;
            uint32_t* row = sB + static_cast<size_t>(kt) * 32;
            const uint2 a0 = pair(q.x, q.y), a1 = pair(q.z, q.w);
            row[t * 4 + reg] = a0.x;
            row[(4 + t) * 4 + reg] = a0.y;
            row[(t + 1) * 4 + reg] = a1.x;
            row[(5 + t) * 4 + reg] = a1.y;
          }
        }
      }
      note_token(0);
      staged = true;
    }
  }
  if constexpr (FUSED && SINGLE) {
    // one token, whole row in this CTA: a single pass -- the sum of squares
    // comes from the values loaded for the conversion (one L2 round trip)
    const int items = KTc * 16;
    if (!staged && a.xform == EGT_INPUT_RMSNORM && kq0 == 0 && KTc * 32 >= a.cols &&
        items <= XU * static_cast<int>(blockDim.x)) {
      const float* xr = a.x + static_cast<size_t>(m0) * a.ldx;
      float2 v[XU];
      float ss = 0.f;
#pragma unroll
      for (int u = 0; u < XU; ++u) {
        const int i = tid + u * blockDim.x;
        v[u] = make_float2(0.f, 0.f);
        if (i < items) {
          const int k = (i >> 4) * 32 + 2 * ((i >> 2) & 3) + 8 * (i & 3);
          if (k < a.cols)
            v[u] = bulk_x ? reinterpret_cast<const float2*>(sB)[k >> 1] : make_float2(__ldg(xr + k), __ldg(xr + k + 1));
        }
        ss = fmaf(v[u].x, v[u].x, fmaf(v[u].y, v[u].y, ss));
      }
      ss = warp_sum(ss);
      if (lane == 0) s_red[warp] = ss;
      __syncthreads();
      float tot = 0.f;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += s_red[w];
      const float inv = 1.0f / sqrtf(tot / static_cast<float>(a.cols) + a.eps);
      if (tid == 0) s_inv[0] = inv;
#pragma unroll
      for (int u = 0; u < XU; ++u) {
        const int i = tid + u * blockDim.x;
        if (i < items) {
          const int reg = i & 3, t = (i >> 2) & 3, kt = i >> 4;
          const float x0 = v[u].x * inv, x1 = v[u].y * inv;
          xbits = max(xbits, max(__float_as_uint(x0) & 0x7fffffffu, __float_as_uint(x1) & 0x7fffffffu));
          const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
          const __half l0 = __float2half_rn(x0 - __half2float(h0));
          const __half l1 = __float2half_rn(x1 - __half2float(h1));
          uint32_t* row = sB + static_cast<size_t>(kt) * LS * 4;
          row[t * 4 + reg] = static_cast<uint32_t>(__half_as_ushort(h0)) |
                             (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
          row[(4 + t) * 4 + reg] = static_cast<uint32_t>(__half_as_ushort(l0)) |
                                   (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
        }
      }
      note_token(0);
      staged = true;
    }
  }
  if (FUSED && !staged && a.xform == EGT_INPUT_RMSNORM) {
    for (int m = 0; m < Mc; ++m) {
      const float4* xr4 = reinterpret_cast<const float4*>(a.x + static_cast<size_t>(m0 + m) * a.ldx);
      float ss = 0.f;
      for (int i = tid; i < (a.cols >> 2); i += blockDim.x) {
        const float4 w = __ldg(xr4 + i);
        ss = fmaf(w.x, w.x, fmaf(w.y, w.y, fmaf(w.z, w.z, fmaf(w.w, w.w, ss))));
      }
      ss = warp_sum(ss);
      if (lane == 0) s_red[warp] = ss;
      __syncthreads();
      if (tid == 0) {
        float tot = 0.f;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += s_red[w];
        s_inv[m] = 1.0f / sqrtf(tot / static_cast<float>(a.cols) + a.eps);
      }
      __syncthreads();
    }
  }
#pragma unroll
  // Several tokens: the n-tile's (up to 4) tokens are loaded together --
  // every load of a pass in flight at once -- then converted; one token at a
  // time put one L2 round trip per token on the critical path (M = 4: ~4 us
  // of staging per dependent call).
  constexpr int XJ = 4;  // float2 per thread per token per pass
  for (int nt = 0; nt < NT; ++nt) {
    const int mc = (a.dbg == 3 || staged) ? 0 : min(4, Mc - 4 * nt);
    if (mc == 0) continue;
    const int items = KTc * 16;
    float inv[4];
    uint32_t xbm[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int m = 0; m < 4; ++m) inv[m] = FUSED && a.xform == EGT_INPUT_RMSNORM && m < mc ? s_inv[4 * nt + m] : 1.f;
    for (int i0 = 0; i0 < items; i0 += XJ * static_cast<int>(blockDim.x)) {
      float2 v[4][XJ];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const float* xr = a.x + static_cast<size_t>(m0 + 4 * nt + min(m, mc - 1)) * a.ldx;
#pragma unroll
        for (int u = 0; u < XJ; ++u) {
          const int i = i0 + tid + u * static_cast<int>(blockDim.x);
          v[m][u] = make_float2(0.f, 0.f);
          if (m < mc && i < items) {
            const int k = (kq0 * 4 + (i >> 4)) * 32 + 2 * ((i >> 2) & 3) + 8 * (i & 3);
            if (k < a.cols) v[m][u] = make_float2(__ldg(xr + k), __ldg(xr + k + 1));
          }
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        if (m >= mc) break;
#pragma unroll
        for (int u = 0; u < XJ; ++u) {
          const int i = i0 + tid + u * static_cast<int>(blockDim.x);
          if (i < items) {
            const int reg = i & 3, t = (i >> 2) & 3, kt = i >> 4;
            float2 q = v[m][u];
            if (FUSED && a.xform == EGT_INPUT_RMSNORM) {
              q.x *= inv[m];
              q.y *= inv[m];
            } else if (FUSED && a.xform == EGT_INPUT_SILU) {
              q = silu2(q);
            }
            xbm[m] = max(xbm[m], max(__float_as_uint(q.x) & 0x7fffffffu, __float_as_uint(q.y) & 0x7fffffffu));
            const __half h0 = __float2half_rn(q.x), h1 = __float2half_rn(q.y);
            const __half l0 = __float2half_rn(q.x - __half2float(h0));
            const __half l1 = __float2half_rn(q.y - __half2float(h1));
            uint32_t* row = sB + static_cast<size_t>(nt * KTc + kt) * LS * 4;
            row[(8 * m + t) * 4 + reg] = static_cast<uint32_t>(__half_as_ushort(h0)) |
                                         (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
            row[(8 * m + 4 + t) * 4 + reg] = static_cast<uint32_t>(__half_as_ushort(l0)) |
                                             (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
          }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (m < mc) {
        xbits = xbm[m];
        note_token(4 * nt + m);
      }
  }
  // the range check at the end-of-staging barrier (see note_token)
  uint32_t restage = 0u;  // token slots to stage again (CTA-uniform)
  if constexpr (SINGLE) {
    const int any_big = __syncthreads_or(xbig & 1u);
    const int any_mid = __syncthreads_or(xmid & 1u);
    restage = (a.dbg != 3 && (any_big || !any_mid)) ? 1u : 0u;
  } else {
    const uint32_t big = __reduce_or_sync(0xffffffffu, xbig), mid = __reduce_or_sync(0xffffffffu, xmid);
    if (lane == 0 && (big | mid)) {
      atomicOr(s_rng, big);
      atomicOr(s_rng + 1, mid);
    }
    __syncthreads();
    if (a.dbg != 3) restage = (s_rng[0] | ~s_rng[1]) & ((1u << Mc) - 1u);
  }
  if (restage) {
    for (int tl = 0; tl < Mc; ++tl)
      if ((restage >> tl) & 1u)
        restage_token<FUSED>(a, sB, m0 + tl, tl >> 2, tl & 3, kq0, KTc, LS, s_inv[tl], s_xmx + tl, s_xnf + tl,
                             s_unsc + tl);
    __syncthreads();
  }
  if (tr && cta0) tr[2] = gtimer();

  if (warp == nw) {
    // producer: refill each stage once all consumer warps released it
    if (lane == 0) {
      int i = NST / NCH, c = NST - (NST / NCH) * NCH, s = 0;
      uint32_t phase = 0;
      for (int q = NST; q < NQ; ++q) {
        mbar_wait(empty + s, phase);
        issue(s, i, c);
        if (++c == NCH) { c = 0; ++i; }
        if (++s == NST) { s = 0; phase ^= 1u; }
      }
      // after this CTA's own weights are requested: its share of the next
      // product's weights into L2 (behind them in the TMA queue)
      if (a.pf_ptr[0] != nullptr) {
        const uint32_t nb = gridDim.x * gridDim.y * gridDim.z;
        const uint32_t bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t chunk = ((a.pf_bytes[r] + nb - 1) / nb + 15u) & ~15u;
          const uint32_t off = bid * chunk;
          if (a.pf_ptr[r] && off < a.pf_bytes[r]) {
            const uint32_t len = min(chunk, a.pf_bytes[r] - off) & ~15u;
            if (len) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a.pf_ptr[r] + off), "r"(len) : "memory");
          }
        }
      }
    }
  } else {
    const int g = lane >> 2, t = lane & 3;
    int s = 0;
    uint32_t phase = 0;
    for (int i = 0; i < RBc; ++i) {
      float acc[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.f;
      for (int c = 0; c < NCH; ++c) {
        const int CHc = min(CH, KCs - c * CH);
        mbar_wait(full + s, phase);
        const uint8_t* st = stages + static_cast<size_t>(s) * sbytes;
        if (a.dbg != 2 && warp < CHc) {
          Cursor c0 = make_cursor<FMT, E>(st, CHc, warp, lane, sB, (c * CH + warp) * 4, LS);
          int kql = warp;
          for (; kql + nw < CHc; kql += 2 * nw) {  // two independent units in flight
            Cursor c1 = c0;
            advance<FMT, E>(c1, nw, LS);
            Unit<FMT, E> u0, u1;
            lds_unit<FMT, E>(u0, c0);
            lds_unit<FMT, E>(u1, c1);
            compute_unit<FMT, SS, NT>(u0, c0.b, KTc, LS, acc);
            compute_unit<FMT, SS, NT>(u1, c1.b, KTc, LS, acc);
            advance<FMT, E>(c0, 2 * nw, LS);
          }
          if (kql < CHc) {
            Unit<FMT, E> u;
            lds_unit<FMT, E>(u, c0);
            compute_unit<FMT, SS, NT>(u, c0.b, KTc, LS, acc);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
        if (++s == NST) { s = 0; phase ^= 1u; }
      }
      float* r = red + (static_cast<size_t>(i) * nw + warp) * Mc * 16;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        if (4 * nt + t < Mc) {
          r[(4 * nt + t) * 16 + g] = acc[nt][0];
          r[(4 * nt + t) * 16 + g + 8] = acc[nt][1];
        }
    }
  }
  __syncthreads();
  if (tr && cta0) tr[3] = gtimer();

  const int rows_pad = a.RT * 16;
  const int nOut = RBc * Mc * 16;
  for (int idx = tid; idx < nOut; idx += blockDim.x) {
    const int row16 = idx & 15, tl = (idx >> 4) % Mc, i = (idx >> 4) / Mc;
    float v = 0.f;
    for (int w = 0; w < nw; ++w) v += red[((static_cast<size_t>(i) * nw + w) * Mc + tl) * 16 + row16];
    const int row = (rt0 + i) * 16 + row16;
    const int tok = m0 + tl;
    if (row < a.rows) {
      v *= s_unsc[tl];  // undo the window's 2^e (xrange.cuh)
      if (s_xnf[tl]) v += nonfinite_terms<FMT, SS, FUSED>(a, row, tok, kq0 * 128, min(a.cols, (kq0 + KCs) * 128),
                                                         s_inv[tl]);
      if (a.S == 1) {
        float o = (FUSED && a.res ? (idx == tid ? res_pre : a.res[static_cast<size_t>(tok) * a.ldr + row]) : 0.f) + v;
        if (FUSED && a.out_silu) o = o * (1.0f / (1.0f + expf(-o)));  // model.cpp:80-84
        store_out<FUSED>(a, tok, row, o);
      }
      else
        a.partial[(static_cast<size_t>(blockIdx.y) * a.M + tok) * rows_pad + row] = v;
    }
  }
  if (a.S == 1) {
    if (FUSED && a.npeer > 0) peer_complete(a, gridDim.x * gridDim.y * gridDim.z);
    if (a.indep) pdl_wait();
    if (tr && threadIdx.x == 0) atomicMax(tr + 4, gtimer());
    return;
  }

  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  const int cidx = blockIdx.x + gridDim.x * blockIdx.z;
  if (tid == 0) s_last = (atomicAdd(a.counters + cidx, 1u) == static_cast<uint32_t>(a.S - 1));
  __syncthreads();
  if (!s_last) {
    if (a.indep) pdl_wait();
    return;
  }
  __threadfence();
  for (int idx = tid; idx < nOut; idx += blockDim.x) {
    const int row16 = idx & 15, tl = (idx >> 4) % Mc, i = (idx >> 4) / Mc;
    const int row = (rt0 + i) * 16 + row16;
    const int tok = m0 + tl;
    if (row < a.rows) {
      float v = 0.f;
      for (int sidx = 0; sidx < a.S; ++sidx)
        v += __ldcg(a.partial + (static_cast<size_t>(sidx) * a.M + tok) * rows_pad + row);
      float o = (FUSED && a.res ? a.res[static_cast<size_t>(tok) * a.ldr + row] : 0.f) + v;
      if (FUSED && a.out_silu) o = o * (1.0f / (1.0f + expf(-o)));
      store_out<FUSED>(a, tok, row, o);
    }
  }
  if (tid == 0) a.counters[cidx] = 0u;  // ready for the next launch / graph replay
  if (FUSED && a.npeer > 0) peer_complete(a, gridDim.x * gridDim.z);
  if (a.indep) pdl_wait();
}

// ---------------------------------------------------------------- planning

namespace {

template <int FMT, int SS, int NT, bool SINGLE = false>
void* kernel_ptr(bool fused) {
  return fused ? reinterpret_cast<void*>(&tiled_spmm_kernel<FMT, SS, NT, SINGLE, true>)
               : reinterpret_cast<void*>(&tiled_spmm_kernel<FMT, SS, NT, SINGLE, false>);
}

// FUSED: the variant with the input transform / residual code (decode);
// the plain variant keeps the x staging minimal.
template <int FMT, int SS>
void* pick_nt(int NT, bool fused) {  // NT == 0: one token (NT = 1, compile-time B stride)
  switch (NT) {
    case 0: return kernel_ptr<FMT, SS, 1, true>(fused);
    case 1: return kernel_ptr<FMT, SS, 1>(fused);
    case 2: return kernel_ptr<FMT, SS, 2>(fused);
    default: return kernel_ptr<FMT, SS, 4>(fused);
  }
}

template <int FMT>
void* pick_ss(int SS, int NT, bool fused) {
  switch (SS) {
    case 1: return pick_nt<FMT, 1>(NT, fused);
    case 2: return pick_nt<FMT, 2>(NT, fused);
    default: return pick_nt<FMT, 4>(NT, fused);
  }
}

void* pick_kernel(int fmt, int SS, int NT, bool fused) {
  switch (fmt) {
    case I4_SP24: return SS == 0 ? pick_nt<I4_SP24, 0>(NT, fused) : pick_ss<I4_SP24>(SS, NT, fused);
    case I4_SP14: return pick_ss<I4_SP14>(SS, NT, fused);
    case I4_DENSE: return pick_ss<I4_DENSE>(SS, NT, fused);
    case F16_SP24: return pick_nt<F16_SP24, 4>(NT, fused);
    default: return pick_nt<F16_SP14, 4>(NT, fused);
  }
}

int stage_bytes_rt(int fmt, int KCs, int E) {
  return KCs * 32 * (val_lane_bytes(fmt) + meta_lane_bytes(fmt)) + (has_scales(fmt) ? KCs * E * 80 : 0);
}
}  // namespace

// Picks the CTA tile (RB row tiles x KC k-quads), the split-K factor S, the
// stage depth NST and the consumer warp count with a small model of one
// launch: the busiest SM's HBM bytes at its 1/148 share of bandwidth, the
// issue time of the dequant + mma.sp stream per scheduler, the number of
// waves, and a fixed tail for the split-K reduction.
static thread_local int g_force[6] = {0, 0, 0, 0, 0, 0};  // RB, S, nw, NST, on, CH
void force_plan(int RB, int S, int nw, int NST, int CH) {
  g_force[0] = RB;
  g_force[1] = S;
  g_force[2] = nw;
  g_force[3] = NST;
  g_force[4] = RB > 0;
  g_force[5] = CH;
}
bool plan_forced() { return g_force[4] != 0; }

static thread_local bool g_allow_waves = false;  // fallback: several CTAs per SM

TiledSchedule plan_tiled_rt(const egt_dev_packed* h, int RT, int M, int num_sms, bool indep);
TiledSchedule plan_tiled(const egt_dev_packed* h, int M, int num_sms, bool indep) {
  return plan_tiled_rt(h, h->tiled.RT, M, num_sms, indep);
}

TiledSchedule plan_tiled_rt(const egt_dev_packed* h, int RT, int M, int num_sms, bool indep) {
  TiledSchedule best;
  const int KQ = h->tiled.KQ, E = h->tiled.E, f = h->format;
  const int NT = M <= 4 ? 1 : (M <= 8 ? 2 : 4);
  const int NB = (M + 4 * NT - 1) / (4 * NT);
  const int tok = std::min(M, 4 * NT);
  const double unit_b = static_cast<double>(stage_bytes_rt(f, 1, E));
  const double sm_bw = 44.0;             // B/ns per SM (6.5 TB/s / 148)
  const double unit_cycles = 90.0 * NT;  // issue slots per (warp, k-quad unit)
  // <= ~100 KB and <= one CTA per SM: the next kernel's CTAs fit beside this
  // kernel's (programmatic dependent launch) and prefetch their weights.
  static const size_t indep_cap = getenv("EGT_INDEP_SMEM_KB") ? atoi(getenv("EGT_INDEP_SMEM_KB")) * 1024 : 100 * 1024;
  const size_t smem_cap = indep ? indep_cap : 100 * 1024;
  double best_cost = 1e300;
  for (int S = 1; S <= std::min(KQ, g_allow_waves ? 64 : 8); ++S) {
    const int KC = (KQ + S - 1) / S;
    if (S > 1 && (S - 1) * KC >= KQ) continue;
    if (g_force[4] && S != g_force[1]) continue;
    if (indep && S > 1 && !g_force[4]) continue;  // (forced plans: split-K with the alternating workspaces)
    for (int RB = 1; RB <= 128; ++RB) {
      if (g_force[4] && RB != g_force[0]) continue;
      const long grid = static_cast<long>((RT + RB - 1) / RB) * S * NB;
      if (grid > num_sms && RB < 128 && !g_force[4] && !g_allow_waves) continue;  // one CTA per SM
      if (indep && !g_force[4]) {
        // Independent products run several launches side by side on disjoint
        // SMs; measured best (bench sweep, EGT_INDEP_RB_* sweeps) is ~250 KB
        // of weights per CTA plus ~1.6x the CTA's x staging (KB of f32 x),
        // i.e. few CTAs per launch, longer rows per CTA when x is wide:
        // 4096-wide layers 11 row tiles, 11008-wide 5.
        const double total = static_cast<double>(RT) * KQ * unit_b;
        static const double kb0 = getenv("EGT_INDEP_CTA_KB") ? atof(getenv("EGT_INDEP_CTA_KB")) : 250.0;
        static const double kx = getenv("EGT_INDEP_X_W") ? atof(getenv("EGT_INDEP_X_W")) : 1.6;
        const double kb = kb0 + kx * (h->cols * 4.0 / 1024.0);
        const int target = std::max(16, std::min(num_sms, static_cast<int>(total / (kb * 1024) + 0.5)));
        char key[64];  // tuning: EGT_INDEP_RB_<rows>x<cols> forces this shape's row tiles per CTA
        snprintf(key, sizeof key, "EGT_INDEP_RB_%ux%u", h->rows, h->cols);
        const int rb_env = getenv(key) ? atoi(getenv(key)) : 0;
        if (RB != (rb_env > 0 ? rb_env : (RT + target - 1) / target)) continue;
      }
      for (int nw : {4, 8, 12}) {
        if (g_force[4] && g_force[2] > 0 && nw != g_force[2]) continue;
        if (nw > 8 && NT > 1) continue;  // launch bounds: 288 threads when NT > 1
        if (!g_force[4] && nw != 8) continue;
        // chunk: all of the CTA's k-quads if that stage is small, else a
        // multiple of 2*nw k-quads (two units per consumer warp) of ~24 KB
        // chunk: the largest multiple of 2*nw k-quads (two units per consumer
        // warp) that still leaves room for >= 2 stages (measured: whole
        // 4096-column row tiles in 2 stages beat 16-k-quad chunks in 5)
        const size_t red = static_cast<size_t>(RB) * nw * tok * 64;
        const size_t sbx = static_cast<size_t>(NT) * KC * 4 * 32 * std::min(4, tok) * 4;
        const long room = static_cast<long>(smem_cap) - static_cast<long>(sbx + red + 1280);
        int CH = 0;
        for (int want : {2, 1}) {
          for (int ch = (KC + 2 * nw - 1) / (2 * nw) * (2 * nw); ch >= 2 * nw; ch -= 2 * nw) {
            const int chc = std::min(ch, KC);
            const int nq = RB * ((KC + chc - 1) / chc);
            if (room >= static_cast<long>(std::min(want, nq)) * stage_bytes_rt(f, chc, E)) {
              CH = chc;
              break;
            }
          }
          if (CH) break;
        }
        if (!CH) CH = std::min(KC, 2 * nw);
        if (g_force[4] && g_force[5] > 0) CH = std::min(g_force[5], KC);
        const int sb = stage_bytes_rt(f, CH, E);
        const int NQ = RB * ((KC + CH - 1) / CH);
        if (room < sb) continue;
        int nst = std::max(1, std::min<int>(NQ, static_cast<int>(room / sb)));
        if (g_force[4] && g_force[3] > 0) nst = std::min(nst, g_force[3]);
        const size_t smem = (16 * nst + 127) / 128 * 128 + 128 + sbx + static_cast<size_t>(nst) * sb + red;
        if (smem > smem_cap) continue;
        const double ctas_per_sm = std::ceil(static_cast<double>(grid) / num_sms);
        const double bytes_cta = RB * KC * unit_b + KC * 512.0 * tok + (S > 1 ? 2.0 * RB * 64 * tok : 0.0);
        const double t_mem = ctas_per_sm * bytes_cta / sm_bw;
        const double units_per_warp = RB * std::ceil(static_cast<double>(KC) / nw);
        const double t_issue = ctas_per_sm * units_per_warp * unit_cycles * std::max(1.0, nw / 4.0) / 1.9;
        const double t_tail = (S > 1 ? 2500.0 : 0.0) + 0.3 * (t_mem / ctas_per_sm) + (nst < NQ ? 300.0 : 0.0);
        const double cost = std::max(t_mem, t_issue) + t_tail + ctas_per_sm * 600.0;
        if (cost < best_cost * 0.999) {
          best_cost = cost;
          best.RB = RB;
          best.WK = 1;
          best.KC = KC;
          best.S = S;
          best.NT = NT;
          best.NB = NB;
          best.grid_x = (RT + RB - 1) / RB;
          best.grid_y = S;
          best.grid_z = NB;
          best.nw = nw;
          best.NST = nst;
          best.CH = CH;
          best.smem = smem;
        }
      }
    }
  }
  if (best_cost >= 1e300 && g_force[4]) {  // forced plan infeasible: automatic plan
    const int saved = g_force[4];
    g_force[4] = 0;
    best = plan_tiled_rt(h, RT, M, num_sms, indep);
    g_force[4] = saved;
  } else if (best_cost >= 1e300 && indep) {  // no split-free plan fits: dependent plan
    best = plan_tiled_rt(h, RT, M, num_sms, false);
  } else if (best_cost >= 1e300 && !g_allow_waves) {
    // nothing fits in one wave (wide rows x many tokens): allow several waves
    g_allow_waves = true;
    best = plan_tiled_rt(h, RT, M, num_sms, indep);
    g_allow_waves = false;
  }
  return best;
}

size_t tiled_workspace_floats(const egt_dev_packed* h, const TiledSchedule& sc, int M) {
  if (sc.S <= 1) return 0;
  return static_cast<size_t>(sc.S) * M * h->tiled.RT * 16;
}

unsigned long long* tiled_trace_buffer() {
  static unsigned long long* b = [] {
    unsigned long long* p = nullptr;
    if (getenv("EGT_TILED_TRACE")) {
      cudaMalloc(&p, sizeof(unsigned long long) * 8 * 4096);
      cudaMemset(p, 0, sizeof(unsigned long long) * 8 * 4096);
    }
    return p;
  }();
  return b;
}

cudaError_t launch_tiled(const egt_dev_packed* h, const TiledSchedule& sc, const float* x, int ldx,
                         int M, float* y, int ldy, const LaunchCtx& ctx, bool indep) {
  TiledArgs a;
  unsigned long long* trace_buf = tiled_trace_buffer();
  static int trace_next = 0;
  a.trace = trace_buf;
  a.trace_slot = trace_buf ? (trace_next++ % 4096) : 0;
  for (int r = 0; r < 4; ++r) {
    a.pf_ptr[r] = nullptr;
    a.pf_bytes[r] = 0;
  }
  if (const egt_dev_packed* nx = ctx.l2_next; nx && nx->path == EGT_PATH_TILED) {
    const int VB = val_lane_bytes(nx->format), MB = meta_lane_bytes(nx->format);
    const size_t blk0 = static_cast<size_t>(nx->tiled.rt_begin) * nx->tiled.KQ;
    const size_t nblk = static_cast<size_t>(nx->tiled.RT) * nx->tiled.KQ;
    a.pf_ptr[0] = nx->tiled.vals + blk0 * 32 * VB;
    a.pf_bytes[0] = static_cast<uint32_t>(std::min<size_t>(nblk * 32 * VB, 0xFFFFFFF0u));
    if (MB > 0) {
      a.pf_ptr[1] = nx->tiled.meta + blk0 * 32 * MB;
      a.pf_bytes[1] = static_cast<uint32_t>(std::min<size_t>(nblk * 32 * MB, 0xFFFFFFF0u));
    }
    if (has_scales(nx->format)) {
      a.pf_ptr[2] = reinterpret_cast<const uint8_t*>(nx->tiled.scales + blk0 * nx->tiled.E * 16);
      a.pf_bytes[2] = static_cast<uint32_t>(nblk * nx->tiled.E * 64);
      a.pf_ptr[3] = nx->tiled.zps + blk0 * nx->tiled.E * 16;
      a.pf_bytes[3] = static_cast<uint32_t>(nblk * nx->tiled.E * 16);
    }
  }
  a.nseg = 1;
  a.RTs = h->tiled.RT;
  a.rows_s = static_cast<int>(h->rows);
  if (ctx.nseg > 1) {
    a.nseg = ctx.nseg;
    for (int g = 0; g < ctx.nseg; ++g) {
      const egt_dev_packed* hg = ctx.segs[g];
      a.seg_vals[g] = hg->tiled.vals;
      a.seg_meta[g] = hg->tiled.meta;
      a.seg_scales[g] = hg->tiled.scales;
      a.seg_zps[g] = hg->tiled.zps;
      a.seg_y[g] = ctx.seg_y[g];
      a.seg_rtb[g] = hg->tiled.rt_begin;
      a.seg_pad14[g] = hg->tiled.pad14;
    }
  }
  a.pad14 = h->tiled.pad14;
  a.npeer = ctx.npeer;
  a.peer_rank = ctx.peer_rank;
  a.peer_row0 = ctx.peer_row0;
  a.peer_wait = ctx.peer_wait;
  a.peer_ctrl = ctx.peer_ctrl;
  for (int p = 0; p < kMaxPeers; ++p) {
    a.peer_y[p] = p < ctx.npeer ? ctx.peer_y[p] : nullptr;
    a.peer_flag[p] = p < ctx.npeer ? ctx.peer_flag[p] : nullptr;
  }
  a.xform = ctx.xform;
  a.out_silu = ctx.out_silu;
  a.eps = ctx.eps;
  a.res = ctx.res;
  a.ldr = ctx.ldr;
  a.vals = h->tiled.vals;
  a.meta = h->tiled.meta;
  a.scales = h->tiled.scales;
  a.zps = h->tiled.zps;
  a.KQ = h->tiled.KQ;
  a.rt_begin = h->tiled.rt_begin;
  a.RT = h->tiled.RT * std::max(1, ctx.nseg);
  a.rows = static_cast<int>(h->rows) * std::max(1, ctx.nseg);
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
  a.NST = sc.NST;
  a.CH = sc.CH;
  static const int dbg = getenv("EGT_DEBUG_MODE") ? atoi(getenv("EGT_DEBUG_MODE")) : 0;
  a.dbg = dbg;
  a.indep = indep ? 1 : 0;  // split-K workspaces alternate for independent launches (capi.cu)
  static const bool plan_log = getenv("EGT_PLAN_LOG") != nullptr;  // tuning
  if (plan_log)
    fprintf(stderr, "tiled plan %ux%u M=%d: RB=%d S=%d NT=%d nw=%d NST=%d CH=%d grid=(%d,%d,%d) smem=%zu indep=%d\n",
            h->rows, h->cols, M, sc.RB, sc.S, sc.NT, sc.nw, sc.NST, sc.CH, sc.grid_x, sc.grid_y, sc.grid_z, sc.smem,
            indep ? 1 : 0);
  void* fn = pick_kernel(h->format, h->tiled.SS, M == 1 ? 0 : sc.NT, a.xform != 0 || a.res != nullptr || a.pf_ptr[0] || a.out_silu || a.nseg > 1 || a.npeer > 0);
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sc.smem));
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sc.grid_x, sc.grid_y, sc.grid_z);
  cfg.blockDim = dim3(32 * (sc.nw + 1));
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
