// Persistent multi-GEMV "program" kernel: one launch streams the weights of
// an ordered list of batch-1 SparseGemv ops (any mix of the tiled formats),
// one CTA per SM, through a single shared-memory ring.
//
// Why: a decode step is a chain of GEMVs of 7-19 MB each (1-3 us at HBM
// speed).  As separate launches every GEMV pays the launch ramp and its tail,
// and a dependent GEMV cannot start streaming until its predecessor's CTAs
// drain.  Here the producer warp of every CTA streams its share of op j+1's
// weights while the consumer warps still wait for op j's output -- weights
// never depend on activations -- so HBM stays busy across op boundaries.
//
// Work split (host-planned, egt_program_create): each CTA owns a contiguous
// range of whole row tiles of every op, so every output row is reduced inside
// one CTA and stored directly.  Ops with too few row tiles to occupy the grid
// are also split along K into S slices (CTA groups); their slice partials are
// summed by the last-arriving slice in slice order (deterministic).  Within a
// CTA the K range is walked in panels of <= 96 k-quads (48 KB of x fragments
// in shared memory), accumulating per row tile across panels.
//
// Warp roles: 1 producer warp (cp.async.bulk into an mbarrier ring),
// kProgNW consumer warps (dequant + mma.sp), 1 epilogue warp (cross-warp sums,
// stores, slice reductions, completion counters) fed through a second
// mbarrier ring, so the compute warps never wait on global-memory round trips.
//
// Ordering: after its share of op j (stores and reductions included) a CTA's
// epilogue warp increments done[j].  Every CTA processes the ops in order, so
// done[j] == G means ops 0..j are complete; op j waits on done[w_j] before
// reading x / the residual.  All CTAs are co-resident (cooperative launch, one
// CTA per SM), spin waits are bounded (trap after 2 s), and the last CTA to
// exit resets the counters for the next launch / graph replay.
//
// Reference: each op is spmv (packed.cpp:211-220) / quant_dense_gemv
// (packed.cpp:266-281); the input transforms are rmsnorm (model.cpp:57-67)
// and silu (model.cpp:80-84) of forward_impl (model.cpp:155-190), the
// residual epilogue is x += t (model.cpp:186,190).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "egt_b200.h"
#include "handle.h"
#include "tiled_compute.cuh"

#ifndef EGT_PROG_NW
#define EGT_PROG_NW 16
#endif

namespace egt_impl {
void set_last_error(const std::string& msg);

constexpr int kProgPanelMax = 96;  // k-quads per panel: 48 KB of x fragments
constexpr int kProgNW = EGT_PROG_NW;   // consumer warps
constexpr int kProgCH = 2 * kProgNW;  // blocks per ring stage (2 per consumer warp)

constexpr int kProgRed = 8;        // consumer -> epilogue ring slots
constexpr int kProgRowsAcc = 128;  // row tiles accumulated across panels at once
constexpr int kProgThreads = 32 * (kProgNW + 2);
constexpr int kProgDesc = 16;     // op descriptor ring slots (shared memory)

// One CTA's share of one op: row tiles [rt_a, rt_b) x k-quads [kq_a, kq_b),
// K slice s of S.
struct ProgItem {
  uint16_t rt_a, rt_b, kq_a, kq_b, s, S, pad0, pad1;
};

struct ProgOp {
  const uint8_t* vals;
  const uint8_t* meta;
  const float* scales;
  const uint8_t* zps;
  const float* x;
  float* y;
  const float* res;
  float* partial;         // S > 1: [RT][S][16]
  uint32_t* cnt;          // S > 1: [RT] arrival counters
  const ProgItem* items;  // [G]
  int fmt, SS, E, KQ, rt_begin, RT, rows, cols;
  int xform, wait, blk_bytes, need_done;
  float eps;
  int pad[3];
};

struct ProgArgs {
  const ProgOp* ops;
  int n_ops;
  uint32_t* done;  // n_ops op counters + 1 exit counter
  uint32_t* err;
  int NST, stage_bytes, sB_bytes, CH, PF;
  int spin;  // which mbarrier waits poll (test_wait) instead of try_wait: 1 full, 2 rempty, 4 empty, 8 rfull
  int dbg;  // tuning experiments: 1 = skip the mma compute, 2 = also skip x staging
  long long* trace;  // tuning: CTA 0 event clocks [4][kTraceN] (producer issue, full, done, epilogue)
};
constexpr int kTraceN = 4096;

namespace {

__device__ __forceinline__ void consumer_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}

// Op descriptors are read-only for the launch: fetched once per op through
// the non-coherent path into registers (a reference into global memory would
// be re-read after every mbarrier / barrier asm with a memory clobber).
template <typename T>
__device__ __forceinline__ T ldg_struct(const T* src) {
  static_assert(sizeof(T) % 16 == 0, "copied in 16-byte pieces");
  T v;
  const int4* s4 = reinterpret_cast<const int4*>(src);
  int4* d4 = reinterpret_cast<int4*>(&v);
#pragma unroll
  for (int i = 0; i < static_cast<int>(sizeof(T) / 16); ++i) d4[i] = __ldg(s4 + i);
  return v;
}

// Panels of a CTA's K range: NP equal pieces of <= kProgPanelMax k-quads.
__device__ __forceinline__ int n_panels(const ProgItem& it) {
  return (it.kq_b - it.kq_a + kProgPanelMax - 1) / kProgPanelMax;
}
__device__ __forceinline__ int panel_lo(const ProgItem& it, int p, int NP) {
  return it.kq_a + (p * (it.kq_b - it.kq_a)) / NP;
}

// Bulk copies of one chunk (n blocks of one row tile, contiguous in storage).
__device__ __forceinline__ void issue_chunk(const ProgOp& op, uint8_t* st, uint64_t* bar, int rt, int kq, int n,
                                            uint64_t pol) {
  const int VB = val_lane_bytes(op.fmt), MB = meta_lane_bytes(op.fmt);
  const size_t blk = static_cast<size_t>(op.rt_begin + rt) * op.KQ + kq;
  mbar_expect_tx(bar, static_cast<uint32_t>(n * op.blk_bytes));
  bulk_g2s(st, op.vals + blk * 32 * VB, n * 32 * VB, bar, pol);
  if (MB > 0) bulk_g2s(st + n * 32 * VB, op.meta + blk * 32 * MB, n * 32 * MB, bar, pol);
  if (has_scales(op.fmt)) {
    uint8_t* sp = st + n * 32 * (VB + MB);
    bulk_g2s(sp, op.scales + blk * op.E * 16, n * op.E * 64, bar, pol);
    bulk_g2s(sp + n * op.E * 64, op.zps + blk * op.E * 16, n * op.E * 16, bar, pol);
  }
}

__device__ __forceinline__ float xform1(float v, int xf, float inv) {
  if (xf == EGT_INPUT_RMSNORM) return v * inv;
  if (xf == EGT_INPUT_SILU) return v * (1.0f / (1.0f + expf(-v)));
  return v;
}

__device__ __forceinline__ void store_frag(uint32_t* sB, int i, float a, float b) {
  const int reg = i & 3, t = (i >> 2) & 3, kt = i >> 4;
  const __half h0 = __float2half_rn(a), h1 = __float2half_rn(b);
  const __half l0 = __float2half_rn(a - __half2float(h0));
  const __half l1 = __float2half_rn(b - __half2float(h1));
  uint32_t* row = sB + static_cast<size_t>(kt) * 32;
  row[t * 4 + reg] = static_cast<uint32_t>(__half_as_ushort(h0)) | (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
  row[(4 + t) * 4 + reg] =
      static_cast<uint32_t>(__half_as_ushort(l0)) | (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
}

// x[k-quads kq0, kq1) -> fp16 hi/lo B fragments (the SINGLE layout of
// spmm_tiled.cu: per k-tile 8 lanes x 4 u32; lane t holds hi, 4+t the
// residual).  Item i covers x[k], x[k+1] with k = kt*32 + 2t + 8reg.  When the
// panel is the whole vector (the usual case) every element is loaded exactly
// once, into registers, and the rmsnorm sum of squares comes from them.
__device__ void stage_x(const ProgOp& op, int kq0, int kq1, uint32_t* sB, float* red_ss, int ctid, int nthr) {
  constexpr int XU = 16;
  const int items = (kq1 - kq0) * 64;
  const float* x = op.x;
  const bool whole = kq0 == 0 && kq1 * 128 >= op.cols && items <= XU * nthr;
  float inv = 1.f;
  float2 v[XU];
  if (op.xform == EGT_INPUT_RMSNORM) {
    float ss = 0.f;
    if (whole) {
#pragma unroll
      for (int u = 0; u < XU; ++u) {
        const int i = ctid + u * nthr;
        v[u] = make_float2(0.f, 0.f);
        if (i < items) {
          const int k = (i >> 4) * 32 + 2 * ((i >> 2) & 3) + 8 * (i & 3);
          if (k < op.cols) v[u] = __ldcg(reinterpret_cast<const float2*>(x + k));
        }
        ss = fmaf(v[u].x, v[u].x, ss);
        ss = fmaf(v[u].y, v[u].y, ss);
      }
    } else {
      for (int i = ctid; i < (op.cols >> 2); i += nthr) {
        const float4 w = __ldcg(reinterpret_cast<const float4*>(x) + i);
        ss = fmaf(w.x, w.x, fmaf(w.y, w.y, fmaf(w.z, w.z, fmaf(w.w, w.w, ss))));
      }
    }
    ss = warp_sum(ss);
    if ((ctid & 31) == 0) red_ss[ctid >> 5] = ss;
    consumer_bar(nthr);
    float tot = 0.f;
    for (int w = 0; w < (nthr >> 5); ++w) tot += red_ss[w];
    inv = 1.0f / sqrtf(tot / static_cast<float>(op.cols) + op.eps);
    if (whole) {
#pragma unroll
      for (int u = 0; u < XU; ++u) {
        const int i = ctid + u * nthr;
        if (i < items) store_frag(sB, i, v[u].x * inv, v[u].y * inv);
      }
      return;
    }
  }
  for (int i0 = 0; i0 < items; i0 += XU * nthr) {
#pragma unroll
    for (int u = 0; u < XU; ++u) {
      const int i = i0 + ctid + u * nthr;
      v[u] = make_float2(0.f, 0.f);
      if (i < items) {
        const int k = (kq0 * 4 + (i >> 4)) * 32 + 2 * ((i >> 2) & 3) + 8 * (i & 3);
        if (k < op.cols) v[u] = __ldcg(reinterpret_cast<const float2*>(x + k));
      }
    }
#pragma unroll
    for (int u = 0; u < XU; ++u) {
      const int i = i0 + ctid + u * nthr;
      if (i < items) store_frag(sB, i, xform1(v[u].x, op.xform, inv), xform1(v[u].y, op.xform, inv));
    }
  }
}

// One chunk of n blocks (k-quads of one row tile) in stage st, consumed by nw
// warps (units warp, warp+nw, ...), two units in flight per warp.
template <int FMT, int SS, int MODE = 0>
__device__ __forceinline__ void consume_chunk(const uint8_t* st, int n, int kt_base, int warp, int nw, int lane,
                                              const uint32_t* sB, float (&acc)[1][2]) {
  constexpr int E = 4 / SS;
  constexpr bool kB = MODE != 4;
  constexpr bool kOnesMma = MODE != 11;
  if (warp >= n) return;
  if constexpr (MODE == 5) {  // tuning experiment: no stage reads
    Unit<FMT, E> u;
#pragma unroll
    for (int i = 0; i < Unit<FMT, E>::NV; ++i) u.v[i] = lane * 0x01010101u + i;
#pragma unroll
    for (int i = 0; i < Unit<FMT, E>::NM; ++i) u.m[i] = 0x44444444u;
#pragma unroll
    for (int i = 0; i < 2 * Unit<FMT, E>::NS; ++i) u.s[i] = 0x3c000000u;
#pragma unroll
    for (int i = 0; i < Unit<FMT, E>::NS; ++i) u.z[i] = 0x0808u;
    const uint32_t* pb = sB + (kt_base + warp * 4) * 32 + (lane & 7) * 4;
    for (int kql = warp; kql < n; kql += nw) {
      compute_unit<FMT, SS, 1>(u, pb, 0, 8, acc);
      pb += nw * 4 * 32;
      u.v[0] += acc[0][0] > 0.f;
    }
    return;
  }
  Cursor c0 = make_cursor<FMT, E>(st, n, warp, lane, sB, kt_base + warp * 4, 8);
  int kql = warp;
  for (; kql + nw < n; kql += 2 * nw) {
    Cursor c1 = c0;
    advance<FMT, E>(c1, nw, 8);
    Unit<FMT, E> u0, u1;
    lds_unit<FMT, E>(u0, c0);
    lds_unit<FMT, E>(u1, c1);
    compute_unit<FMT, SS, 1, kB, kOnesMma>(u0, c0.b, 0, 8, acc);
    compute_unit<FMT, SS, 1, kB, kOnesMma>(u1, c1.b, 0, 8, acc);
    advance<FMT, E>(c0, 2 * nw, 8);
  }
  if (kql < n) {
    Unit<FMT, E> u;
    lds_unit<FMT, E>(u, c0);
    compute_unit<FMT, SS, 1, kB, kOnesMma>(u, c0.b, 0, 8, acc);
  }
}

__device__ __forceinline__ void consume_dispatch(int fmt, int SS, const uint8_t* st, int n, int kt_base, int warp,
                                                 int nw, int lane, const uint32_t* sB, float (&acc)[1][2]) {
  switch (fmt * 8 + SS) {
    case I4_SP24 * 8 + 4: consume_chunk<I4_SP24, 4>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    case I4_SP24 * 8 + 2: consume_chunk<I4_SP24, 2>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    case I4_SP24 * 8 + 1: consume_chunk<I4_SP24, 1>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    case I4_SP14 * 8 + 4: consume_chunk<I4_SP14, 4>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    case I4_SP14 * 8 + 2: consume_chunk<I4_SP14, 2>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    case I4_SP14 * 8 + 1: consume_chunk<I4_SP14, 1>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    case I4_DENSE * 8 + 4: consume_chunk<I4_DENSE, 4>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    case I4_DENSE * 8 + 2: consume_chunk<I4_DENSE, 2>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    case I4_DENSE * 8 + 1: consume_chunk<I4_DENSE, 1>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    case F16_SP24 * 8 + 4: consume_chunk<F16_SP24, 4>(st, n, kt_base, warp, nw, lane, sB, acc); break;
    default: consume_chunk<F16_SP14, 4>(st, n, kt_base, warp, nw, lane, sB, acc); break;
  }
}

// The producer's walk over this CTA's chunks (the iteration order below),
// holding just what a bulk copy needs.  Two cursors run over the same
// sequence: the ring's and an L2-prefetch cursor PF chunks ahead of it.
struct ChunkCursor {
  const uint8_t* vals;
  const uint8_t* meta;
  const float* scales;
  const uint8_t* zps;
  int fmt, E, KQ, rt_begin, blk_bytes;
  int j, NP, r0, r1, p, k0, k1, rt, kq, n;
  ProgItem it;
  bool valid;

  __device__ __forceinline__ void begin() {
    j = -1;
    valid = true;
    rt = r1 = 0;
    p = NP = 0;
    kq = k1 = 0;
    n = 0;
  }
  // advance to the next chunk; false at the end of the program
  __device__ __forceinline__ bool next(const ProgArgs& a, int c, int CH) {
    kq += n;
    while (true) {
      if (kq < k1) {
        n = min(CH, k1 - kq);
        return true;
      }
      if (++rt < r1) {
        kq = k0;
        continue;
      }
      if (++p < NP) {
        k0 = panel_lo(it, p, NP);
        k1 = panel_lo(it, p + 1, NP);
        rt = r0;
        kq = k0;
        continue;
      }
      if (r1 < it.rt_b && j >= 0) {
        r0 = r1;
        r1 = min(static_cast<int>(it.rt_b), r0 + kProgRowsAcc);
        p = -1;
        k1 = kq = 0;
        rt = r1;
        continue;
      }
      // next op with work for this CTA
      do {
        if (++j >= a.n_ops) {
          valid = false;
          return false;
        }
        const ProgOp* o = a.ops + j;
        const ProgItem* items =
            reinterpret_cast<const ProgItem*>(__ldg(reinterpret_cast<const unsigned long long*>(&o->items)));
        it = ldg_struct(items + c);
      } while (it.rt_a >= it.rt_b);
      const ProgOp* o = a.ops + j;
      vals = reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(&o->vals)));
      meta = reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(&o->meta)));
      scales = reinterpret_cast<const float*>(__ldg(reinterpret_cast<const unsigned long long*>(&o->scales)));
      zps = reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(&o->zps)));
      fmt = __ldg(&o->fmt);
      E = __ldg(&o->E);
      KQ = __ldg(&o->KQ);
      rt_begin = __ldg(&o->rt_begin);
      blk_bytes = __ldg(&o->blk_bytes);
      NP = n_panels(it);
      r0 = it.rt_a;
      r1 = min(static_cast<int>(it.rt_b), r0 + kProgRowsAcc);
      p = 0;
      k0 = panel_lo(it, 0, NP);
      k1 = panel_lo(it, 1, NP);
      rt = r0;
      kq = k0;
      n = 0;
    }
  }
  __device__ __forceinline__ size_t blk() const { return static_cast<size_t>(rt_begin + rt) * KQ + kq; }
};

__device__ __forceinline__ void issue_cursor(const ChunkCursor& q, uint8_t* st, uint64_t* bar, uint64_t pol,
                                             int dbg = 0) {
  const int VB = val_lane_bytes(q.fmt), MB = meta_lane_bytes(q.fmt);
  const size_t blk = q.blk();
  if (dbg == 6) {  // tuning experiment: one bulk copy of the chunk's byte count
    mbar_expect_tx(bar, static_cast<uint32_t>(q.n * q.blk_bytes));
    bulk_g2s(st, q.vals + blk * 32 * VB, q.n * q.blk_bytes, bar, pol);
    return;
  }
  mbar_expect_tx(bar, static_cast<uint32_t>(q.n * q.blk_bytes));
  bulk_g2s(st, q.vals + blk * 32 * VB, q.n * 32 * VB, bar, pol);
  if (MB > 0) bulk_g2s(st + q.n * 32 * VB, q.meta + blk * 32 * MB, q.n * 32 * MB, bar, pol);
  if (has_scales(q.fmt)) {
    uint8_t* sp = st + q.n * 32 * (VB + MB);
    bulk_g2s(sp, q.scales + blk * q.E * 16, q.n * q.E * 64, bar, pol);
    bulk_g2s(sp + q.n * q.E * 64, q.zps + blk * q.E * 16, q.n * q.E * 16, bar, pol);
  }
}

__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void prefetch_cursor(const ChunkCursor& q) {
  const int VB = val_lane_bytes(q.fmt), MB = meta_lane_bytes(q.fmt);
  const size_t blk = q.blk();
  prefetch_l2(q.vals + blk * 32 * VB, q.n * 32 * VB);
  if (MB > 0) prefetch_l2(q.meta + blk * 32 * MB, q.n * 32 * MB);
  if (has_scales(q.fmt)) {
    prefetch_l2(q.scales + blk * q.E * 16, q.n * q.E * 64);
    prefetch_l2(q.zps + blk * q.E * 16, q.n * q.E * 16);
  }
}

__device__ __forceinline__ void trap_after(uint64_t t0, uint32_t* err) {
  if (globaltimer() - t0 > 2000000000ull) {
    atomicExch(err, 1u);
    __trap();
  }
}

}  // namespace

// The iteration order shared by all three roles (per op, per CTA):
//   for row-tile block [r0, r1) of <= kProgRowsAcc row tiles of [rt_a, rt_b):
//     for panel p of [kq_a, kq_b):            (consumers restage x if needed)
//       for rt in [r0, r1):                    one segment -> one red slot
//         chunks of <= kProgCH k-quads of (rt, panel p)
__global__ void __launch_bounds__(kProgThreads, 1) program_kernel(const ProgArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int nw = kProgNW;
  const int G = gridDim.x, c = blockIdx.x;
  const int NST = a.NST;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + NST;
  uint64_t* rfull = empty + NST;
  uint64_t* rempty = rfull + kProgRed;
  uint64_t* dfull = rempty + kProgRed;
  uint64_t* dempty = dfull + kProgDesc;
  ProgOp* sdesc = reinterpret_cast<ProgOp*>(smem_raw + ((16 * NST + 16 * kProgRed + 16 * kProgDesc + 127) / 128) * 128);
  ProgItem* sitem = reinterpret_cast<ProgItem*>(sdesc + kProgDesc);
  float* red = reinterpret_cast<float*>(sitem + kProgDesc);  // [R][nw][16]
  float* red_ss = red + kProgRed * nw * 16;         // [32]
  float* acc_s = red_ss + 32;                       // [kProgRowsAcc][16]
  float* res_s = acc_s + kProgRowsAcc * 16;         // [kProgRowsAcc][16] residual rows of the op
  uint32_t* sB = reinterpret_cast<uint32_t*>(res_s + kProgRowsAcc * 16);
  uint8_t* stages = reinterpret_cast<uint8_t*>(sB) + a.sB_bytes;

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, nw);
    }
    for (int s = 0; s < kProgRed; ++s) {
      mbar_init(rfull + s, nw);
      mbar_init(rempty + s, 1);
    }
    for (int s = 0; s < kProgDesc; ++s) {
      mbar_init(dfull + s, 1);
      mbar_init(dempty + s, nw + 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == nw) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int s = 0;
      uint32_t phase = 0;
      long long q = 0;
      ChunkCursor cur, pf;
      cur.begin();
      pf.begin();
      // op descriptors (+ this CTA's item) go into a shared-memory ring for
      // the consumer and epilogue warps, published ahead of their use
      int pub = 0;
      auto publish = [&](int upto) {
        for (; pub <= upto && pub < a.n_ops; ++pub) {
          const int ds = pub % kProgDesc;
          if (pub >= kProgDesc) mbar_wait(dempty + ds, ((pub / kProgDesc) - 1) & 1);
          const ProgOp o = ldg_struct(a.ops + pub);
          sdesc[ds] = o;
          sitem[ds] = ldg_struct(o.items + c);
          mbar_arrive(dfull + ds);
        }
      };
      publish(1);
      // L2 prefetch runs a.PF chunks ahead of the ring: DRAM latency under
      // load is several us, far more than the ring's ~200 KB covers
      for (int i = 0; i < a.PF && pf.next(a, c, a.CH); ++i) prefetch_cursor(pf);
      while (cur.next(a, c, a.CH)) {
        publish(cur.j + 2);
        if (q >= NST) {
          if (a.spin & 4)
            mbar_wait_spin(empty + s, phase ^ 1u);
          else
            mbar_wait(empty + s, phase ^ 1u);
        }
        if (a.trace && c == 0 && q < kTraceN) a.trace[q] = clock64();
        issue_cursor(cur, stages + static_cast<size_t>(s) * a.stage_bytes, full + s, pol, a.dbg);
        if (a.PF > 0 && pf.valid && pf.next(a, c, a.CH)) prefetch_cursor(pf);
        ++q;
        if (++s == NST) {
          s = 0;
          phase ^= 1u;
        }
      }
      publish(a.n_ops - 1);
    }
    return;
  }

  if (warp == nw + 1) {
    // ------------------------------------------------------------ epilogue
    int slot = 0;
    long long qe = 0;
    uint32_t rphase = 0;
    for (int j = 0; j < a.n_ops; ++j) {
      const int ds = j % kProgDesc;
      mbar_wait(dfull + ds, (j / kProgDesc) & 1);
      const ProgOp& op = sdesc[ds];
      const ProgItem it = sitem[ds];
      if (it.rt_a < it.rt_b) {
        const int NP = n_panels(it);
        // residual rows of the first kProgRowsAcc row tiles, fetched in one
        // round trip once the op's inputs are complete (not one dependent
        // load per segment)
        const bool res_pre = op.res != nullptr && it.S == 1;
        if (res_pre) {
          if (op.wait >= 0) {
            if (lane == 0) {
              const uint64_t t0 = globaltimer();
              while (ld_acquire(a.done + op.wait) < static_cast<uint32_t>(G)) trap_after(t0, a.err);
              __threadfence();
            }
            __syncwarp();
          }
          const int n = min(static_cast<int>(it.rt_b - it.rt_a), kProgRowsAcc) * 16;
          const int row0 = it.rt_a * 16;
          for (int i = lane; i < n; i += 32) res_s[i] = row0 + i < op.rows ? __ldcg(op.res + row0 + i) : 0.f;
          __syncwarp();
        }
        for (int r0 = it.rt_a; r0 < it.rt_b; r0 += kProgRowsAcc) {
          const int r1 = min(static_cast<int>(it.rt_b), r0 + kProgRowsAcc);
          for (int p = 0; p < NP; ++p)
            for (int rt = r0; rt < r1; ++rt) {
              if (a.spin & 8)
                mbar_wait_spin(rfull + slot, rphase);
              else
                mbar_wait(rfull + slot, rphase);
              if (a.trace && c == 0 && lane == 0 && qe < kTraceN) a.trace[3 * kTraceN + qe] = clock64();
              ++qe;
              float v = 0.f;
              if (lane < 16) {
                const float* rs = red + slot * nw * 16 + lane;
#pragma unroll
                for (int w = 0; w < nw; ++w) v += rs[w * 16];
              }
              __syncwarp();
              if (lane == 0) mbar_arrive(rempty + slot);
              if (++slot == kProgRed) {
                slot = 0;
                rphase ^= 1u;
              }
              if (NP > 1) {
                float* as = acc_s + (rt - r0) * 16 + lane;
                if (lane < 16) v = p == 0 ? v : *as + v;
                if (p < NP - 1) {
                  if (lane < 16) *as = v;
                  continue;
                }
              }
              const int row = rt * 16 + lane;
              if (lane < 16 && row < op.rows) {
                if (it.S == 1) {
                  float r = 0.f;
                  if (op.res) r = rt - it.rt_a < kProgRowsAcc ? res_s[(rt - it.rt_a) * 16 + lane] : __ldcg(op.res + row);
                  op.y[row] = r + v;
                }
                else
                  op.partial[(static_cast<size_t>(rt) * it.S + it.s) * 16 + lane] = v;
              }
            }
        }
        if (it.S > 1) {
          // slice partials of this CTA's row tiles: one fence, the arrival
          // counters in parallel, then the last slice of a row tile sums all
          // slices in slice order
          __threadfence();
          __syncwarp();
          for (int rb = it.rt_a; rb < it.rt_b; rb += 32) {
            const int rt = rb + lane;
            uint32_t last = 0;
            if (rt < it.rt_b) last = atomicAdd(op.cnt + rt, 1u) == static_cast<uint32_t>(it.S - 1);
            uint32_t mask = __ballot_sync(0xffffffffu, last);
            if (mask) __threadfence();
            while (mask) {
              const int i = __ffs(mask) - 1;
              mask &= mask - 1;
              const int rr = rb + i;
              const int row = rr * 16 + (lane & 15);
              if (lane < 16 && row < op.rows) {
                float s = 0.f;
                for (int k = 0; k < it.S; ++k) s += __ldcg(op.partial + (static_cast<size_t>(rr) * it.S + k) * 16 + lane);
                op.y[row] = (op.res ? __ldcg(op.res + row) : 0.f) + s;
              }
              if (lane == 0) op.cnt[rr] = 0u;  // ready for the next launch
            }
          }
        }
      }
      const int need_done = op.need_done;
      __syncwarp();
      if (lane == 0) mbar_arrive(dempty + ds);
      if (need_done) {
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(a.done + j, 1u);
      }
      if (a.trace && c == 0 && lane == 0 && j < kTraceN) a.trace[7 * kTraceN + j] = clock64();
    }
    // the last CTA out resets the op counters for the next launch
    if (lane == 0) {
      __threadfence();
      if (atomicAdd(a.done + a.n_ops, 1u) == static_cast<uint32_t>(G - 1)) {
        for (int j = 0; j <= a.n_ops; ++j) a.done[j] = 0u;
        __threadfence();
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int nthr = nw * 32;
  int s = 0, slot = 0;
  uint32_t phase = 0, rphase = 0;
  long long qc = 0;  // chunk counter (trace)
  // the x fragments in shared memory: (x, transform, k-quad range) of the
  // op that staged them; a wait invalidates them (x may have been rewritten)
  const float* staged_x = nullptr;
  int staged_xf = -1, staged_k0 = -1, staged_k1 = -1;
  for (int j = 0; j < a.n_ops; ++j) {
    const int ds = j % kProgDesc;
    mbar_wait(dfull + ds, (j / kProgDesc) & 1);
    const ProgOp& op = sdesc[ds];
    const ProgItem it = sitem[ds];
    if (it.rt_a >= it.rt_b) {
      __syncwarp();
      if (lane == 0) mbar_arrive(dempty + ds);
      continue;
    }
    if (a.trace && c == 0 && tid == 0 && j < kTraceN) a.trace[4 * kTraceN + j] = clock64();
    if (op.wait >= 0) {
      if (tid == 0) {
        const uint64_t t0 = globaltimer();
        while (ld_acquire(a.done + op.wait) < static_cast<uint32_t>(G)) trap_after(t0, a.err);
        __threadfence();
        if (a.trace && c == 0 && j < kTraceN) a.trace[5 * kTraceN + j] = clock64();
      }
      staged_x = nullptr;  // the other threads pass the restaging barrier after thread 0
    }
    const int NP = n_panels(it);
    for (int r0 = it.rt_a; r0 < it.rt_b; r0 += kProgRowsAcc) {
      const int r1 = min(static_cast<int>(it.rt_b), r0 + kProgRowsAcc);
      for (int p = 0; p < NP; ++p) {
        const int k0 = panel_lo(it, p, NP), k1 = panel_lo(it, p + 1, NP);
        if (a.dbg < 2 && (staged_x != op.x || staged_xf != op.xform || staged_k0 != k0 || staged_k1 != k1)) {
          consumer_bar(nthr);  // every warp is done with the previous fragments
          stage_x(op, k0, k1, sB, red_ss, tid, nthr);
          consumer_bar(nthr);
          if (a.trace && c == 0 && tid == 0 && j < kTraceN) a.trace[6 * kTraceN + j] = clock64();
          staged_x = op.x;
          staged_xf = op.xform;
          staged_k0 = k0;
          staged_k1 = k1;
        }
        for (int rt = r0; rt < r1; ++rt) {
          float acc[1][2] = {{0.f, 0.f}};
          for (int kq = k0; kq < k1; kq += a.CH) {
            const int n = min(a.CH, k1 - kq);
            if (a.spin & 1)
              mbar_wait_spin(full + s, phase);
            else
              mbar_wait(full + s, phase);
            if (a.trace && c == 0 && tid == 0 && qc < kTraceN) a.trace[kTraceN + qc] = clock64();
            if (a.dbg == 4 && op.fmt == I4_SP24 && op.SS == 4)
              consume_chunk<I4_SP24, 4, 4>(stages + static_cast<size_t>(s) * a.stage_bytes, n, (kq - k0) * 4, warp,
                                           nw, lane, sB, acc);
            else if (a.dbg == 11 && op.fmt == I4_SP24 && op.SS == 4)
              consume_chunk<I4_SP24, 4, 11>(stages + static_cast<size_t>(s) * a.stage_bytes, n, (kq - k0) * 4, warp,
                                            nw, lane, sB, acc);
            else if (a.dbg == 5 && op.fmt == I4_SP24 && op.SS == 4)
              consume_chunk<I4_SP24, 4, 5>(stages + static_cast<size_t>(s) * a.stage_bytes, n, (kq - k0) * 4, warp,
                                           nw, lane, sB, acc);
            else if (a.dbg == 9) {  // tuning experiment: ALU-only busy work of a chunk's length
              float v = acc[0][0] + lane;
              for (int i = 0; i < 2 * 60; ++i) v = fmaf(v, 1.0001f, 0.5f);
              acc[0][0] = v;
            } else if (a.dbg == 10) {  // tuning experiment: LDS-only reads of the stage
              const uint4* sp = reinterpret_cast<const uint4*>(stages + static_cast<size_t>(s) * a.stage_bytes);
              uint32_t t = 0;
              for (int i = warp * 32 + lane; i < n * 53; i += nw * 32) t ^= sp[i].x ^ sp[i].w;
              acc[0][0] += static_cast<float>(t & 1);
            } else if (a.dbg == 0 || a.dbg == 6)
              consume_dispatch(op.fmt, op.SS, stages + static_cast<size_t>(s) * a.stage_bytes, n, (kq - k0) * 4,
                               warp, nw, lane, sB, acc);
            __syncwarp();
            if (a.trace && c == 0 && tid == 0 && qc < kTraceN) a.trace[2 * kTraceN + qc] = clock64();
            ++qc;
            if (lane == 0) mbar_arrive(empty + s);
            if (++s == NST) {
              s = 0;
              phase ^= 1u;
            }
          }
          // lane (g, t = 0) holds token 0 (B columns 0 = hi, 1 = lo, summed by
          // compute_unit): rows g and g+8 of the row tile
          if (a.spin & 2)
            mbar_wait_spin(rempty + slot, rphase ^ 1u);
          else
            mbar_wait(rempty + slot, rphase ^ 1u);
          if ((lane & 3) == 0) {
            float* rs = red + (slot * nw + warp) * 16;
            rs[lane >> 2] = acc[0][0];
            rs[(lane >> 2) + 8] = acc[0][1];
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(rfull + slot);
          if (++slot == kProgRed) {
            slot = 0;
            rphase ^= 1u;
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(dempty + ds);
  }
}

}  // namespace egt_impl

// ---------------------------------------------------------------- host side

struct egt_program {
  int device = 0;
  int G = 0, NST = 0, stage_bytes = 0, sB_bytes = 0, smem = 0, CH = 0;
  uint32_t n_ops = 0;
  bool coop = true;
  double max_load = 0, avg_load = 0;  // bytes per CTA (whole program)
  char* dev = nullptr;  // descriptors, items, counters, partial sums
  egt_impl::ProgOp* d_ops = nullptr;
  uint32_t* d_done = nullptr;
  uint32_t* d_err = nullptr;
  long long* trace = nullptr;  // EGT_PROGRAM_TRACE=1: CTA 0 event clocks
};

namespace egt_impl {
namespace {

egt_status pfail(egt_status s, const std::string& m) {
  set_last_error(m);
  return s;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  if (!a || !b || !na || !nb) return false;
  const char* pa = static_cast<const char*>(a);
  const char* pb = static_cast<const char*>(b);
  return pa < pb + nb && pb < pa + na;
}

size_t al256(size_t v) { return (v + 255) / 256 * 256; }

// K slices for an op with RT row tiles of KQ k-quads on G CTAs.  A slice
// split costs the epilogue warp a fence + atomic round trip + partial reloads
// (several us), so S = 1 unless the row tiles leave most of the grid idle;
// then the S minimising the busiest CTA's blocks, ceil(RT / CTAs per slice)
// x ceil(KQ / S), plus a per-slice penalty.
int choose_slices(int RT, int KQ, int G) {
  if (2 * RT >= G) return 1;
  int best_S = 1;
  double best = 1e300;
  for (int S = 1; S <= std::min({KQ, G, 64}); ++S) {
    const int g_min = G / S;  // smallest group
    const double rows = std::ceil(static_cast<double>(RT) / g_min);
    const double cost = rows * std::ceil(static_cast<double>(KQ) / S) + (S > 1 ? 24.0 + 2.0 * S : 0.0);
    if (cost < best * 0.98) {
      best = cost;
      best_S = S;
    }
  }
  return best_S;
}

// Row-tile ranges of one op: slice s is owned by the CTA group
// [s*G/S, (s+1)*G/S); inside a group the RT row tiles are cut into
// contiguous ranges of q or q+1, the extra ones going to the CTAs with the
// least load so far (balances independent ops over the whole program).
void assign_items(int RT, int KQ, int S, int G, double blk_bytes, std::vector<double>& load,
                  std::vector<ProgItem>& items) {
  items.assign(G, ProgItem{0, 0, 0, 0, 0, 1, 0, 0});
  for (int s = 0; s < S; ++s) {
    const int g0 = static_cast<int>(static_cast<long long>(s) * G / S);
    const int g1 = static_cast<int>(static_cast<long long>(s + 1) * G / S);
    const int n = g1 - g0;
    const int k0 = static_cast<int>(static_cast<long long>(s) * KQ / S);
    const int k1 = static_cast<int>(static_cast<long long>(s + 1) * KQ / S);
    const int q = RT / n, r = RT % n;
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = g0 + i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return load[x] < load[y]; });
    std::vector<int> cnt(n, q);
    for (int i = 0; i < r; ++i) cnt[order[i] - g0] += 1;
    int rt = 0;
    for (int i = 0; i < n; ++i) {
      ProgItem& it = items[g0 + i];
      it.rt_a = static_cast<uint16_t>(rt);
      it.rt_b = static_cast<uint16_t>(rt + cnt[i]);
      it.kq_a = static_cast<uint16_t>(k0);
      it.kq_b = static_cast<uint16_t>(k1);
      it.s = static_cast<uint16_t>(s);
      it.S = static_cast<uint16_t>(S);
      rt += cnt[i];
      load[g0 + i] += cnt[i] * static_cast<double>(k1 - k0) * blk_bytes;
    }
  }
}

}  // namespace
}  // namespace egt_impl

using egt_impl::ProgItem;
using egt_impl::ProgOp;
using egt_impl::pfail;

extern "C" {

egt_status egt_program_create(const egt_program_op* ops, uint32_t n_ops, void* stream, egt_program** out) {
  using namespace egt_impl;
  if (!ops || !out || n_ops == 0) return pfail(EGT_EINVAL, "program: null argument or no ops");
  *out = nullptr;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148, smem_optin = 232448;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (const char* e = getenv("EGT_PROGRAM_GRID")) sms = std::max(1, std::min(sms, atoi(e)));
  const int G = sms;
  std::vector<ProgOp> d(n_ops);
  std::vector<std::vector<ProgItem>> items(n_ops);
  std::vector<double> load(G, 0.0);
  size_t ws_floats = 0, ws_cnt = 0;
  int max_blk = 0, max_panel = 1;
  for (uint32_t j = 0; j < n_ops; ++j) {
    const egt_program_op& o = ops[j];
    const std::string tag = "program: op " + std::to_string(j) + ": ";
    if (!o.w) return pfail(EGT_EINVAL, tag + "null matrix");
    const egt_dev_packed* h = o.w;
    if (h->path != EGT_PATH_TILED) return pfail(EGT_EINVAL, tag + "matrix is not on the tiled path");
    if (h->rows == 0 || h->cols == 0) return pfail(EGT_EINVAL, tag + "empty matrix");
    if (h->tiled.RT > 65535 || h->tiled.KQ > 65535) return pfail(EGT_EINVAL, tag + "matrix too large for a program");
    if (!o.x || !o.y) return pfail(EGT_EINVAL, tag + "null vector");
    if (reinterpret_cast<uintptr_t>(o.x) % 16 != 0) return pfail(EGT_EINVAL, tag + "x must be 16-byte aligned");
    if (o.input > EGT_INPUT_SILU) return pfail(EGT_EINVAL, tag + "unknown input transform");
    if (o.wait >= static_cast<int32_t>(j) || o.wait < -1) return pfail(EGT_EINVAL, tag + "wait must name an earlier op");
    // hazards against every earlier op: RAW (x / residual produced earlier),
    // WAR (this op overwrites an earlier op's input), WAW
    for (uint32_t i = 0; i < j; ++i) {
      const egt_program_op& e = ops[i];
      const size_t xb = 4ull * h->cols, yb = 4ull * h->rows, rb = o.residual ? yb : 0;
      const size_t exb = 4ull * e.w->cols, eyb = 4ull * e.w->rows, erb = e.residual ? eyb : 0;
      const bool raw = overlaps(e.y, eyb, o.x, xb) || overlaps(e.y, eyb, o.residual, rb);
      const bool war = overlaps(e.x, exb, o.y, yb) || overlaps(e.residual, erb, o.y, yb);
      const bool waw = overlaps(e.y, eyb, o.y, yb);
      if ((raw || war || waw) && o.wait < static_cast<int32_t>(i))
        return pfail(EGT_EINVAL, tag + "depends on op " + std::to_string(i) + " but waits on " +
                                     std::to_string(o.wait));
    }
    if (o.residual && o.residual != o.y && overlaps(o.residual, 4ull * h->rows, o.y, 4ull * h->rows))
      return pfail(EGT_EINVAL, tag + "residual partially overlaps y");
    if (overlaps(o.x, 4ull * h->cols, o.y, 4ull * h->rows)) return pfail(EGT_EINVAL, tag + "x overlaps y");
    ProgOp& p = d[j];
    std::memset(&p, 0, sizeof(p));
    p.vals = h->tiled.vals;
    p.meta = h->tiled.meta;
    p.scales = h->tiled.scales;
    p.zps = h->tiled.zps;
    p.x = o.x;
    p.y = o.y;
    p.res = o.residual;
    p.fmt = h->format;
    p.SS = h->tiled.SS;
    p.E = h->tiled.E;
    p.KQ = h->tiled.KQ;
    p.rt_begin = h->tiled.rt_begin;
    p.RT = h->tiled.RT;
    p.rows = static_cast<int>(h->rows);
    p.cols = static_cast<int>(h->cols);
    p.xform = static_cast<int>(o.input);
    p.eps = o.eps;
    p.wait = o.wait;
    p.blk_bytes = 32 * (val_lane_bytes(p.fmt) + meta_lane_bytes(p.fmt)) + (has_scales(p.fmt) ? p.E * 80 : 0);
    const int S = choose_slices(p.RT, p.KQ, G);
    assign_items(p.RT, p.KQ, S, G, p.blk_bytes, load, items[j]);
    for (const ProgItem& it : items[j]) {
      const int len = it.kq_b - it.kq_a;
      if (len > 0) {
        const int NP = (len + kProgPanelMax - 1) / kProgPanelMax;
        max_panel = std::max(max_panel, (len + NP - 1) / NP);
      }
    }
    if (S > 1) {
      ws_floats += al256(static_cast<size_t>(p.RT) * S * 16 * 4) / 4;
      ws_cnt += al256(static_cast<size_t>(p.RT) * 4) / 4;
    }
    max_blk = std::max(max_blk, p.blk_bytes);
  }
  for (uint32_t j = 0; j < n_ops; ++j)
    if (ops[j].wait >= 0) d[ops[j].wait].need_done = 1;
  auto prog = new egt_program();
  prog->device = dev;
  prog->G = G;
  prog->n_ops = n_ops;
  prog->coop = getenv("EGT_PROGRAM_NO_COOP") == nullptr;
  prog->max_load = *std::max_element(load.begin(), load.end());
  double tot = 0;
  for (double v : load) tot += v;
  prog->avg_load = tot / G;
  prog->sB_bytes = max_panel * 4 * 128;
  prog->CH = kProgCH;
  if (const char* e = getenv("EGT_PROGRAM_CH")) prog->CH = std::max(1, atoi(e));
  prog->stage_bytes = prog->CH * max_blk;
  const int bars = (16 * 64 + 16 * kProgRed + 16 * kProgDesc + 127) / 128 * 128;  // room for up to 64 stages
  const int fixed = bars + kProgDesc * static_cast<int>(sizeof(ProgOp) + sizeof(ProgItem)) +
                    (kProgRed * kProgNW * 16 + 32 + 2 * kProgRowsAcc * 16) * 4 + prog->sB_bytes;
  int nst = std::min(64, (smem_optin - fixed) / prog->stage_bytes);
  if (const char* e = getenv("EGT_PROGRAM_NST")) nst = std::min(nst, atoi(e));
  if (nst < 2) {
    delete prog;
    return pfail(EGT_EINVAL, "program: shared memory cannot hold two stages");
  }
  prog->NST = nst;
  prog->smem = (16 * nst + 16 * kProgRed + 16 * kProgDesc + 127) / 128 * 128 + (fixed - bars) + nst * prog->stage_bytes;
  const size_t ops_b = al256(sizeof(ProgOp) * n_ops);
  const size_t items_b = al256(sizeof(ProgItem) * static_cast<size_t>(G) * n_ops);
  const size_t done_b = al256(4ull * (n_ops + 2));
  const size_t total = ops_b + items_b + done_b + ws_cnt * 4 + ws_floats * 4;
  if (cudaMalloc(&prog->dev, total) != cudaSuccess) {
    delete prog;
    return pfail(EGT_ECUDA, "program: device allocation failed");
  }
  prog->d_ops = reinterpret_cast<ProgOp*>(prog->dev);
  ProgItem* d_items = reinterpret_cast<ProgItem*>(prog->dev + ops_b);
  prog->d_done = reinterpret_cast<uint32_t*>(prog->dev + ops_b + items_b);
  prog->d_err = prog->d_done + n_ops + 1;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(prog->dev + ops_b + items_b + done_b);
  float* part = reinterpret_cast<float*>(cnt + ws_cnt);
  std::vector<ProgItem> all(static_cast<size_t>(G) * n_ops);
  for (uint32_t j = 0; j < n_ops; ++j) {
    std::copy(items[j].begin(), items[j].end(), all.begin() + static_cast<size_t>(j) * G);
    d[j].items = d_items + static_cast<size_t>(j) * G;
    const int S = items[j][0].S;
    if (S > 1) {
      d[j].cnt = cnt;
      d[j].partial = part;
      cnt += al256(static_cast<size_t>(d[j].RT) * 4) / 4;
      part += al256(static_cast<size_t>(d[j].RT) * S * 16 * 4) / 4;
    }
  }
  cudaError_t e = cudaMemsetAsync(prog->dev + ops_b + items_b, 0, done_b + ws_cnt * 4, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(prog->d_ops, d.data(), sizeof(ProgOp) * n_ops, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_items, all.data(), sizeof(ProgItem) * all.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&program_kernel),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, prog->smem);
  if (e != cudaSuccess) {
    cudaFree(prog->dev);
    delete prog;
    return pfail(EGT_ECUDA, std::string("program: setup failed: ") + cudaGetErrorString(e));
  }
  if (getenv("EGT_PROGRAM_TRACE")) {
    cudaMalloc(&prog->trace, sizeof(long long) * 8 * egt_impl::kTraceN);
    cudaMemset(prog->trace, 0, sizeof(long long) * 8 * egt_impl::kTraceN);
  }
  *out = prog;
  return EGT_OK;
}

egt_status egt_program_debug_trace(const egt_program* prog, long long* host, size_t n) {
  if (!prog || !prog->trace) return pfail(EGT_EINVAL, "program: tracing is off (EGT_PROGRAM_TRACE)");
  n = std::min<size_t>(n, 8 * egt_impl::kTraceN);
  if (cudaMemcpy(host, prog->trace, n * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return pfail(EGT_ECUDA, "program: trace copy failed");
  return EGT_OK;
}

egt_status egt_program_run(const egt_program* prog, void* stream) {
  using namespace egt_impl;
  if (!prog) return pfail(EGT_EINVAL, "program: null program");
  ProgArgs a;
  a.ops = prog->d_ops;
  a.n_ops = static_cast<int>(prog->n_ops);
  a.done = prog->d_done;
  a.err = prog->d_err;
  a.NST = prog->NST;
  a.stage_bytes = prog->stage_bytes;
  a.sB_bytes = prog->sB_bytes;
  a.CH = prog->CH;
  a.PF = prog->NST;
  a.spin = getenv("EGT_PROGRAM_SPIN") ? atoi(getenv("EGT_PROGRAM_SPIN")) : 0;
  if (const char* e = getenv("EGT_PROGRAM_PF")) a.PF = atoi(e);
  static const int dbg = getenv("EGT_PROGRAM_DEBUG") ? atoi(getenv("EGT_PROGRAM_DEBUG")) : 0;
  a.dbg = dbg;
  a.trace = prog->trace;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(prog->G);
  cfg.blockDim = dim3(kProgThreads);
  cfg.dynamicSmemBytes = prog->smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = prog->coop ? 1 : 0;
  void* args[] = {&a};
  cudaError_t e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(&program_kernel), args);
  if (e != cudaSuccess) return pfail(EGT_ECUDA, std::string("program: launch failed: ") + cudaGetErrorString(e));
  ++launch_counter();
  return EGT_OK;
}

egt_status egt_program_query(const egt_program* prog, egt_program_info* info) {
  if (!prog || !info) return pfail(EGT_EINVAL, "program: null argument");
  info->n_ops = prog->n_ops;
  info->grid = static_cast<uint32_t>(prog->G);
  info->stages = static_cast<uint32_t>(prog->NST);
  info->stage_bytes = static_cast<uint32_t>(prog->stage_bytes);
  info->smem_bytes = static_cast<uint32_t>(prog->smem);
  info->max_cta_bytes = prog->max_load;
  info->avg_cta_bytes = prog->avg_load;
  return EGT_OK;
}

egt_status egt_program_destroy(egt_program* prog) {
  if (prog) {
    cudaFree(prog->dev);
    cudaFree(prog->trace);
    delete prog;
  }
  return EGT_OK;
}

}  // extern "C"
