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
// Work split: op j's (row tile, k-quad) blocks are linearised panel-major
// (panels of <= 96 k-quads, so a panel's x fits in shared memory) and cut
// into G equal contiguous ranges, one per CTA.  A row tile covered by one CTA
// in a single panel is stored directly; otherwise each covering CTA writes a
// 16-float partial and the last to arrive (per-row-tile counter) sums the
// partials in (panel, CTA) order -- deterministic for a fixed grid.
//
// Ordering: after finishing its share of op j (including any reductions it
// performed) a CTA increments done[j].  Since every CTA processes the ops in
// order, done[j] == G means ops 0..j are complete; op j waits on done[w_j]
// before reading x / the residual.  All CTAs are co-resident (cooperative
// launch, one CTA per SM), spin waits are bounded (trap after 2 s), and the
// last CTA to exit resets the counters for the next launch / graph replay.
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

namespace egt_impl {
void set_last_error(const std::string& msg);

constexpr int kProgPanelMax = 96;  // k-quads per panel: 48 KB of x fragments
constexpr int kProgCH = 16;        // blocks per ring stage (2 per consumer warp)
constexpr int kProgNW = 8;         // consumer warps

struct ProgOp {
  const uint8_t* vals;
  const uint8_t* meta;
  const float* scales;
  const uint8_t* zps;
  const float* x;
  float* y;
  const float* res;
  float* partial;
  uint32_t* cnt;
  long long nblk;
  int fmt, SS, E, KQ, rt_begin, RT, rows, cols;
  int NP, PK, maxp, xform;
  int wait, blk_bytes;
  float eps;
  int pad;
};

struct ProgArgs {
  const ProgOp* ops;
  int n_ops;
  uint32_t* done;  // n_ops op counters + 1 exit counter
  uint32_t* err;
  int NST, stage_bytes, sB_bytes, CH;
};

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

__device__ __forceinline__ long long range_lo_(long long nblk, int c, int G) { return nblk * c / G; }

// Op descriptors are read-only for the launch: fetched once per op through
// the non-coherent path into registers (a reference into global memory would
// be re-read after every mbarrier / barrier asm with a memory clobber).
__device__ __forceinline__ ProgOp load_op(const ProgOp* src) {
  static_assert(sizeof(ProgOp) % 16 == 0, "descriptor is copied in 16-byte pieces");
  ProgOp op;
  const int4* s4 = reinterpret_cast<const int4*>(src);
  int4* d4 = reinterpret_cast<int4*>(&op);
#pragma unroll
  for (int i = 0; i < static_cast<int>(sizeof(ProgOp) / 16); ++i) d4[i] = __ldg(s4 + i);
  return op;
}

// CTAs of [c0, c1] owning at least one block (every CTA does when nblk >= G).
__device__ __forceinline__ bool cta_nonempty(long long nblk, int c, int G) {
  return nblk >= G || range_lo_(nblk, c + 1, G) > range_lo_(nblk, c, G);
}

// Block b of an op -> (panel p, row tile rt, k-quad kq) and its unit (p, rt).
struct BlockPos {
  int p, rt, kq, PKp;
  long long ustart;  // first block of the unit
};
__device__ __forceinline__ BlockPos decode_block(const ProgOp& op, long long b) {
  BlockPos r;
  const long long pb = static_cast<long long>(op.RT) * op.PK;
  r.p = static_cast<int>(min(b / pb, static_cast<long long>(op.NP - 1)));
  const long long off = b - r.p * pb;
  r.PKp = r.p == op.NP - 1 ? op.KQ - (op.NP - 1) * op.PK : op.PK;
  r.rt = static_cast<int>(off / r.PKp);
  r.kq = r.p * op.PK + static_cast<int>(off - static_cast<long long>(r.rt) * r.PKp);
  r.ustart = r.p * pb + static_cast<long long>(r.rt) * r.PKp;
  return r;
}
__device__ __forceinline__ long long range_lo(long long nblk, int c, int G) {
  return nblk * c / G;
}
__device__ __forceinline__ int cta_of(long long nblk, long long b, int G) {
  return static_cast<int>(((b + 1) * G - 1) / nblk);
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

// x panel -> fp16 hi/lo B fragments (SINGLE layout of spmm_tiled.cu: per
// k-tile 8 lanes x 4 u32; lanes t hold hi, 4+t the residual).  Input
// transforms: rmsnorm over the whole vector, or silu.
__device__ void stage_x(const ProgOp& op, int p, uint32_t* sB, float* red_ss, int ctid, int nthr) {
  const int kq0 = p * op.PK;
  const int PKp = p == op.NP - 1 ? op.KQ - kq0 : op.PK;
  const int items = PKp * 4 * 16;
  const float* x = op.x;
  float inv = 1.f;
  if (op.xform == EGT_INPUT_RMSNORM) {
    float ss = 0.f;
    const int n4 = op.cols >> 2;
    for (int i = ctid; i < n4; i += nthr) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(x) + i);
      ss = fmaf(v.x, v.x, ss);
      ss = fmaf(v.y, v.y, ss);
      ss = fmaf(v.z, v.z, ss);
      ss = fmaf(v.w, v.w, ss);
    }
    ss = warp_sum(ss);
    if ((ctid & 31) == 0) red_ss[ctid >> 5] = ss;
    consumer_bar(nthr);
    float tot = 0.f;
    for (int w = 0; w < (nthr >> 5); ++w) tot += red_ss[w];
    inv = 1.0f / sqrtf(tot / static_cast<float>(op.cols) + op.eps);
  }
  constexpr int XU = 8;
  for (int i0 = 0; i0 < items; i0 += XU * nthr) {
    float2 v[XU];
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
      if (i < items) {
        float a = v[u].x, b = v[u].y;
        if (op.xform == EGT_INPUT_RMSNORM) {
          a *= inv;
          b *= inv;
        } else if (op.xform == EGT_INPUT_SILU) {
          a = a * (1.0f / (1.0f + expf(-a)));
          b = b * (1.0f / (1.0f + expf(-b)));
        }
        const int reg = i & 3, t = (i >> 2) & 3, kt = i >> 4;
        const __half h0 = __float2half_rn(a), h1 = __float2half_rn(b);
        const __half l0 = __float2half_rn(a - __half2float(h0));
        const __half l1 = __float2half_rn(b - __half2float(h1));
        uint32_t* row = sB + static_cast<size_t>(kt) * 32;
        row[t * 4 + reg] = static_cast<uint32_t>(__half_as_ushort(h0)) |
                           (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
        row[(4 + t) * 4 + reg] = static_cast<uint32_t>(__half_as_ushort(l0)) |
                                 (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
      }
    }
  }
}

// One chunk of n blocks (k-quads kq .. kq+n of one row tile) in stage st,
// consumed by nw warps (units warp, warp+nw, ...), two units in flight.
template <int FMT, int SS>
__device__ __forceinline__ void consume_chunk(const uint8_t* st, int n, int kt_base, int warp, int nw, int lane,
                                              const uint32_t* sB, float (&acc)[1][2]) {
  constexpr int E = 4 / SS;
  if (warp >= n) return;
  Cursor c0 = make_cursor<FMT, E>(st, n, warp, lane, sB, kt_base + warp * 4, 8);
  int kql = warp;
  for (; kql + nw < n; kql += 2 * nw) {
    Cursor c1 = c0;
    advance<FMT, E>(c1, nw, 8);
    Unit<FMT, E> u0, u1;
    lds_unit<FMT, E>(u0, c0);
    lds_unit<FMT, E>(u1, c1);
    compute_unit<FMT, SS, 1>(u0, c0.b, 0, 8, acc);
    compute_unit<FMT, SS, 1>(u1, c1.b, 0, 8, acc);
    advance<FMT, E>(c0, 2 * nw, 8);
  }
  if (kql < n) {
    Unit<FMT, E> u;
    lds_unit<FMT, E>(u, c0);
    compute_unit<FMT, SS, 1>(u, c0.b, 0, 8, acc);
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

// Warp 0's epilogue of one segment: sum the consumer warps' partial rows, then
// store (unit complete) or publish a partial and reduce if last.
__device__ void segment_epilogue(const ProgOp& op, const BlockPos& bp, bool whole, const float* red, int nw, int lane,
                                 int c, int G) {
  float v = 0.f;
  if (lane < 16)
    for (int w = 0; w < nw; ++w) v += red[w * 16 + lane];
  const int row = bp.rt * 16 + lane;
  if (whole) {
    if (lane < 16 && row < op.rows) op.y[row] = (op.res ? __ldcg(op.res + row) : 0.f) + v;
    return;
  }
  const long long u = static_cast<long long>(bp.p) * op.RT + bp.rt;
  const int piece = c - cta_of(op.nblk, bp.ustart, G);
  if (lane < 16) op.partial[(u * op.maxp + piece) * 16 + lane] = v;
  __threadfence();
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    int expected = 0;
    for (int p = 0; p < op.NP; ++p) {
      const int PKp = p == op.NP - 1 ? op.KQ - (op.NP - 1) * op.PK : op.PK;
      const long long us = static_cast<long long>(p) * op.RT * op.PK + static_cast<long long>(bp.rt) * PKp;
      const int c0 = cta_of(op.nblk, us, G), c1 = cta_of(op.nblk, us + PKp - 1, G);
      for (int cc = c0; cc <= c1; ++cc) expected += cta_nonempty(op.nblk, cc, G) ? 1 : 0;
    }
    last = atomicAdd(op.cnt + bp.rt, 1u) == static_cast<uint32_t>(expected - 1);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  float s = 0.f;
  if (lane < 16) {
    for (int p = 0; p < op.NP; ++p) {
      const int PKp = p == op.NP - 1 ? op.KQ - (op.NP - 1) * op.PK : op.PK;
      const long long us = static_cast<long long>(p) * op.RT * op.PK + static_cast<long long>(bp.rt) * PKp;
      const int c0 = cta_of(op.nblk, us, G), c1 = cta_of(op.nblk, us + PKp - 1, G);
      const long long uu = static_cast<long long>(p) * op.RT + bp.rt;
      for (int k = 0; k <= c1 - c0; ++k)
        if (cta_nonempty(op.nblk, c0 + k, G)) s += __ldcg(op.partial + (uu * op.maxp + k) * 16 + lane);
    }
    if (row < op.rows) op.y[row] = (op.res ? __ldcg(op.res + row) : 0.f) + s;
  }
  if (lane == 0) op.cnt[bp.rt] = 0u;  // ready for the next launch
}

}  // namespace

__global__ void __launch_bounds__(32 * (kProgNW + 1), 1) program_kernel(const ProgArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = (blockDim.x >> 5) - 1;
  const int G = gridDim.x, c = blockIdx.x;
  const int NST = a.NST;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + NST;
  float* red = reinterpret_cast<float*>(smem_raw + ((16 * NST + 127) / 128) * 128);  // [2][nw][16]
  float* red_ss = red + 2 * 16 * kProgNW;                                            // [nw]
  uint32_t* sB = reinterpret_cast<uint32_t*>(red_ss + 32);
  uint8_t* stages = reinterpret_cast<uint8_t*>(sB) + a.sB_bytes;

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, nw);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == nw) {
    // producer: stream every op's block range of this CTA, in program order
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int s = 0;
      uint32_t phase = 0;
      long long q = 0;
      for (int j = 0; j < a.n_ops; ++j) {
        const ProgOp op = load_op(a.ops + j);
        const long long b1 = range_lo(op.nblk, c + 1, G);
        long long b = range_lo(op.nblk, c, G);
        while (b < b1) {
          const BlockPos bp = decode_block(op, b);
          const int n = static_cast<int>(min(min(static_cast<long long>(a.CH), bp.ustart + bp.PKp - b), b1 - b));
          if (q >= NST) mbar_wait(empty + s, phase ^ 1u);
          issue_chunk(op, stages + static_cast<size_t>(s) * a.stage_bytes, full + s, bp.rt, bp.kq, n, pol);
          ++q;
          b += n;
          if (++s == NST) {
            s = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }

  // consumers
  const int nthr = nw * 32;
  int s = 0;
  uint32_t phase = 0;
  int slot = 0;
  // the x fragments in shared memory: (x, transform, panel, PK, KQ) of the
  // op that staged them; any wait invalidates them (x may have been rewritten)
  const float* staged_x = nullptr;
  int staged_p = -1, staged_xf = -1, staged_PK = -1, staged_KQ = -1;
  for (int j = 0; j < a.n_ops; ++j) {
    const ProgOp op = load_op(a.ops + j);
    const long long b0 = range_lo(op.nblk, c, G), b1 = range_lo(op.nblk, c + 1, G);
    if (b0 < b1) {
      if (op.wait >= 0) {
        if (tid == 0) {
          const uint64_t t0 = globaltimer();
          while (ld_acquire(a.done + op.wait) < static_cast<uint32_t>(G)) {
            if (globaltimer() - t0 > 2000000000ull) {
              atomicExch(a.err, 1u);
              __trap();
            }
          }
          __threadfence();
        }
        staged_x = nullptr;  // the other threads pass the restaging barrier after thread 0
      }
      long long b = b0;
      while (b < b1) {
        const BlockPos bp = decode_block(op, b);
        const long long seg_end = min(bp.ustart + bp.PKp, b1);
        const bool whole = op.NP == 1 && b == bp.ustart && seg_end == bp.ustart + bp.PKp;
        if (staged_x != op.x || staged_xf != op.xform || staged_p != bp.p || staged_PK != op.PK ||
            staged_KQ != op.KQ) {
          consumer_bar(nthr);  // every warp is done with the previous fragments
          stage_x(op, bp.p, sB, red_ss, tid, nthr);
          consumer_bar(nthr);
          staged_x = op.x;
          staged_xf = op.xform;
          staged_p = bp.p;
          staged_PK = op.PK;
          staged_KQ = op.KQ;
        }
        float acc[1][2] = {{0.f, 0.f}};
        const int kt_panel0 = bp.p * op.PK * 4;
        for (long long cb = b; cb < seg_end;) {
          const int n = static_cast<int>(min(static_cast<long long>(a.CH), seg_end - cb));
          const int kq = bp.kq + static_cast<int>(cb - b);
          mbar_wait(full + s, phase);
          consume_dispatch(op.fmt, op.SS, stages + static_cast<size_t>(s) * a.stage_bytes, n, kq * 4 - kt_panel0,
                           warp, nw, lane, sB, acc);
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + s);
          if (++s == NST) {
            s = 0;
            phase ^= 1u;
          }
          cb += n;
        }
        // lane (g, t = 0) holds token 0 (B columns 0 = hi, 1 = lo, summed by
        // compute_unit): rows g and g+8 of the row tile
        const float r0 = acc[0][0], r1 = acc[0][1];
        float* rs = red + (slot * kProgNW + warp) * 16;
        if ((lane & 3) == 0) {
          rs[lane >> 2] = r0;
          rs[(lane >> 2) + 8] = r1;
        }
        consumer_bar(nthr);
        if (warp == 0) segment_epilogue(op, bp, whole, red + slot * kProgNW * 16, nw, lane, c, G);
        slot ^= 1;
        b = seg_end;
      }
    }
    if (warp == 0) {
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(a.done + j, 1u);
    }
  }
  // the last CTA out resets the op counters for the next launch
  if (warp == 0 && lane == 0) {
    __threadfence();
    if (atomicAdd(a.done + a.n_ops, 1u) == static_cast<uint32_t>(G - 1)) {
      for (int j = 0; j <= a.n_ops; ++j) a.done[j] = 0u;
      __threadfence();
    }
  }
}

}  // namespace egt_impl

// ---------------------------------------------------------------- host side

struct egt_program {
  int device = 0;
  int G = 0, NST = 0, stage_bytes = 0, sB_bytes = 0, smem = 0;
  uint32_t n_ops = 0;
  bool coop = true;
  std::vector<egt_program_op> ops;
  char* dev = nullptr;  // ops descriptors, counters, partial sums
  egt_impl::ProgOp* d_ops = nullptr;
  uint32_t* d_done = nullptr;
  uint32_t* d_err = nullptr;
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

}  // namespace
}  // namespace egt_impl

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
  std::vector<ProgOp> d(n_ops);
  size_t ws_floats = 0, ws_cnt = 0;
  int max_blk = 0, max_PK = 1;
  for (uint32_t j = 0; j < n_ops; ++j) {
    const egt_program_op& o = ops[j];
    const std::string tag = "program: op " + std::to_string(j) + ": ";
    if (!o.w) return pfail(EGT_EINVAL, tag + "null matrix");
    const egt_dev_packed* h = o.w;
    if (h->path != EGT_PATH_TILED) return pfail(EGT_EINVAL, tag + "matrix is not on the tiled path");
    if (h->rows == 0 || h->cols == 0) return pfail(EGT_EINVAL, tag + "empty matrix");
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
    p.NP = (p.KQ + kProgPanelMax - 1) / kProgPanelMax;
    p.PK = (p.KQ + p.NP - 1) / p.NP;
    p.xform = static_cast<int>(o.input);
    p.eps = o.eps;
    p.wait = o.wait;
    p.blk_bytes = 32 * (val_lane_bytes(p.fmt) + meta_lane_bytes(p.fmt)) + (has_scales(p.fmt) ? p.E * 80 : 0);
    p.nblk = static_cast<long long>(p.RT) * p.KQ;
    // partial slots per unit: the most CTAs any (panel, row tile) spans
    int maxp = 1;
    auto cta = [&](long long b) { return static_cast<int>(((b + 1) * sms - 1) / p.nblk); };
    for (int q = 0; q < p.NP; ++q) {
      const int PKp = q == p.NP - 1 ? p.KQ - (p.NP - 1) * p.PK : p.PK;
      for (int rt = 0; rt < p.RT; ++rt) {
        const long long us = static_cast<long long>(q) * p.RT * p.PK + static_cast<long long>(rt) * PKp;
        maxp = std::max(maxp, cta(us + PKp - 1) - cta(us) + 1);
      }
    }
    p.maxp = maxp;
    ws_floats += al256(static_cast<size_t>(p.NP) * p.RT * maxp * 16 * 4) / 4;
    ws_cnt += al256(static_cast<size_t>(p.RT) * 4) / 4;
    max_blk = std::max(max_blk, p.blk_bytes);
    max_PK = std::max(max_PK, p.PK);
  }
  auto prog = new egt_program();
  prog->device = dev;
  prog->G = sms;
  prog->n_ops = n_ops;
  prog->ops.assign(ops, ops + n_ops);
  prog->coop = getenv("EGT_PROGRAM_NO_COOP") == nullptr;
  prog->sB_bytes = max_PK * 4 * 128;
  prog->stage_bytes = kProgCH * max_blk;
  const int fixed = 2 * 16 * kProgNW * 4 + 32 * 4 + prog->sB_bytes + 128;
  int nst = (smem_optin - fixed - 1024) / (prog->stage_bytes + 16);
  if (const char* e = getenv("EGT_PROGRAM_NST")) nst = std::min(nst, atoi(e));
  if (nst < 2) {
    delete prog;
    return pfail(EGT_EINVAL, "program: shared memory cannot hold two stages");
  }
  prog->NST = nst;
  prog->smem = (16 * nst + 127) / 128 * 128 + fixed + nst * prog->stage_bytes;
  const size_t ops_b = al256(sizeof(ProgOp) * n_ops);
  const size_t done_b = al256(4ull * (n_ops + 2));
  const size_t total = ops_b + done_b + ws_cnt * 4 + ws_floats * 4;
  if (cudaMalloc(&prog->dev, total) != cudaSuccess) {
    delete prog;
    return pfail(EGT_ECUDA, "program: device allocation failed");
  }
  prog->d_ops = reinterpret_cast<ProgOp*>(prog->dev);
  prog->d_done = reinterpret_cast<uint32_t*>(prog->dev + ops_b);
  prog->d_err = prog->d_done + n_ops + 1;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(prog->dev + ops_b + done_b);
  float* part = reinterpret_cast<float*>(cnt + ws_cnt);
  for (uint32_t j = 0; j < n_ops; ++j) {
    d[j].cnt = cnt;
    d[j].partial = part;
    cnt += al256(static_cast<size_t>(d[j].RT) * 4) / 4;
    part += al256(static_cast<size_t>(d[j].NP) * d[j].RT * d[j].maxp * 16 * 4) / 4;
  }
  cudaError_t e = cudaMemsetAsync(prog->dev + ops_b, 0, done_b + ws_cnt * 4, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(prog->d_ops, d.data(), sizeof(ProgOp) * n_ops, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&program_kernel),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, prog->smem);
  if (e != cudaSuccess) {
    cudaFree(prog->dev);
    delete prog;
    return pfail(EGT_ECUDA, std::string("program: setup failed: ") + cudaGetErrorString(e));
  }
  *out = prog;
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
  a.CH = kProgCH;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(prog->G);
  cfg.blockDim = dim3(32 * (kProgNW + 1));
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
  return EGT_OK;
}

egt_status egt_program_destroy(egt_program* prog) {
  if (prog) {
    cudaFree(prog->dev);
    delete prog;
  }
  return EGT_OK;
}

}  // extern "C"
