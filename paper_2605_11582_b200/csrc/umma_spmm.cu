// Many-token SparseGemv on the 5th-generation tensor cores (tcgen05 + TMEM):
// the X * W^T products of the prefix-tree verification pass (forward_impl,
// model.cpp:156-195; M = committed prefix + tree nodes, 64-272 rows in the
// BASELINE configs) for INT4 2:4 (and 1:4 stored as 2:4), dense INT4 and
// FP16 2:4 layers.
//
// One CTA = 128 weight rows x one token tile (T <= 128 tokens) x a K range.
// The accumulator lives in TMEM: D[128 rows x T].  x enters as fp16 hi and
// lo (x - hi) tiles; per K = 16 step two tcgen05.mma (M = 128, N = T) add
// A x_hi and A x_lo into the same accumulator (x keeps ~22 mantissa bits,
// xrange.cuh scales it), so the epilogue reads T columns per scale step --
// TMEM reads (64 B/cycle/SM) are what paces the per-group epilogue.
//
// Warp roles (448 threads, one CTA per SM -- it owns all of TMEM):
//   warp 0      producer: cp.async.bulk of the packed weight blocks (2 k-quads
//               x 8 row tiles per raw stage, issued before the PDL wait:
//               weights never depend on the previous kernel) and of the
//               pre-laid-out x stages (64 K each) into mbarrier rings;
//   warp 1      TMEM allocator + single-thread MMA issuer (4 x K=16 per stage;
//               tcgen05.commit releases the smem stages / signals the epilogue);
//   warps 2-5   dequantisers: packed stage -> the A stage in the UMMA
//               canonical K-major layout (8-row x 16-byte core matrices), the
//               2:4 pairs expanded in place with zeros (c - z exactly in fp16:
//               the 0x6400 exponent trick), then fence.proxy.async;
//   warps 6-13  epilogue: INT4 accumulates one scale step (128 or 64 columns)
//               per TMEM buffer (two buffers, ping-pong) and folds it into
//               registers as acc += s_g * (D_hi + D_lo) -- the reference's
//               (c - z) * s per group, summed in f32; FP16 layers accumulate
//               the whole K range in TMEM and are read once.
// Split-K (S > 1) partials are summed by the last-arriving CTA in slice order
// (deterministic), as in spmm_tiled.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "device_common.cuh"
#include "handle.h"
#include "xrange.cuh"

namespace egt_impl {
using namespace egt_dev;
using namespace egt_fmt;

namespace {

constexpr int kThreads = 448;
constexpr int kDeqWarp0 = 2, kNumDeq = 4, kEpiWarp0 = 6, kNumEpi = 8;
constexpr int kStageK = 64;  // K per A / B stage: four K = 16 MMAs
// k-quads per packed-weight (raw) stage (FP16 blocks are 4.5x larger)
__host__ __device__ constexpr int raw_kq(int fmt) { return fmt == egt_fmt::F16_SP24 ? 1 : 2; }
constexpr int kNA = 3, kNX = 3, kNR = 3;
constexpr int kMaxT = 128;   // tokens per tile (N = 2T <= 256)

struct UmmaArgs {
  const uint8_t* vals;
  const uint8_t* meta;
  const float* scales;
  const uint8_t* zps;
  int KQ, rt_begin, RT, rows, SS, E;
  const uint8_t* xf;  // B stages [tile][k-stage][N rows x 64 K fp16, canonical K-major]
  const float* unsc;  // per padded token: 2^-e (xrange.cuh)
  const uint32_t* nonfin;
  const float* x;  // the raw activations (non-finite fix-up only)
  int ldx, cols;
  int M, T, N;  // tokens, tokens per tile (the MMA's N), N = 2T rows per x stage
  int KS;       // B k-stages of the whole K (2 per k-quad)
  int KQC;      // k-quads per CTA (the split size)
  int S;        // K splits (gridDim.z)
  float* y;
  int ldy;
  const float* res;
  int ldr;
  int out_silu;
  float* partial;
  uint32_t* counters;
  int pad14;
  uint32_t raw_rt_bytes;  // bytes per row tile in a raw stage
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return smem_u32(p); }

// UMMA shared-memory descriptor, K-major, no swizzle: 8-row x 16-byte core
// matrices; lbo = byte stride between core matrices along K, sbo = along M/N.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // version 1 (sm_100)
}

// kind::f16 instruction descriptor: D f32, A/B f16, both K-major, M = 128.
__host__ __device__ constexpr uint32_t umma_idesc(int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// 2:4-sparse A (compressed K: 16 stored of 32 logical per row), metadata in
// TMEM at e_tmem: per 16-row block, lane 16b + g + 8kh holds rows g (bits
// [0,16)) and g + 8 (bits [16,32)) of logical columns [16kh, 16kh + 16),
// a nibble per group of 4 (bits[1:0] first kept index, [3:2] second) -- the
// same words the fragment-tiled stream stores for mma.sp (tiled_format.h).
// The metadata column's low bit goes into the descriptor (sparse id2).
__device__ __forceinline__ void umma_f16_sp(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t e_tmem, uint32_t idesc,
                                            uint32_t acc) {
  const uint32_t id = idesc | (1u << 2) | (e_tmem & 1u);
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n"
      "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(e_tmem & ~1u), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t v0, uint32_t v1) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr), "r"(v0), "r"(v1) : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// 8 consecutive TMEM columns of this warp's 32 lanes (tcgen05.wait::ld before use)
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// c - z for two codes, exact in fp16 (1024 + c minus 1024 + z)
__device__ __forceinline__ uint32_t cz_pair(uint32_t c0, uint32_t c1, uint32_t z) {
  return hsub2_u32((0x6400u | c0) | ((0x6400u | c1) << 16), (0x6400u | z) * 0x00010001u);
}

// 4 fp16 of one group of 4 columns: a at slot o0, b at slot o1, zeros elsewhere
__device__ __forceinline__ uint2 place2(uint32_t ab, uint32_t o0, uint32_t o1) {
  const uint64_t a = ab & 0xFFFFu, b = ab >> 16;
  const uint64_t w = (a << (16 * o0)) | (b << (16 * o1));
  return make_uint2(static_cast<uint32_t>(w), static_cast<uint32_t>(w >> 32));
}

__device__ __forceinline__ void st_shared_v2(uint32_t addr, uint2 v) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};\n" ::"r"(addr), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void st_shared_b32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// A-operand byte offset of (row r, column k) in a 128 x 64 stage
__device__ __forceinline__ uint32_t a_off(int r, int k) {
  return static_cast<uint32_t>((k >> 3) * 2048 + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

template <int FMT>
__device__ __noinline__ float umma_nonfinite_terms(const UmmaArgs& a, int row, int tok, int c0, int c1) {
  const TiledRef m{a.vals, a.meta, a.scales, a.zps, a.KQ, a.rt_begin, a.SS, a.pad14};
  const float* xr = a.x + static_cast<size_t>(tok) * a.ldx;
  float add = 0.f;
  for (int c = c0; c < c1; ++c) {
    const float xv = xr[c];
    if ((__float_as_uint(xv) & 0x7fffffffu) < 0x7f800000u) continue;
    float w;
    if (tiled_value<FMT>(m, row, c, &w)) add += w * xv;
  }
  return add;
}

template <int FMT, bool SPARSE>
__global__ void __launch_bounds__(kThreads, 1) umma_spmm_kernel(const UmmaArgs a) {
  static_assert(!SPARSE || FMT != I4_DENSE, "dense INT4 has no 2:4 metadata");
  constexpr bool kScaled = has_scales(FMT);
  constexpr int kRawKQ = raw_kq(FMT);
  constexpr int VB = val_lane_bytes(FMT), MB = meta_lane_bytes(FMT);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rt0 = blockIdx.x * 8;  // first 16-row tile of this CTA (128 rows)
  const int tile = blockIdx.y;     // token tile
  const int kq0 = blockIdx.z * a.KQC;
  const int KQC = min(a.KQC, a.KQ - kq0);
  const int NSTG = 2 * KQC;                     // A / B stages of this CTA
  const int NRAW = (KQC + kRawKQ - 1) / kRawKQ;  // raw stages
  const int T = a.T, N = a.N;
  const int steps_per_scale = kScaled ? a.SS / 2 : NSTG;  // stages per accumulation round
  const int NROUND = kScaled ? NSTG / steps_per_scale : 1;

  // ---- shared memory carve-up
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = raw_full + kNR;
  uint64_t* a_full = raw_empty + kNR;
  uint64_t* a_empty = a_full + kNA;
  uint64_t* x_full = a_empty + kNA;
  uint64_t* x_empty = x_full + kNX;
  uint64_t* tm_full = x_empty + kNX;
  uint64_t* tm_empty = tm_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tm_empty + 2);
  __shared__ int s_last;
  uint8_t* a_st = smem_raw + 1024;                                   // kNA x 16 KB
  uint8_t* x_st = a_st + kNA * 16384;                                // kNX x (N x 128 B)
  const uint32_t x_bytes = static_cast<uint32_t>(N) * kStageK * 2;
  uint8_t* raw_st = x_st + kNX * x_bytes;                            // kNR x (8 x raw_rt_bytes)
  const uint32_t raw_bytes = 8 * a.raw_rt_bytes;

  if (tid == 0) {
    for (int i = 0; i < kNR; ++i) {
      mbar_init(raw_full + i, 1);
      mbar_init(raw_empty + i, kNumDeq);
    }
    for (int i = 0; i < kNA; ++i) {
      mbar_init(a_full + i, kNumDeq);
      mbar_init(a_empty + i, 1);
    }
    for (int i = 0; i < kNX; ++i) {
      mbar_init(x_full + i, 1);
      mbar_init(x_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tm_full + i, 1);
      mbar_init(tm_empty + i, kNumEpi);
    }
    mbar_fence_init();
  }
  // TMEM: accumulator buffer(s) at column 0, sparse metadata (2 columns per
  // A stage ring slot) at column 256
  constexpr uint32_t kMetaCol = 256;
  const uint32_t tmem_cols = SPARSE ? 512u : ((kScaled ? 2 * T : T) <= 128 ? 128u : 256u);
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(tmem_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= producer
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      auto issue_raw = [&](int rs) {
        const int s = rs % kNR;
        if (rs >= kNR) mbar_wait(raw_empty + s, ((rs / kNR) - 1) & 1);
        const int kq = kq0 + rs * kRawKQ, nq = min(kRawKQ, kq0 + KQC - kq);
        uint32_t bytes = 0;
        uint8_t* dst0 = raw_st + s * raw_bytes;
        // values, metadata and zero points (the epilogue reads the scales itself)
        const uint32_t vb = nq * 32 * VB, mbb = nq * 32 * MB, zb = kScaled ? nq * a.E * 16 : 0;
        for (int i = 0; i < 8; ++i)
          if (rt0 + i < a.RT) bytes += vb + mbb + zb;
        mbar_expect_tx(raw_full + s, bytes);
        for (int i = 0; i < 8; ++i) {
          if (rt0 + i >= a.RT) continue;
          const size_t blk = static_cast<size_t>(a.rt_begin + rt0 + i) * a.KQ + kq;
          uint8_t* dst = dst0 + i * a.raw_rt_bytes;
          bulk_g2s(dst, a.vals + blk * 32 * VB, vb, raw_full + s, pol);
          if (MB > 0) bulk_g2s(dst + kRawKQ * 32 * VB, a.meta + blk * 32 * MB, mbb, raw_full + s, pol);
          if (kScaled) bulk_g2s(dst + kRawKQ * 32 * (VB + MB), a.zps + blk * a.E * 16, zb, raw_full + s, pol);
        }
      };
      int rs_next = 0;
      for (; rs_next < min(kNR, NRAW); ++rs_next) issue_raw(rs_next);  // before the PDL wait
      pdl_wait();  // x stages come from the preceding xprep kernel
      for (int st = 0; st < NSTG; ++st) {
        if (st % (2 * kRawKQ) == 0 && st / (2 * kRawKQ) >= rs_next && rs_next < NRAW) issue_raw(rs_next++);
        const int s = st % kNX;
        if (st >= kNX) mbar_wait(x_empty + s, ((st / kNX) - 1) & 1);
        mbar_expect_tx(x_full + s, x_bytes);
        const uint8_t* src = a.xf + (static_cast<size_t>(tile) * a.KS + 2 * kq0 + st) * x_bytes;
        bulk_g2s_plain(x_st + s * x_bytes, src, x_bytes, x_full + s);
        // keep the weight ring ahead of the x ring
        while (rs_next < NRAW && rs_next * 2 * kRawKQ <= st + kNX) issue_raw(rs_next++);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(T);
      const uint32_t lbo_b = static_cast<uint32_t>(N / 8) * 128;  // x stage: hi rows [0, T), lo rows [T, 2T)
      const uint32_t lo_off = static_cast<uint32_t>(T / 8) * 128;
      for (int st = 0; st < NSTG; ++st) {
        const int round = st / steps_per_scale, first = st % steps_per_scale == 0;
        const int buf = kScaled ? (round & 1) : 0;
        if (kScaled && first && round >= 2) mbar_wait(tm_empty + buf, ((round / 2) - 1) & 1);
        mbar_wait(a_full + st % kNA, (st / kNA) & 1);
        mbar_wait(x_full + st % kNX, (st / kNX) & 1);
        tc_fence_after();
        const uint32_t abase = smem_addr(a_st + (st % kNA) * 16384);
        const uint32_t bbase = smem_addr(x_st + (st % kNX) * x_bytes);
        const uint32_t d = tmem + static_cast<uint32_t>(buf * T);
        if constexpr (SPARSE) {  // two K = 32 (logical) sparse MMAs per stage, x hi and lo
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const uint64_t ad = umma_desc(abase + jj * 2 * 2048, 2048, 128);
            const uint32_t e = tmem + kMetaCol + static_cast<uint32_t>(2 * (st % kNA) + jj);
            umma_f16_sp(d, ad, umma_desc(bbase + jj * 4 * lbo_b, lbo_b, 128), e, idesc,
                        (first && jj == 0) ? 0u : 1u);
            umma_f16_sp(d, ad, umma_desc(bbase + lo_off + jj * 4 * lbo_b, lbo_b, 128), e, idesc, 1u);
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = umma_desc(abase + kk * 2 * 2048, 2048, 128);
            umma_f16(d, ad, umma_desc(bbase + kk * 2 * lbo_b, lbo_b, 128), idesc, (first && kk == 0) ? 0u : 1u);
            umma_f16(d, ad, umma_desc(bbase + lo_off + kk * 2 * lbo_b, lbo_b, 128), idesc, 1u);
          }
        }
        umma_commit(a_empty + st % kNA);
        umma_commit(x_empty + st % kNX);
        if ((st + 1) % steps_per_scale == 0 || st + 1 == NSTG) umma_commit(tm_full + buf);
      }
    }
  } else if (warp < kEpiWarp0) {
    // ================= dequantisers: raw stage -> A stage
    // warp w writes TMEM lanes [32 (w % 4), +32) (the tcgen05.st lane rule):
    // its row tiles are 2 (w % 4) and 2 (w % 4) + 1
    const int dq = warp & 3;
    const int g = lane >> 2, t = lane & 3;
    for (int st = 0; st < NSTG; ++st) {
      const int sa = st % kNA;
      if (st >= kNA) mbar_wait(a_empty + sa, ((st / kNA) - 1) & 1);
      const int kql = st >> 1, hs = st & 1;
      const int rs = kql / kRawKQ, b = kql % kRawKQ;
      mbar_wait(raw_full + rs % kNR, (rs / kNR) & 1);
      const uint8_t* rstage = raw_st + (rs % kNR) * raw_bytes;
      const uint32_t abase = smem_addr(a_st + sa * 16384);
      for (int ii = 0; ii < 2; ++ii) {
        const int i = 2 * dq + ii;  // row tile within the CTA
        if (rt0 + i >= a.RT) {      // past the matrix: zero rows
          for (int w = lane; w < 16 * 64 * 2 / 16; w += 32) {
            const int r = i * 16 + (w & 15), ch = w >> 4;
            st_shared_v4(abase + ch * 2048 + (r >> 3) * 128 + (r & 7) * 16, make_uint4(0, 0, 0, 0));
          }
          continue;
        }
        const uint8_t* rt_base = rstage + i * a.raw_rt_bytes;
        const uint32_t* v = reinterpret_cast<const uint32_t*>(rt_base + (b * 32 + lane) * VB);
        const uint32_t* mb = reinterpret_cast<const uint32_t*>(rt_base + kRawKQ * 32 * VB + b * 32 * MB);
        const uint8_t* zp = rt_base + kRawKQ * 32 * (VB + MB) + b * a.E * 16;
        if constexpr (FMT == I4_DENSE) {
#pragma unroll
          for (int w4 = 0; w4 < 4; ++w4) {
            const int w16 = 4 * hs + w4;
            const uint32_t word = v[w16];
            const int e = (w16 >> 1) / a.SS;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t z = zp[e * 16 + 2 * g + h];
              const int r = i * 16 + g + 8 * h;
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int p = h + 2 * q;
                const uint32_t pr = cz_pair((word >> (4 * p)) & 0xFu, (word >> (16 + 4 * p)) & 0xFu, z);
                st_shared_b32(abase + a_off(r, 16 * w4 + 2 * t + 8 * q), pr);
              }
            }
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int j = 2 * hs + jj;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t mw = mb[(4 * g + 2 * (j & 1) + q) * 2 + (j >> 1)];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint32_t nib = (mw >> (16 * h + 4 * t)) & 0xFu;
                uint32_t pr;
                if constexpr (FMT == I4_SP24) {
                  const int p = h + 2 * q;
                  const uint32_t z = zp[(j / a.SS) * 16 + 2 * g + h];
                  pr = cz_pair((v[j] >> (4 * p)) & 0xFu, (v[j] >> (16 + 4 * p)) & 0xFu, z);
                } else {  // F16_SP24: the two kept fp16 values
                  pr = v[4 * j + h + 2 * q];
                }
                const int r = i * 16 + g + 8 * h, G = t + 4 * q;
                if constexpr (SPARSE)  // the kept pair, compressed K: groups of 4 -> 2 slots
                  st_shared_b32(abase + a_off(r, jj * 16 + 2 * G), pr);
                else
                  st_shared_v2(abase + a_off(r, jj * 32 + 4 * G), place2(pr, nib & 3u, nib >> 2));
              }
            }
          }
        }
      }
      if constexpr (SPARSE) {
        // metadata of this stage's two sparse MMAs -> TMEM lanes [32 dq, +32)
        const int ti = 2 * dq + (lane >> 4), l16 = lane & 15, gg = l16 & 7, kh = l16 >> 3;
        uint32_t w[2] = {0x44444444u, 0x44444444u};  // (0,1) pattern for rows past the matrix
        if (rt0 + ti < a.RT) {
          const uint32_t* mbt = reinterpret_cast<const uint32_t*>(rstage + ti * a.raw_rt_bytes + kRawKQ * 32 * VB +
                                                                  b * 32 * MB);
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int j = 2 * hs + jj;
            w[jj] = mbt[(4 * gg + 2 * (j & 1) + kh) * 2 + (j >> 1)];
          }
        }
        tmem_st2(tmem + (static_cast<uint32_t>(32 * dq) << 16) + kMetaCol + 2 * sa, w[0], w[1]);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
      }
      fence_async_smem();  // generic-proxy writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(a_full + sa);
        if (hs == 1 && (b == kRawKQ - 1 || kql == KQC - 1)) mbar_arrive(raw_empty + rs % kNR);
      }
    }
  } else {
    // ================= epilogue: TMEM -> registers
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2;
    const int r = 32 * q + lane;  // accumulator row = TMEM lane
    const int grow = rt0 * 16 + r;
    const int th = T / 2, c0 = half * th;  // this thread's token columns [c0, c0 + th)
    float acc[kMaxT / 2];
#pragma unroll
    for (int i = 0; i < kMaxT / 2; ++i) acc[i] = 0.f;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * q) << 16);
    const bool row_ok = grow < a.rows && (rt0 + (r >> 4)) < a.RT;
    for (int round = 0; round < NROUND; ++round) {
      const int buf = kScaled ? (round & 1) : 0;
      float s = 1.f;
      if (kScaled && row_ok) {  // the row's scale of this round's column group
        const int kql = (round * steps_per_scale) / 2;
        const int e = ((round * steps_per_scale) % 2) * 2 / a.SS;
        const size_t blk = static_cast<size_t>(a.rt_begin + rt0 + (r >> 4)) * a.KQ + kq0 + kql;
        s = __ldg(a.scales + (blk * a.E + e) * 16 + 2 * (r & 7) + ((r >> 3) & 1));
      }
      mbar_wait(tm_full + buf, kScaled ? ((round >> 1) & 1) : 0);
      tc_fence_after();
      // batches of up to 32 columns: every load in flight, then one wait
#pragma unroll
      for (int bb = 0; bb < kMaxT / 2; bb += 32) {
        if (bb < th) {
          uint32_t v[32];
#pragma unroll
          for (int cb = 0; cb < 4; ++cb)
            if (bb + cb * 8 < th) tmem_ld8_nowait(lane_base + static_cast<uint32_t>(buf * T + c0 + bb + cb * 8), v + cb * 8);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (bb + i < th) acc[bb + i] = fmaf(s, __uint_as_float(v[i]), acc[bb + i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (kScaled && lane == 0) mbar_arrive(tm_empty + buf);
    }
    // ---- outputs: rescale (xrange.cuh), fix-up, residual / silu or partials
    pdl_wait();  // residual rows / x scales belong to earlier kernels
    const int kc0 = kq0 * 128, kc1 = min(a.cols, (kq0 + KQC) * 128);
    if (row_ok) {
#pragma unroll
      for (int i = 0; i < kMaxT / 2; ++i) {
        if (i < th) {
          const int tok = tile * T + c0 + i;
          if (tok < a.M) {
            float v = acc[i] * a.unsc[tok];
            if (a.nonfin[tok]) v += umma_nonfinite_terms<FMT>(a, grow, tok, kc0, kc1);
            if (a.S == 1) {
              float o = (a.res ? a.res[static_cast<size_t>(tok) * a.ldr + grow] : 0.f) + v;
              if (a.out_silu) o = o * (1.0f / (1.0f + expf(-o)));  // model.cpp:80-84
              a.y[static_cast<size_t>(tok) * a.ldy + grow] = o;
            } else {
              a.partial[(static_cast<size_t>(blockIdx.z) * a.M + tok) * a.rows + grow] = v;
            }
          }
        }
      }
    }
  }

  // ---- teardown: TMEM back, then the split-K reduction by the last CTA
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tmem_cols) : "memory");
  pdl_launch_dependents();
  if (a.S == 1) return;
  __threadfence();
  __syncthreads();
  const int cidx = blockIdx.x + gridDim.x * blockIdx.y;
  if (tid == 0) s_last = atomicAdd(a.counters + cidx, 1u) == static_cast<uint32_t>(a.S - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int rows_here = min(128, a.rows - rt0 * 16);
  const int toks_here = min(T, a.M - tile * T);
  for (int idx = tid; idx < rows_here * toks_here; idx += blockDim.x) {
    const int rr = idx % rows_here, tt = idx / rows_here;
    const int grow = rt0 * 16 + rr, tok = tile * T + tt;
    float v = 0.f;
    for (int z = 0; z < a.S; ++z) v += __ldcg(a.partial + (static_cast<size_t>(z) * a.M + tok) * a.rows + grow);
    float o = (a.res ? a.res[static_cast<size_t>(tok) * a.ldr + grow] : 0.f) + v;
    if (a.out_silu) o = o * (1.0f / (1.0f + expf(-o)));
    a.y[static_cast<size_t>(tok) * a.ldy + grow] = o;
  }
  if (tid == 0) a.counters[cidx] = 0u;  // ready for the next launch / graph replay
}

// X [M x cols] -> B stages: per token tile, per 64-column k-stage, N = 2T rows
// (row n < T: fp16 hi of token n; row T + n: its residual lo), K-major
// canonical layout (element (n, k): (k/8)*lbo + (n/8)*128 + (n%8)*16 +
// (k%8)*2, lbo = N/8 * 128).  One CTA per padded token: its range first
// (xrange.cuh), then one thread per 8-column chunk (two 16-byte stores).
__global__ void __launch_bounds__(256) umma_xprep_kernel(const float* __restrict__ x, int ldx, int M, int cols,
                                                         int T, int KS, uint8_t* __restrict__ xf,
                                                         float* __restrict__ unsc, uint32_t* __restrict__ nonfin) {
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
  const int N = 2 * T, tl = tok % T, tile = tok / T;
  const uint32_t lbo = static_cast<uint32_t>(N / 8) * 128, stage_bytes = static_cast<uint32_t>(N) * kStageK * 2;
  for (int ch = tid; ch < KS * (kStageK / 8); ch += blockDim.x) {
    const int ks = ch / (kStageK / 8), cin = ch % (kStageK / 8), k0 = ch * 8;
    uint32_t h[4], l[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      float v0 = 0.f, v1 = 0.f;
      if (tok < M) {
        if (k0 + 2 * p < cols) v0 = xr_scaled(__ldg(xr + k0 + 2 * p), sc);
        if (k0 + 2 * p + 1 < cols) v1 = xr_scaled(__ldg(xr + k0 + 2 * p + 1), sc);
      }
      const __half h0 = __float2half_rn(v0), h1 = __float2half_rn(v1);
      const __half l0 = __float2half_rn(v0 - __half2float(h0)), l1 = __float2half_rn(v1 - __half2float(h1));
      h[p] = static_cast<uint32_t>(__half_as_ushort(h0)) | (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
      l[p] = static_cast<uint32_t>(__half_as_ushort(l0)) | (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
    }
    uint8_t* st = xf + (static_cast<size_t>(tile) * KS + ks) * stage_bytes + cin * lbo;
    const int nh = tl, nl = T + tl;
    *reinterpret_cast<uint4*>(st + (nh >> 3) * 128 + (nh & 7) * 16) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(st + (nl >> 3) * 128 + (nl & 7) * 16) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

struct UmmaPlan {
  int T = 0, TT = 0, S = 1, KQC = 0;
  size_t smem = 0;
};

UmmaPlan plan_umma(const egt_dev_packed* h, int M, int num_sms) {
  UmmaPlan p;
  const int tiles = (M + kMaxT - 1) / kMaxT;
  p.T = ((M + tiles - 1) / tiles + 15) / 16 * 16;  // N = 2T a multiple of 32
  p.TT = (M + p.T - 1) / p.T;
  const int KQ = h->tiled.KQ;
  const int R = (h->tiled.RT + 7) / 8;
  // split K while it removes a wave: cost ~ waves x k-quads per CTA
  double best = 1e300;
  for (int S = 1; S <= std::min(8, KQ); ++S) {
    const int kqc = (KQ + S - 1) / S;
    const int Seff = (KQ + kqc - 1) / kqc;
    const long long ctas = static_cast<long long>(R) * p.TT * Seff;
    const double waves = std::ceil(static_cast<double>(ctas) / num_sms);
    const double cost = waves * (kqc + 1.5) + (Seff > 1 ? 0.75 : 0.0);
    if (cost < best - 1e-9) {
      best = cost;
      p.S = Seff;
      p.KQC = kqc;
    }
  }
  return p;
}

uint32_t raw_rt_bytes(int fmt, int E) {
  return static_cast<uint32_t>(raw_kq(fmt) * 32 * (val_lane_bytes(fmt) + meta_lane_bytes(fmt)) +
                               (has_scales(fmt) ? raw_kq(fmt) * E * 16 : 0));
}

// EGT_UMMA_DENSE: 2:4 layers expanded with zeros on the dense kind::f16 MMA
// instead of the sparse one (A/B comparison)
void* pick_umma(int fmt) {
  static const bool dense = getenv("EGT_UMMA_DENSE") != nullptr;
  switch (fmt) {
    case I4_SP24:
      return dense ? reinterpret_cast<void*>(&umma_spmm_kernel<I4_SP24, false>)
                   : reinterpret_cast<void*>(&umma_spmm_kernel<I4_SP24, true>);
    case I4_DENSE: return reinterpret_cast<void*>(&umma_spmm_kernel<I4_DENSE, false>);
    default:
      return dense ? reinterpret_cast<void*>(&umma_spmm_kernel<F16_SP24, false>)
                   : reinterpret_cast<void*>(&umma_spmm_kernel<F16_SP24, true>);
  }
}

}  // namespace

bool umma_eligible(const egt_dev_packed* h, int M) {
  static const bool off = getenv("EGT_NO_UMMA") != nullptr;
  if (off || M < 17 || h->path != 0) return false;
  const int f = h->format;
  if (f != I4_SP24 && f != I4_DENSE && f != F16_SP24) return false;
  if (has_scales(f) && h->tiled.SS != 4 && h->tiled.SS != 2) return false;
  return true;
}

size_t umma_workspace_bytes(const egt_dev_packed* h, int M) {
  const int tiles = (M + kMaxT - 1) / kMaxT;
  const int T = ((M + tiles - 1) / tiles + 15) / 16 * 16;
  const int TT = (M + T - 1) / T;
  const size_t KS = 2 * static_cast<size_t>(h->tiled.KQ);
  return static_cast<size_t>(TT) * KS * (2 * T) * kStageK * 2 + static_cast<size_t>(TT) * T * 8;
}

size_t umma_partial_floats(const egt_dev_packed* h, int M, int num_sms) {
  const UmmaPlan p = plan_umma(h, M, num_sms);
  return p.S > 1 ? static_cast<size_t>(p.S) * M * h->rows : 0;
}
size_t umma_counters(const egt_dev_packed* h, int M, int num_sms) {
  const UmmaPlan p = plan_umma(h, M, num_sms);
  return static_cast<size_t>((h->tiled.RT + 7) / 8) * p.TT;
}

cudaError_t launch_umma(const egt_dev_packed* h, const float* x, int ldx, int M, float* y, int ldy,
                        uint8_t* ws, const LaunchCtx& ctx, int num_sms) {
  const UmmaPlan p = plan_umma(h, M, num_sms);
  const int KS = 2 * h->tiled.KQ;
  uint8_t* xf = ws;
  float* unsc = reinterpret_cast<float*>(ws + static_cast<size_t>(p.TT) * KS * (2 * p.T) * kStageK * 2);
  uint32_t* nonfin = reinterpret_cast<uint32_t*>(unsc + p.TT * p.T);
  {
    cudaLaunchConfig_t xc = {};
    xc.gridDim = dim3(p.TT * p.T);
    xc.blockDim = dim3(256);
    xc.stream = ctx.stream;
    cudaLaunchAttribute xa[1];
    xa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    xa[0].val.programmaticStreamSerializationAllowed = 1;
    xc.attrs = xa;
    xc.numAttrs = ctx.pdl ? 1 : 0;
    int cols = static_cast<int>(h->cols), T = p.T, ks = KS;
    void* xargs[] = {const_cast<float**>(&x), &ldx, &M, &cols, &T, &ks, &xf, &unsc, &nonfin};
    cudaError_t e = cudaLaunchKernelExC(&xc, reinterpret_cast<void*>(&umma_xprep_kernel), xargs);
    if (e != cudaSuccess) return e;
    ++launch_counter();
  }
  UmmaArgs a;
  a.vals = h->tiled.vals;
  a.meta = h->tiled.meta;
  a.scales = h->tiled.scales;
  a.zps = h->tiled.zps;
  a.KQ = h->tiled.KQ;
  a.rt_begin = h->tiled.rt_begin;
  a.RT = h->tiled.RT;
  a.rows = static_cast<int>(h->rows);
  a.SS = h->tiled.SS;
  a.E = h->tiled.E;
  a.xf = xf;
  a.unsc = unsc;
  a.nonfin = nonfin;
  a.x = x;
  a.ldx = ldx;
  a.cols = static_cast<int>(h->cols);
  a.M = M;
  a.T = p.T;
  a.N = 2 * p.T;
  a.KS = KS;
  a.KQC = p.KQC;
  a.S = p.S;
  a.y = y;
  a.ldy = ldy;
  a.res = ctx.res;
  a.ldr = ctx.ldr;
  a.out_silu = ctx.out_silu;
  a.partial = ctx.partial;
  a.counters = ctx.counters;
  a.pad14 = h->tiled.pad14;
  a.raw_rt_bytes = raw_rt_bytes(h->format, h->tiled.E);
  const size_t smem = 1024 + kNA * 16384 + kNX * static_cast<size_t>(a.N) * kStageK * 2 + kNR * 8 * a.raw_rt_bytes;
  void* fn = pick_umma(h->format);
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((h->tiled.RT + 7) / 8, p.TT, p.S);
  cfg.blockDim = dim3(kThreads);
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
