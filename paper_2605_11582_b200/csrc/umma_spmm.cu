// Many-token SparseGemv on the 5th-generation tensor cores (tcgen05 + TMEM):
// the X * W^T products of the prefix-tree verification pass (forward_impl,
// model.cpp:155-195; M = committed prefix + tree nodes, 64-272 rows in the
// BASELINE configs) and every product of >= 9 tokens, for INT4 2:4 (and 1:4
// stored as 2:4), dense INT4 and FP16 2:4 layers with 64- / 128-column groups.
//
// One CTA = 128 weight rows x one token tile (T <= 96 tokens) x a K range;
// with several same-shape matrices (Q, K, V) blockIdx.x = segment x row block.
// The accumulator lives in TMEM: D[128 rows x 2T] -- x enters as fp16 hi
// (columns [0, T)) and lo = x - hi (columns [T, 2T)) in one B operand, so a
// single tcgen05.mma (M = 128, N = 2T) multiplies both and the epilogue sums
// them in f32 (x keeps ~22 mantissa bits; umma_xprep_kernel scales each token
// by a power of two (xrange.cuh) and folds an input rmsnorm).
//
// Warp roles (19 warps, 608 threads, one CTA per SM -- it owns all of TMEM):
//   warp 0      weight producer: per raw stage (8 row tiles x 1-2 k-quads)
//               2-D TMA tensor-map loads of values, metadata, zero points,
//               scales, the first ones before the PDL wait -- weights never
//               depend on the previous kernel;
//   warp 18     x producer: the pre-laid-out x stages, one bulk copy per
//               k-quad slot (two 64-column sub-stages), counted on the slot's
//               full barrier with the dequantisers (optionally multicast to
//               a pair of row blocks, EGT_UMMA_MCAST);
//   warp 1      TMEM allocator + single-thread MMA issuer: per k-quad slot one
//               barrier wait, 4 sparse (8 dense) MMAs, one commit -- the
//               issue chain (~250 cycles per tcgen05.mma whatever N) is what
//               bounds the kernel (DESIGN 3.1c);
//   warps 2-9   dequantisers: two groups of four (one sub-stage each), two
//               row tiles per warp: packed stage -> the A stage in the UMMA
//               canonical K-major swizzled layout, c - z exact in fp16 (the
//               0x6400 exponent trick); the 2:4 metadata into TMEM
//               (tcgen05.st), then fence.proxy.async;
//   warps 10-17 epilogue: one scale step (128 or 64 columns) per TMEM buffer
//               (two buffers, ping-pong), acc += s_g * (D_hi + D_lo) -- the
//               reference's (c - z) * s per group, summed in f32; FP16 layers
//               accumulate the whole K range in TMEM and are read once.
// Split-K (S > 1): the S slices of a row block form a thread-block cluster;
// each slice owns a 1/S share of the token groups: every slice bulk-copies
// the other slices' shares of its partial tile into their shared memory
// (cp.async.bulk shared::cta -> shared::cluster, completing on the owner's
// mbarrier) and the owner sums the S shares in slice order (deterministic,
// no global round trip).  Loading the shares with DSMEM loads instead ran a
// ~7 us tail per launch (cold, unrolled straight-line code and remote-load
// latency; EGT_UMMA_PULL=1 keeps that path for comparison).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "device_common.cuh"
#include "egt_b200.h"
#include "handle.h"
#include "xrange.cuh"

#ifndef EGT_UMMA_NR
#define EGT_UMMA_NR 3
#endif
namespace egt_impl {
using namespace egt_dev;
using namespace egt_fmt;

namespace {

constexpr int kThreads = 608;  // 19 warps
// dequantisers: two groups of 4 warps take alternate stages (per stage a
// group's warps cover the 8 row tiles, two each)
constexpr int kDeqWarp0 = 2, kNumDeq = 8, kDeqGroup = 4, kEpiWarp0 = 10, kNumEpi = 8, kXWarp = 18;
constexpr int kStageK = 64;  // K per A / B stage: four K = 16 MMAs
// k-quads per packed-weight (raw) stage (FP16 blocks are 4.5x larger)
__host__ __device__ constexpr int raw_kq(int fmt) { return fmt == egt_fmt::F16_SP24 ? 1 : 2; }
// ring depths: raw weight stages kNR; A stages and x stages runtime (a.NA,
// a.NX).  The A ring spans the MMA -> commit -> dequantiser -> MMA round
// trip (~2 us measured with EGT_UMMA_TRACE): 4 slots capped the kernel at
// ~0.5 us per stage whatever the work.
constexpr int kNR = EGT_UMMA_NR, kMaxNA = 6;
// scale hand-off ring (rounds): the dequantisers run up to kMaxNA stages
// (= rounds at 64-column groups) ahead of the MMA, the epilogue up to two
// rounds behind it
constexpr int kScaleRing = 16;
static_assert(kScaleRing > 2 * kMaxNA + 2, "scale ring too shallow");
// tokens per tile: a tcgen05.mma costs ~170 cycles to issue whatever its N
// (measured, tools/micro/umma_rate.cu), so each MMA takes the tile's hi AND lo
// halves (N = 2T <= 192); two accumulator buffers + the metadata ring fit
// the 512 TMEM columns
constexpr int kMaxT = 96;

constexpr int kMaxSeg = 3;  // same-shape matrices of one launch (Q, K, V)

struct UmmaArgs {
  // per segment (matrix): 2-D tensor maps over the handle's row tiles (int64
  // elements) of values, metadata, zero points, scales; box = one raw stage
  // of 8 row tiles
  CUtensorMap tm[kMaxSeg][4];
  int nseg, RB1;  // segments; 128-row blocks per segment (blockIdx.x = seg * RB1 + block)
  // 1: row blocks in pairs (cluster x = 2, S = 1) share the token tile's x
  // stages: each CTA loads one 64-column half of a k-quad slot, multicast to
  // both (L2 x traffic halved); a slot is refilled once both CTAs consumed it
  int mcast;
  // 1: split-K partials are pushed (default; EGT_UMMA_PULL=1 off): each slice's tile is
  // stored token-group-major (float4 per (4-token group, row)) and every
  // slice bulk-copies the other slices' shares into their shared memory
  // (cp.async.bulk shared::cta -> shared::cluster, one mbarrier per CTA);
  // the owner then sums S local shares with a short rolled loop
  int push;
  int NX;  // x ring depth
  int NA;  // A ring depth
  const uint8_t* vals[kMaxSeg];
  const uint8_t* meta[kMaxSeg];
  const float* scales[kMaxSeg];
  const uint8_t* zps[kMaxSeg];
  int rt_begin[kMaxSeg];
  int KQ, RT, rows, SS, E;
  const uint8_t* xf;  // B stages [tile][k-stage][N rows x 64 K fp16, canonical K-major]
  const float* unsc;  // per padded token: 2^-e (xrange.cuh)
  const float* tinv;  // per padded token: the rmsnorm factor (x' = x * tinv), or null
  const uint32_t* nonfin;
  const float* x;  // the raw activations (non-finite fix-up only)
  int ldx, cols;
  int M, T, N;  // tokens, tokens per tile (the MMA's N), N = 2T rows per x stage
  int TTpad;    // padded tokens (token tiles x T) of unsc / nonfin
  int KS;       // B k-stages of the whole K (2 per k-quad)
  int KQC;      // k-quads per CTA (the split size)
  int S;        // K splits (gridDim.z)
  float* y[kMaxSeg];
  int ldy;
  const float* res;
  int ldr;
  int out_silu;
  float* partial;
  uint32_t* counters;
  int pad14;
  uint32_t raw_rt_bytes;  // bytes per row tile in a raw stage
  // tuning (EGT_UMMA_TRACE): globaltimer stamps of CTA (0,0,0): [0] start,
  // [1] past alloc, [8+st] x issued, [80+st] MMA issued, [160+st] stage
  // dequantised (warp 2), [240+r] round folded (warp 6), [320+rs] raw issued
  unsigned long long* trace;
  int dbg;  // tuning (EGT_UMMA_DBG): 1 dequantisers skip the A writes, 2 epilogue skips TMEM loads, 4 no MMAs
};

__device__ __forceinline__ unsigned long long umma_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return smem_u32(p); }

// UMMA shared-memory descriptor, K-major, swizzled: rows of 128 B (x stages,
// dense A) or 64 B (compressed sparse A), 8-row swizzle atoms (sbo = the
// atom's bytes), the 16-byte chunks of row r XOR-permuted by r's position in
// the atom; K steps within the atom advance the start address.
__device__ __forceinline__ uint64_t umma_desc_sw(uint32_t saddr, uint32_t row_bytes) {
  const uint64_t layout = row_bytes == 128 ? 2ull : 4ull;  // SWIZZLE_128B / SWIZZLE_64B
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) |
         (static_cast<uint64_t>(((8 * row_bytes) >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}
// byte offset of (row, byte-in-row) in a swizzled tile with 128- / 64-byte rows
__device__ __forceinline__ uint32_t sw128(int r, int byte) {
  return static_cast<uint32_t>(r * 128 + (byte ^ ((r & 7) << 4)));
}
__device__ __forceinline__ uint32_t sw64(int r, int byte) {
  return static_cast<uint32_t>(r * 64 + (byte ^ (((r >> 1) & 3) << 4)));
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

// 2-D tensor-map load into shared memory, completing on an mbarrier
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}

// x halves multicast to both CTAs of a row-block pair (cluster x = 2)
__device__ __forceinline__ void bulk_g2s_mcast(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "h"(mask)
      : "memory");
}
// commit arriving on the same barrier offset in every CTA of `mask`
__device__ __forceinline__ void umma_commit_mcast(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                   smem_addr(bar)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_addr(bar))
               : "memory");
}
// shared::cta -> a cluster peer's shared memory, completing on the peer's mbarrier
__device__ __forceinline__ void bulk_s2peer(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   dst_cluster),
               "r"(src), "r"(bytes), "r"(bar_cluster)
               : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
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

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];\n" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
// mbarrier wait that sleeps between probes (the epilogue waits a whole scale
// step: polling would steal issue slots from the dequantisers)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITH_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITH_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(20000u)
      : "memory");
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

// A-operand byte offset of (row r, column k): a 128 x 64 fp16 stage with
// 128-byte rows (dense), or 128 x 32 compressed with 64-byte rows (sparse)
template <bool SPARSE>
__device__ __forceinline__ uint32_t a_off(int r, int k) {
  return SPARSE ? sw64(r, 2 * k) : sw128(r, 2 * k);
}

template <int FMT>
__device__ __noinline__ float umma_nonfinite_terms(const UmmaArgs& a, int sg, int row, int tok, int c0, int c1) {
  const TiledRef m{a.vals[sg], a.meta[sg], a.scales[sg], a.zps[sg], a.KQ, a.rt_begin[sg], a.SS, a.pad14};
  const float* xr = a.x + static_cast<size_t>(tok) * a.ldx;
  const float inv = a.tinv ? a.tinv[tok] : 1.f;
  float add = 0.f;
  for (int c = c0; c < c1; ++c) {
    const float xv = xr[c] * inv;
    if ((__float_as_uint(xv) & 0x7fffffffu) < 0x7f800000u) continue;
    float w;
    if (tiled_value<FMT>(m, row, c, &w)) add += w * xv;
  }
  return add;
}

template <int FMT, bool SPARSE>
__global__ void __launch_bounds__(kThreads, 1) umma_spmm_kernel(const __grid_constant__ UmmaArgs a) {
  static_assert(!SPARSE || FMT != I4_DENSE, "dense INT4 has no 2:4 metadata");
  constexpr bool kScaled = has_scales(FMT);
  constexpr int kRawKQ = raw_kq(FMT);
  constexpr int VB = val_lane_bytes(FMT), MB = meta_lane_bytes(FMT);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long* tr =
      (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) ? a.trace : nullptr;
  if (tr && tid == 0) tr[0] = umma_clock();
  const int sg = a.nseg > 1 ? static_cast<int>(blockIdx.x) / a.RB1 : 0;  // segment (matrix)
  const int rt0 = (static_cast<int>(blockIdx.x) - sg * a.RB1) * 8;      // first 16-row tile of this CTA (128 rows)
  const int tile = blockIdx.y;     // token tile
  const int kq0 = blockIdx.z * a.KQC;
  const int KQC = min(a.KQC, a.KQ - kq0);
  const int NSTG = 2 * KQC;                     // A / B stages of this CTA
  const int NRAW = (KQC + kRawKQ - 1) / kRawKQ;  // raw stages
  const int T = a.T, N = a.N;
  const int steps_per_scale = kScaled ? a.SS / 2 : NSTG;  // stages per accumulation round
  const int NROUND = kScaled ? NSTG / steps_per_scale : 1;

  // ---- shared memory carve-up
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + ((1024 - (smem_addr(smem_raw) & 1023)) & 1023));
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = raw_full + kNR;
  uint64_t* a_full = raw_empty + kNR;
  const int kNA = a.NA;
  uint64_t* a_empty = a_full + kMaxNA;
  const int kNX = a.NX;
  uint64_t* tm_full = a_empty + kMaxNA;
  uint64_t* tm_empty = tm_full + 2;
  uint64_t* recv_bar = tm_empty + 2;  // push: the other slices' shares landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_bar + 1);
  __shared__ float s_unsc[kMaxT];
  __shared__ uint32_t s_nonf[kMaxT];
  __shared__ int s_anynf;  // some token of the tile has a non-finite x
  // swizzle atoms need 1024-byte aligned tiles
  uint8_t* smem_al = smem_raw + ((1024 - (smem_addr(smem_raw) & 1023)) & 1023);
  uint8_t* a_st = smem_al + 1024;  // kNA x 16 KB
  constexpr uint32_t kASlot = SPARSE ? 8192 : 16384;
  // ring slots hold one k-quad = two 64-column sub-stages: every mbarrier
  // probe / tcgen05.commit in the MMA thread's chain costs ~100-220 cycles
  // (clock64, EGT_UMMA_TRACE), so the chain runs once per k-quad, not per
  // sub-stage
  uint8_t* x_st = a_st + kNA * 2 * kASlot;  // kNX x 2 x (N x 128 B)
  const uint32_t x_bytes = static_cast<uint32_t>(N) * kStageK * 2;
  uint8_t* raw_st = x_st + kNX * 2 * x_bytes;  // kNR x (8 x raw_rt_bytes)
  // raw stage: [values 8 x VBq][metadata 8 x MBq][zero points 8 x ZBq][scales 8 x SBq]
  constexpr int VBq = kRawKQ * 32 * VB, MBq = kRawKQ * 32 * MB;
  const int ZBq = kScaled ? kRawKQ * a.E * 16 : 0, SBq = kScaled ? kRawKQ * a.E * 64 : 0;
  // the scales of the epilogue's rounds, handed over by the dequantisers
  // (ring of kScaleRing rounds; ordered by a_full -> MMA -> tm_full)
  __shared__ float s_scale[kScaleRing * 128];
  const uint32_t raw_bytes = 8 * a.raw_rt_bytes;
  const uint32_t raw_s0 = smem_addr(raw_st);

  if (tid == 0) {
    s_anynf = 0;
    for (int i = 0; i < kNR; ++i) {
      mbar_init(raw_full + i, 1);
      mbar_init(raw_empty + i, kNumDeq);
    }
    for (int i = 0; i < kNA; ++i) {
      // one ring of k-quad slots for A and x: full = both dequantiser groups
      // (one sub-stage each) + the x producer's arrive.expect_tx (and its
      // bytes); empty = one MMA commit
      mbar_init(a_full + i, kNumDeq + 1);
      mbar_init(a_empty + i, a.mcast ? 2 : 1);  // multicast: both CTAs' commits
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tm_full + i, 1);
      mbar_init(tm_empty + i, kNumEpi);
    }
    if (a.push) mbar_init(recv_bar, 1);
    mbar_fence_init();
    if (a.push && a.S > 1) {  // armed before the cluster barrier the senders wait on
      const int G4 = T / 4, per = (G4 + a.S - 1) / a.S;
      const int mine = max(0, min(G4, (static_cast<int>(blockIdx.z) + 1) * per) - static_cast<int>(blockIdx.z) * per);
      mbar_expect_tx(recv_bar, static_cast<uint32_t>((a.S - 1) * mine * 2048));
    }
  }
  // TMEM: accumulator buffer(s) at column 0 (T <= 64 columns each), sparse
  // metadata (2 columns per A-stage ring slot) at column 128
  // metadata ring: 16 stages x 2 columns at 448 (written a raw stage ahead)
  constexpr uint32_t kMetaCol = 448, kMetaRing = 16;
  constexpr uint32_t tmem_cols = 512u;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(tmem_slot)),
                 "n"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tr && tid == 0) tr[1] = umma_clock();

  if (warp == 0) {
    // ================= weight producer: three 2-D tensor loads per raw stage
    if (lane == 0) {
      auto issue_raw = [&](int rs) {
        const int sr = rs % kNR;
        if (rs >= kNR) mbar_wait(raw_empty + sr, ((rs / kNR) - 1) & 1);
        if (tr && rs < 64) tr[320 + rs] = umma_clock();
        const int kq = kq0 + rs * kRawKQ;
        uint8_t* dst = raw_st + sr * raw_bytes;
        mbar_expect_tx(raw_full + sr, raw_bytes);  // full boxes (rows / k-quads past the matrix read as 0)
        tma_load_2d(dst, &a.tm[sg][0], kq * (32 * VB / 8), rt0, raw_full + sr);
        if (MB > 0) tma_load_2d(dst + 8 * VBq, &a.tm[sg][1], kq * (32 * MB / 8), rt0, raw_full + sr);
        if (kScaled) {
          tma_load_2d(dst + 8 * (VBq + MBq), &a.tm[sg][2], kq * (a.E * 2), rt0, raw_full + sr);
          tma_load_2d(dst + 8 * (VBq + MBq + ZBq), &a.tm[sg][3], kq * (a.E * 8), rt0, raw_full + sr);
        }
      };
      for (int rs = 0; rs < NRAW; ++rs) issue_raw(rs);
    }
  } else if (warp == kXWarp) {
    // ================= x producer
    if (lane == 0) {
      pdl_wait();  // x stages come from the preceding xprep kernel
      for (int u = 0; u < KQC; ++u) {  // one k-quad (two contiguous x stages) per slot
        const int s = u % kNA;
        if (u >= kNA) mbar_wait(a_empty + s, ((u / kNA) - 1) & 1);
        mbar_expect_tx(a_full + s, 2 * x_bytes);  // both halves land here (multicast: one from the peer)
        if (tr && u < 72) tr[8 + u] = umma_clock();
        const uint8_t* src = a.xf + (static_cast<size_t>(tile) * a.KS + 2 * (kq0 + u)) * x_bytes;
        if (a.mcast) {
          const int half = static_cast<int>(blockIdx.x & 1);
          bulk_g2s_mcast(x_st + (s * 2 + half) * x_bytes, src + half * x_bytes, x_bytes, a_full + s, 3);
        } else {
          bulk_g2s_plain(x_st + s * 2 * x_bytes, src, 2 * x_bytes, a_full + s);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(N);  // x stage rows: hi [0, T), lo [T, 2T)
      for (int u = 0; u < KQC; ++u) {
        const bool ck = tr && u >= 2 && u < 10;
        const long long c0 = ck ? clock64() : 0;
        if (tr && u < 80) tr[560 + u] = umma_clock();
        mbar_wait(a_full + u % kNA, (u / kNA) & 1);  // A and x of the slot
        tc_fence_after();
        const long long c1 = ck ? clock64() : 0;
        if (tr && u < 80) tr[80 + u] = umma_clock();
#pragma unroll
        for (int hs = 0; hs < 2; ++hs) {
          const int st = 2 * u + hs;
          const int round = st / steps_per_scale, first = st % steps_per_scale == 0;
          const int buf = kScaled ? (round & 1) : 0;
          if (kScaled && first && round >= 2) {
            mbar_wait(tm_empty + buf, ((round / 2) - 1) & 1);
            tc_fence_after();
          }
          const uint32_t abase = smem_addr(a_st + ((u % kNA) * 2 + hs) * kASlot);
          const uint32_t bbase = smem_addr(x_st + ((u % kNA) * 2 + hs) * x_bytes);
          const uint32_t d = tmem + static_cast<uint32_t>(buf * N);
          if (a.dbg & 4) {
          } else if constexpr (SPARSE) {  // two K = 32 (logical) sparse MMAs per sub-stage, x hi and lo
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const uint64_t ad = umma_desc_sw(abase + jj * 32, 64);
              const uint32_t e = tmem + kMetaCol + static_cast<uint32_t>(2 * (st % kMetaRing) + jj);
              umma_f16_sp(d, ad, umma_desc_sw(bbase + jj * 64, 128), e, idesc, (first && jj == 0) ? 0u : 1u);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = umma_desc_sw(abase + kk * 32, 128);
              umma_f16(d, ad, umma_desc_sw(bbase + kk * 32, 128), idesc, (first && kk == 0) ? 0u : 1u);
            }
          }
          if ((st + 1) % steps_per_scale == 0 || st + 1 == NSTG) umma_commit(tm_full + buf);
        }
        const long long c2 = ck ? clock64() : 0;
        if (a.mcast) umma_commit_mcast(a_empty + u % kNA, 3);  // the peer's x producer reuses the slot too
        else umma_commit(a_empty + u % kNA);
        if (a.mcast && u + 1 == KQC)  // both CTAs' last commits landed here before the pair may exit
          mbar_wait(a_empty + u % kNA, (u / kNA) & 1);
        if (ck) {
          const long long c3 = clock64();
          unsigned long long* o = tr + 900 + 8 * (u - 2);
          o[0] = c1 - c0; o[1] = c2 - c1; o[2] = c3 - c2; o[3] = c3 - c0;
        }
      }
    }
  } else if (warp < kEpiWarp0) {
    // ================= dequantisers: raw stage -> A stage, one row tile per
    // warp.  Warp w may write TMEM lanes [32 (w % 4), +32) only (tcgen05.st):
    // warps 2-5 write the metadata of row tiles 2 (w % 4) and 2 (w % 4) + 1.
    const int dq = warp & 3, grp = (warp - kDeqWarp0) / kDeqGroup;
    const int g = lane >> 2, t = lane & 3;
    const int eshift = a.SS == 4 ? 2 : 1;  // k-tile j of a k-quad -> scale entry j >> eshift
    for (int st = grp; st < NSTG; st += 2) {  // group grp: sub-stage hs = grp of every k-quad
      const int un = st >> 1, sa = un % kNA;
      if (un >= kNA) mbar_wait(a_empty + sa, ((un / kNA) - 1) & 1);
      if (tr && warp == kDeqWarp0 && lane == 0 && st < 80) tr[640 + st] = umma_clock();
      const int kql = st >> 1, hs = st & 1;
      const int rs = kql / kRawKQ, b = kql % kRawKQ;
      mbar_wait(raw_full + rs % kNR, (rs / kNR) & 1);
      if (tr && warp == kDeqWarp0 && lane == 0 && st < 80) tr[720 + st] = umma_clock();
      const uint32_t rbase = raw_s0 + (rs % kNR) * raw_bytes;
      if constexpr (SPARSE) {
        if (b == 0) {
          // metadata of this group's sparse MMAs in the raw stage (stages st and
          // st + 2: k-tiles 2 hs, 2 hs + 1 of each k-quad) -> TMEM lanes
          // [32 dq, +32), one wait per raw stage
          const int ti = 2 * dq + (lane >> 4), l16 = lane & 15, gg = l16 & 7, kh = l16 >> 3;
#pragma unroll
          for (int bq = 0; bq < kRawKQ; ++bq) {
            uint32_t w0 = 0x44444444u, w1 = 0x44444444u;  // (0,1): rows / k-quads past the matrix
            if (rt0 + ti < a.RT && kq0 + rs * kRawKQ + bq < a.KQ) {
              const uint32_t mb = rbase + 8 * VBq + ti * MBq + bq * 32 * MB;
              const int j0 = 2 * hs, j1 = 2 * hs + 1;
              w0 = lds_u32(mb + ((4 * gg + 2 * (j0 & 1) + kh) * 2 + (j0 >> 1)) * 4);
              w1 = lds_u32(mb + ((4 * gg + 2 * (j1 & 1) + kh) * 2 + (j1 >> 1)) * 4);
            }
            tmem_st2(tmem + (static_cast<uint32_t>(32 * dq) << 16) + kMetaCol + 2 * ((st + 2 * bq) % kMetaRing), w0,
                     w1);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
          tc_fence_before();
        }
      }
      const uint32_t abase = smem_addr(a_st + (sa * 2 + (st & 1)) * kASlot);
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) {
      if (a.dbg & 1) break;
      const int i = 2 * dq + ii;  // row tile within the CTA
      if (rt0 + i >= a.RT) {  // past the matrix: zero rows
        for (int w = lane; w < (SPARSE ? 64 : 128); w += 32) {  // 16 rows x 4 / 8 chunks
          const int r = i * 16 + (w & 15), ch = w >> 4;
          st_shared_v4(abase + (SPARSE ? sw64(r, 16 * ch) : sw128(r, 16 * ch)), make_uint4(0, 0, 0, 0));
        }
      } else {
        const uint32_t vbase = rbase + i * VBq + (b * 32 + lane) * VB;
        const uint32_t mbase = rbase + 8 * VBq + i * MBq + b * 32 * MB;
        const uint32_t zbase = rbase + 8 * (VBq + MBq) + i * ZBq + b * a.E * 16;
        if constexpr (FMT == I4_DENSE) {
          const uint4 vv = lds_v4(vbase + hs * 16);  // words w16 = 4 hs .. 4 hs + 3
          const uint32_t wv[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
          for (int w4 = 0; w4 < 4; ++w4) {
            const int e = (4 * hs + w4) >> (eshift + 1);
            const uint32_t zz = lds_u16(zbase + e * 16 + 2 * g);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t z = (zz >> (8 * h)) & 0xFFu;
              const int r = i * 16 + g + 8 * h;
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int p = h + 2 * q;
                const uint32_t pr = cz_pair((wv[w4] >> (4 * p)) & 0xFu, (wv[w4] >> (16 + 4 * p)) & 0xFu, z);
                st_shared_b32(abase + a_off<false>(r, 16 * w4 + 2 * t + 8 * q), pr);
              }
            }
          }
        } else {
          uint32_t vw[2][4];  // [jj][h + 2q]: the pair words of k-tiles 2 hs, 2 hs + 1
          if constexpr (FMT == I4_SP24) {
            const uint2 vv = lds_v2(vbase + hs * 8);
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const uint32_t word = jj ? vv.y : vv.x;
#pragma unroll
              for (int p = 0; p < 4; ++p) vw[jj][p] = ((word >> (4 * p)) & 0xFu) | (((word >> (16 + 4 * p)) & 0xFu) << 16);
            }
          } else {  // F16_SP24: 4 pair words per k-tile
            const uint4 v0 = lds_v4(vbase + hs * 32), v1 = lds_v4(vbase + hs * 32 + 16);
            vw[0][0] = v0.x; vw[0][1] = v0.y; vw[0][2] = v0.z; vw[0][3] = v0.w;
            vw[1][0] = v1.x; vw[1][1] = v1.y; vw[1][2] = v1.z; vw[1][3] = v1.w;
          }
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int j = 2 * hs + jj;
            uint32_t zz = 0;
            if constexpr (FMT == I4_SP24) zz = lds_u16(zbase + (j >> eshift) * 16 + 2 * g);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              uint32_t mw = 0;
              if constexpr (!SPARSE) mw = lds_u32(mbase + ((4 * g + 2 * (j & 1) + q) * 2 + (j >> 1)) * 4);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                uint32_t pr = vw[jj][h + 2 * q];
                if constexpr (FMT == I4_SP24) pr = cz_pair(pr & 0xFu, pr >> 16, (zz >> (8 * h)) & 0xFFu);
                const int r = i * 16 + g + 8 * h, G = t + 4 * q;
                if constexpr (SPARSE) {  // the kept pair, compressed K: groups of 4 -> 2 slots
                  st_shared_b32(abase + a_off<true>(r, jj * 16 + 2 * G), pr);
                } else {
                  const uint32_t nib = (mw >> (16 * h + 4 * t)) & 0xFu;
                  st_shared_v2(abase + a_off<false>(r, jj * 32 + 4 * G), place2(pr, nib & 3u, nib >> 2));
                }
              }
            }
          }
        }
      }
      }  // row tiles
      if (kScaled && (a.SS == 2 || hs == 0)) {  // this round's scales of row tiles 2 dq, 2 dq + 1
        const int e = a.SS == 2 ? hs : 0, i = 2 * dq + (lane >> 4), l16 = lane & 15;
        const uint32_t sb = rbase + 8 * (VBq + MBq + ZBq) + i * SBq + b * a.E * 64;
        s_scale[((st / steps_per_scale) % kScaleRing) * 128 + i * 16 + l16] =
            __uint_as_float(lds_u32(sb + (e * 16 + 2 * (l16 & 7) + (l16 >> 3)) * 4));
      }
      fence_async_smem();  // generic-proxy writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(a_full + sa);
        if (b == kRawKQ - 1 || kql == KQC - 1) mbar_arrive(raw_empty + rs % kNR);  // this group's last use
        if (tr && warp == kDeqWarp0 && st < 80) tr[160 + st] = umma_clock();
        if (tr && warp == kEpiWarp0 - 1 && st < 80) tr[480 + st] = umma_clock();  // last dequantiser
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
    for (int k = 0; k < kMaxT / 2; ++k) acc[k] = 0.f;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * q) << 16);
    const bool row_ok = grow < a.rows && (rt0 + (r >> 4)) < a.RT;
    // x scales / non-finite flags (the xprep kernel) and, below, residual
    // rows belong to earlier kernels: wait now, while the first round runs
    pdl_wait();
    {
      const int ew = (warp - kEpiWarp0) * 32 + lane;
      if (ew < T) {
        const int tok = min(tile * T + ew, a.TTpad - 1);
        s_unsc[ew] = a.unsc[tok];
        s_nonf[ew] = a.nonfin[tok];
        if (s_nonf[ew]) s_anynf = 1;
      }
    }
    for (int round = 0; round < NROUND; ++round) {
      const int buf = kScaled ? (round & 1) : 0;
      mbar_wait_sleep(tm_full + buf, kScaled ? ((round >> 1) & 1) : 0);
      tc_fence_after();
      const float s = kScaled ? s_scale[(round % kScaleRing) * 128 + r] : 1.f;  // the row's scale of this round
      // chunks of 16 tokens: their hi and lo columns in flight together, one wait
#pragma unroll
      for (int cb = 0; cb < (kMaxT / 2 + 15) / 16; ++cb) {
        if (cb * 16 < th && !(a.dbg & 2)) {
          uint32_t vh[16], vl[16];
          const uint32_t col = lane_base + static_cast<uint32_t>(buf * N + c0 + cb * 16);
          tmem_ld8_nowait(col, vh);
          tmem_ld8_nowait(col + T, vl);
          if (cb * 16 + 8 < th) {
            tmem_ld8_nowait(col + 8, vh + 8);
            tmem_ld8_nowait(col + T + 8, vl + 8);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (cb * 16 + k < th && cb * 16 + k < kMaxT / 2)
              acc[cb * 16 + k] = fmaf(s, __uint_as_float(vh[k]) + __uint_as_float(vl[k]), acc[cb * 16 + k]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (kScaled && lane == 0) mbar_arrive(tm_empty + buf);
      if (tr && warp == kEpiWarp0 && lane == 0 && round < 80) tr[240 + round] = umma_clock();
    }
    // ---- outputs: rescale (xrange.cuh), fix-up; then residual / silu and the
    // store (one CTA), or the cluster's split-K sum (below)
    if (tr && lane == 0) tr[800 + warp - kEpiWarp0] = umma_clock();
    asm volatile("bar.sync 1, %0;\n" ::"n"(kNumEpi * 32) : "memory");  // s_unsc / s_nonf written
    // The accumulators, times the tokens' 2^-e (xrange.cuh), into shared
    // memory (the x ring is idle now): row-major, tokens contiguous, PT = T + 4
    // (conflict-free float4s).  Straight-line code run once per CTA is kept
    // short -- its instruction fetches are cold (an unrolled per-token tail
    // measured 3.4 us).
    float* part = reinterpret_cast<float*>(x_st);
    // pull: row-major (tokens contiguous, PT = T + 4); push: float4 per
    // (4-token group, row), group-major, so a slice's share is contiguous
    auto pidx = [&](int row, int tl) {
      return a.push ? ((tl >> 2) * 128 + row) * 4 + (tl & 3) : row * (T + 4) + tl;
    };
    {
#pragma unroll
      for (int k = 0; k < kMaxT / 2; k += 4)
        if (k < th) {
          const float4 u = *reinterpret_cast<const float4*>(s_unsc + c0 + k);
          *reinterpret_cast<float4*>(part + pidx(r, c0 + k)) =
              make_float4(acc[k] * u.x, acc[k + 1] * u.y, acc[k + 2] * u.z, acc[k + 3] * u.w);
        }
    }
    if (s_anynf) {  // non-finite x somewhere in the tile: exact fix-up, token by token
      const int kc0 = kq0 * 128, kc1 = min(a.cols, (kq0 + KQC) * 128);
      for (int k = 0; k < th; ++k) {
        const int tl = c0 + k, tok = tile * T + tl;
        if (row_ok && tok < a.M && s_nonf[tl])
          part[pidx(r, tl)] += umma_nonfinite_terms<FMT>(a, sg, grow, tok, kc0, kc1);
      }
    }
    if (a.push) fence_async_smem();  // the partials are read by the bulk-copy engine
    if (tr && lane == 0) tr[840 + warp - kEpiWarp0] = umma_clock();
  }

  // ---- teardown: TMEM back; split K: the cluster's leader sums the slices'
  // partials from their shared memory (DSMEM) in slice order -- deterministic
  if (tr && tid == kEpiWarp0 * 32) tr[2] = umma_clock();
  if (tr && warp >= kEpiWarp0 && warp < kEpiWarp0 + kNumEpi && lane == 0) tr[820 + warp - kEpiWarp0] = umma_clock();
  tc_fence_before();
  __syncthreads();
  if (tr && tid == 0) tr[3] = umma_clock();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(tmem_cols) : "memory");
  pdl_launch_dependents();
  if (a.S > 1)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (tr && tid == 0) tr[4] = umma_clock();
  if (a.push) {
    const int G4 = T / 4, per = (G4 + a.S - 1) / a.S, myz = static_cast<int>(blockIdx.z);
    const uint32_t pbase = smem_addr(x_st), rbase = pbase + static_cast<uint32_t>(T) * 512;
    if (a.S > 1 && tid == 0) {
      // slice z's share of this slice's tile -> z's receive area, slot myz
      for (int z = 0; z < a.S; ++z) {
        const int n = min(G4, (z + 1) * per) - z * per;
        if (z == myz || n <= 0) continue;
        bulk_s2peer(mapa_u32(rbase + static_cast<uint32_t>(myz * per) * 2048, static_cast<uint32_t>(z)),
                    pbase + static_cast<uint32_t>(z * per) * 2048, static_cast<uint32_t>(n) * 2048,
                    mapa_u32(smem_addr(recv_bar), static_cast<uint32_t>(z)));
      }
    }
    // the output tail on the dequantiser and epilogue warps: a latency-bound
    // loop (~0.45 us per item per thread), 8 warps 5.4 us at M = 272, 16
    // warps 3.2 us (all 19 warps: no faster); verify pass 5.70 -> 5.49 ms
    // (64 nodes), 13.60 -> 13.05 ms (256 nodes)
    if (warp >= kDeqWarp0 && warp < kEpiWarp0 + kNumEpi) {
      const int g0 = myz * per, g1 = min(G4, g0 + per);
      if (a.S > 1) mbar_wait_cluster(recv_bar, 0);
      // every copy into this CTA landed (so its sources were read): the exit
      // barrier may complete while the sums below run
      if (a.S > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      const int nit = max(0, g1 - g0) * 128;
      // the tile's shared-memory address recomputed here from the window base
      // (kept from the prologue it was spilled and reloaded from local
      // memory every item)
      uint32_t pb;
      asm volatile("mov.u32 %0, %1;\n" : "=r"(pb) : "r"(((smem_addr(smem_raw) + 1023u) & ~1023u) + 1024u));
      pb += static_cast<uint32_t>(a.NA) * 2 * kASlot;
      const uint32_t rb = pb + static_cast<uint32_t>(T) * 512;
      for (int it = (warp - kDeqWarp0) * 32 + lane; it < nit; it += (kNumDeq + kNumEpi) * 32) {
        const int r = it & 127, gq = g0 + (it >> 7), grow = rt0 * 16 + r;
        float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
        for (int z = 0; z < a.S; ++z) {  // slice order (deterministic)
          const uint32_t ad = z == myz ? pb + static_cast<uint32_t>((gq * 128 + r) * 16)
                                       : rb + static_cast<uint32_t>(((z * per + gq - g0) * 128 + r) * 16);
          const uint4 v = lds_v4(ad);
          sum.x += __uint_as_float(v.x);
          sum.y += __uint_as_float(v.y);
          sum.z += __uint_as_float(v.z);
          sum.w += __uint_as_float(v.w);
        }
        if (grow >= a.rows || (rt0 + (r >> 4)) >= a.RT) continue;
        const float s4[4] = {sum.x, sum.y, sum.z, sum.w};
        float rr[4] = {0.f, 0.f, 0.f, 0.f};
        if (a.res) {  // the four residual loads in flight together
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int tok = tile * T + 4 * gq + u;
            if (tok < a.M) rr[u] = a.res[static_cast<size_t>(tok) * a.ldr + grow];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int tok = tile * T + 4 * gq + u;
          if (tok < a.M) {
            float o = s4[u] + rr[u];
            if (a.out_silu) o = o * (1.0f / (1.0f + expf(-o)));  // model.cpp:80-84
            a.y[sg][static_cast<size_t>(tok) * a.ldy + grow] = o;
          }
        }
      }
    } else if (a.S > 1) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    }
    if (tr && tid == kEpiWarp0 * 32) tr[5] = umma_clock();
    if (a.S > 1) asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    else if (a.mcast)
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (tr && tid == 0) tr[6] = umma_clock();
    return;
  }
  // each slice reduces a 1/S share of the token groups (4 tokens) for all
  // 128 rows: the S partials in slice order (deterministic), float4 DSMEM
  // loads all in flight, then residual / silu and the store (S = 1: this
  // CTA's own rows, consecutive threads on consecutive rows)
  if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kNumEpi) {
    const int PT = T + 4, G4 = T / 4, per = (G4 + a.S - 1) / a.S;
    const int g0 = blockIdx.z * per, g1 = min(G4, g0 + per);
    const uint32_t part0 = smem_addr(x_st);
    constexpr int kB = 2;  // items per thread in flight: all their S DSMEM loads issued before any use
    const int nit = (g1 - g0) * 128;
    for (int it0 = (warp - kEpiWarp0) * 32 + lane; it0 < nit; it0 += kB * kNumEpi * 32) {
      float4 sum[kB], rv[kB], v[kB][8];
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int it = min(it0 + b * kNumEpi * 32, nit - 1);
        const int r = it & 127, gq = g0 + (it >> 7);
        const uint32_t off = static_cast<uint32_t>((r * PT + 4 * gq) * 4);
#pragma unroll
        for (int z = 0; z < 8; ++z) {
          if (z < a.S) {
            uint32_t remote;
            // cluster rank of slice z of this row block (x: the multicast pair)
            const uint32_t zr = static_cast<uint32_t>(z * (a.mcast ? 2 : 1)) + (a.mcast ? (blockIdx.x & 1) : 0);
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(part0 + off), "r"(zr));
            asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                         : "=f"(v[b][z].x), "=f"(v[b][z].y), "=f"(v[b][z].z), "=f"(v[b][z].w)
                         : "r"(remote));
          }
        }
      }
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int it = it0 + b * kNumEpi * 32;
        sum[b] = make_float4(0.f, 0.f, 0.f, 0.f);
        rv[b] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (it >= nit) continue;
        const int r = it & 127, gq = g0 + (it >> 7), grow = rt0 * 16 + r;
#pragma unroll
        for (int z = 0; z < 8; ++z) {  // slice order
          if (z < a.S) {
            sum[b].x += v[b][z].x;
            sum[b].y += v[b][z].y;
            sum[b].z += v[b][z].z;
            sum[b].w += v[b][z].w;
          }
        }
        if (a.res && grow < a.rows) {
          const int tok = tile * T + 4 * gq;
          const float* rp = a.res + static_cast<size_t>(tok) * a.ldr + grow;
          rv[b].x = tok < a.M ? rp[0] : 0.f;
          rv[b].y = tok + 1 < a.M ? rp[a.ldr] : 0.f;
          rv[b].z = tok + 2 < a.M ? rp[2 * static_cast<size_t>(a.ldr)] : 0.f;
          rv[b].w = tok + 3 < a.M ? rp[3 * static_cast<size_t>(a.ldr)] : 0.f;
        }
      }
      if (tr && tid == kEpiWarp0 * 32 && it0 == lane) tr[7] = umma_clock();
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int it = it0 + b * kNumEpi * 32;
        if (it >= nit) continue;
        const int r = it & 127, gq = g0 + (it >> 7), grow = rt0 * 16 + r;
        if (grow >= a.rows || (rt0 + (r >> 4)) >= a.RT) continue;
        const float o4[4] = {rv[b].x + sum[b].x, rv[b].y + sum[b].y, rv[b].z + sum[b].z, rv[b].w + sum[b].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int tok = tile * T + 4 * gq + u;
          if (tok < a.M) {
            float o = o4[u];
            if (a.out_silu) o = o * (1.0f / (1.0f + expf(-o)));  // model.cpp:80-84
            a.y[sg][static_cast<size_t>(tok) * a.ldy + grow] = o;
          }
        }
      }
    }
  }
  if (tr && tid == kEpiWarp0 * 32) tr[5] = umma_clock();
  if (a.S == 1) {
    if (a.mcast)  // the peer multicasts into this CTA's shared memory until it is done too
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    return;
  }
  // every slice's shared memory stays alive until the leader has read it
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (tr && tid == 0) tr[6] = umma_clock();
}

// X [M x cols] -> B stages: per token tile, per 64-column k-stage, N = 2T rows
// (row n < T: fp16 hi of token n; row T + n: its residual lo) of 128 bytes,
// K-major with the 128-byte swizzle (the bulk copy keeps the pattern: stages
// land 1024-byte aligned).  One CTA per padded token: its range first
// (xrange.cuh; every load of a thread in flight together), then one thread
// per 8-column chunk (two 16-byte stores).
// xform = EGT_INPUT_RMSNORM: x' = x * inv_tok, inv = 1 / sqrt(mean(x^2) + eps)
// (model.cpp:57-67) from the same first pass (tinv[tok] for the non-finite
// fix-up); the range is then the transformed one (max |x'| = max |x| * inv).
__global__ void __launch_bounds__(256) umma_xprep_kernel(const float* __restrict__ x, int ldx, int M, int cols,
                                                         int T, int KS, uint8_t* __restrict__ xf,
                                                         float* __restrict__ unsc, uint32_t* __restrict__ nonfin,
                                                         float* __restrict__ tinv, int xform, float eps) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ uint32_t s_mx, s_nf;
  __shared__ float s_ss[8];
  const int tok = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) {
    s_mx = 0u;
    s_nf = 0u;
  }
  __syncthreads();
  const float* xr = x + static_cast<size_t>(tok) * ldx;
  const bool vec = (ldx & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  float ss = 0.f;
  if (tok < M) {
    uint32_t mx = 0u, nf = 0u;
    if (vec) {
      const int n4 = cols >> 2;
      for (int k4 = tid; k4 < n4; k4 += 4 * blockDim.x) {
        float4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          q[u] = k4 + u * static_cast<int>(blockDim.x) < n4 ? __ldg(reinterpret_cast<const float4*>(xr) + k4 + u * blockDim.x)
                                                           : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          xr_note(mx, nf, q[u].x); xr_note(mx, nf, q[u].y); xr_note(mx, nf, q[u].z); xr_note(mx, nf, q[u].w);
          ss = fmaf(q[u].x, q[u].x, fmaf(q[u].y, q[u].y, fmaf(q[u].z, q[u].z, fmaf(q[u].w, q[u].w, ss))));
        }
      }
      for (int k = 4 * n4 + tid; k < cols; k += blockDim.x) {
        const float v = __ldg(xr + k);
        xr_note(mx, nf, v);
        ss = fmaf(v, v, ss);
      }
    } else {
      for (int k = tid; k < cols; k += blockDim.x) {
        const float v = __ldg(xr + k);
        xr_note(mx, nf, v);
        ss = fmaf(v, v, ss);
      }
    }
    xr_commit(mx, nf, &s_mx, &s_nf);
  }
  float inv = 1.f;
  if (xform == EGT_INPUT_RMSNORM) {
    ss = warp_sum(ss);
    if ((tid & 31) == 0) s_ss[tid >> 5] = ss;
  }
  __syncthreads();
  if (xform == EGT_INPUT_RMSNORM) {
    float tot = 0.f;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += s_ss[w];
    inv = 1.0f / sqrtf(tot / static_cast<float>(cols) + eps);
  }
  // range of the transformed row: max |x| * inv (inv > 0), or none when inv = 0
  const uint32_t tmx = xform == EGT_INPUT_RMSNORM ? (__float_as_uint(__uint_as_float(s_mx) * inv) & 0x7fffffffu) : s_mx;
  const int e = xr_exp(tmx < 0x7f800000u ? tmx : 0u);
  const float sc = xr_pow2(e);
  if (tid == 0) {
    unsc[tok] = xr_pow2(-e);
    nonfin[tok] = s_nf;
    tinv[tok] = inv;
  }
  const int N = 2 * T, tl = tok % T, tile = tok / T;
  const uint32_t stage_bytes = static_cast<uint32_t>(N) * kStageK * 2;
  for (int ch = tid; ch < KS * (kStageK / 8); ch += blockDim.x) {
    const int ks = ch / (kStageK / 8), cin = ch % (kStageK / 8), k0 = ch * 8;
    float xv[8];
    if (tok < M && vec && k0 + 8 <= cols) {
      const float4 a0 = __ldg(reinterpret_cast<const float4*>(xr + k0));
      const float4 a1 = __ldg(reinterpret_cast<const float4*>(xr + k0 + 4));
      xv[0] = a0.x; xv[1] = a0.y; xv[2] = a0.z; xv[3] = a0.w;
      xv[4] = a1.x; xv[5] = a1.y; xv[6] = a1.z; xv[7] = a1.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = tok < M && k0 + u < cols ? __ldg(xr + k0 + u) : 0.f;
    }
    if (xform == EGT_INPUT_RMSNORM) {
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] *= inv;
    }
    uint32_t h[4], l[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const float v0 = xr_scaled(xv[2 * p], sc), v1 = xr_scaled(xv[2 * p + 1], sc);
      const __half h0 = __float2half_rn(v0), h1 = __float2half_rn(v1);
      const __half l0 = __float2half_rn(v0 - __half2float(h0)), l1 = __float2half_rn(v1 - __half2float(h1));
      h[p] = static_cast<uint32_t>(__half_as_ushort(h0)) | (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
      l[p] = static_cast<uint32_t>(__half_as_ushort(l0)) | (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
    }
    uint8_t* st = xf + (static_cast<size_t>(tile) * KS + ks) * stage_bytes;
    const int nh = tl, nl = T + tl;
    *reinterpret_cast<uint4*>(st + sw128(nh, 16 * cin)) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(st + sw128(nl, 16 * cin)) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

struct UmmaPlan {
  int T = 0, TT = 0, S = 1, KQC = 0;
  size_t smem = 0;
};

void* pick_umma(int fmt);

// Clusters of S CTAs (one CTA per SM) the GPU runs at once: a cluster's CTAs
// share a GPC, so S that do not divide a GPC's SM count leave SMs idle (the
// occupancy API answers for this GPU; cached per S)
int umma_cluster_capacity(int fmt, int S, int num_sms) {
  static int cap[3][9] = {};
  const int f = fmt == I4_SP24 ? 0 : fmt == I4_DENSE ? 1 : 2;
  if (S < 1 || S > 8) return std::max(1, num_sms / std::max(1, S));
  if (cap[f][S] == 0) {
    int n = 0;
    void* fn = pick_umma(fmt);
    const int smem = 200 * 1024;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1, 1, S);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 1;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = S;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) n = 0;
    }
    cudaGetLastError();
    cap[f][S] = n > 0 ? n : std::max(1, num_sms / S);
    if (getenv("EGT_PLAN_LOG")) fprintf(stderr, "umma cluster capacity S=%d: %d clusters\n", S, cap[f][S]);
  }
  return cap[f][S];
}

UmmaPlan plan_umma(const egt_dev_packed* h, int M, int num_sms, int nseg = 1) {
  UmmaPlan p;
  const int tiles = (M + kMaxT - 1) / kMaxT;
  p.T = ((M + tiles - 1) / tiles + 15) / 16 * 16;  // the MMA's N: a multiple of 16
  p.TT = (M + p.T - 1) / p.T;
  const int KQ = h->tiled.KQ;
  const int R = nseg * ((h->tiled.RT + 7) / 8);
  // cost ~ waves x (k-quads per CTA + a fixed CTA cost of ~8 k-quads for the
  // prologue and pipeline fill + ~6 / S for the output tail, which handles a
  // 1/S share of the tile); fitted to EGT_UMMA_S sweeps of tools/umma_probe.py
  // with the pushed split-K partials (7B shapes, M = 80 / 130 / 272: e.g.
  // 11008 x 4096 at M = 80 S = 1 46.3 us vs S = 3 43.8; 4096 x 11008 at M =
  // 130 S = 1 107 us vs S = 2 66; 4096^2 at M = 272 S = 1 51 us vs S = 2
  // 55); waves count the clusters the GPU holds at once (S = 3 packs badly:
  // 4096^2 at M = 272 63 us in three waves).  Clusters of 7-8 slices measured
  // poorly (4096^2 at M = 80: S = 8 37.7 us vs S = 6 30.7): S <= 6.
  double best = 1e300;
  static const int s_env = getenv("EGT_UMMA_S") ? atoi(getenv("EGT_UMMA_S")) : 0;  // tuning
  for (int S = 1; S <= std::min(s_env > 0 ? 8 : 6, KQ); ++S) {  // S CTAs form one cluster
    if (s_env > 0 && S != std::min(s_env, KQ)) continue;
    const int kqc = (KQ + S - 1) / S;
    const int Seff = (KQ + kqc - 1) / kqc;
    const long long clusters = static_cast<long long>(R) * p.TT;
    const double waves = std::ceil(static_cast<double>(clusters) / umma_cluster_capacity(h->format, Seff, num_sms));
    const double cost = waves * (kqc + 8.0 + 6.0 / Seff);
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
                               (has_scales(fmt) ? raw_kq(fmt) * E * 80 : 0));
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

unsigned long long* umma_trace_buffer() {
  static unsigned long long* b = [] {
    unsigned long long* p = nullptr;
    if (getenv("EGT_UMMA_TRACE")) {
      cudaMalloc(&p, 8 * 1024);
      cudaMemset(p, 0, 8 * 1024);
    }
    return p;
  }();
  return b;
}

bool umma_eligible(const egt_dev_packed* h, int M) {
  static const bool off = getenv("EGT_NO_UMMA") != nullptr;
  // from 9 tokens (tools/umma_probe.py, UMMA_PROBE_M=2,4,8,16: the tcgen05
  // kernel is flat in M up to its 96-token tile -- 16 / 39 / 31 us for 4096^2,
  // 11008 x 4096, 4096 x 11008 -- while the mma.sp token-tiled kernel grows:
  // 19 / 25 / 28 us at M = 8, 34 / 88 / 91 us at M = 16)
  static const int min_m = getenv("EGT_UMMA_MIN_M") ? atoi(getenv("EGT_UMMA_MIN_M")) : 9;
  if (off || M < min_m || h->path != 0) return false;
  const int f = h->format;
  if (f != I4_SP24 && f != I4_DENSE && f != F16_SP24) return false;
  if (has_scales(f) && h->tiled.SS != 4 && h->tiled.SS != 2) return false;
  // measured (tools/umma_probe.py, B200, k-quad ring slots): faster than the
  // mma.sp kernel at every 7B verify shape, M = 80 and 272
  return true;
}

size_t umma_workspace_bytes(const egt_dev_packed* h, int M) {
  const int tiles = (M + kMaxT - 1) / kMaxT;
  const int T = ((M + tiles - 1) / tiles + 15) / 16 * 16;
  const int TT = (M + T - 1) / T;
  const size_t KS = 2 * static_cast<size_t>(h->tiled.KQ);
  return static_cast<size_t>(TT) * KS * (2 * T) * kStageK * 2 + static_cast<size_t>(TT) * T * 12;
}

// split-K partials stay on chip (cluster DSMEM): no global workspace
size_t umma_partial_floats(const egt_dev_packed*, int, int) { return 0; }
size_t umma_counters(const egt_dev_packed*, int, int) { return 0; }

// The handle's three 2-D tensor maps (built once, kept on the handle): rows
// = the handle's row tiles, inner = its k-quads' bytes as int64 elements.
struct UmmaMaps {
  CUtensorMap vals, meta, zps, scales;
};

cudaError_t encode_2d(CUtensorMap* m, const void* base, uint64_t inner_elems, uint64_t rows, uint64_t pitch_bytes,
                      uint32_t box_inner) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {inner_elems, rows};
  const cuuint64_t strides[1] = {pitch_bytes};
  const cuuint32_t box[2] = {box_inner, 8};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t umma_maps(const egt_dev_packed* h, const UmmaMaps** out) {
  std::lock_guard<std::mutex> lk(h->plan_mu);
  if (!h->umma_maps) {
    auto m = std::make_shared<UmmaMaps>();
    const int f = h->format, KQ = h->tiled.KQ, RT = h->tiled.RT, E = h->tiled.E, kr = raw_kq(f);
    const int VB = val_lane_bytes(f), MB = meta_lane_bytes(f);
    const size_t rt0 = static_cast<size_t>(h->tiled.rt_begin) * KQ;
    cudaError_t e = encode_2d(&m->vals, h->tiled.vals + rt0 * 32 * VB, static_cast<uint64_t>(KQ) * 32 * VB / 8, RT,
                              static_cast<uint64_t>(KQ) * 32 * VB, kr * 32 * VB / 8);
    if (e == cudaSuccess && MB > 0)
      e = encode_2d(&m->meta, h->tiled.meta + rt0 * 32 * MB, static_cast<uint64_t>(KQ) * 32 * MB / 8, RT,
                    static_cast<uint64_t>(KQ) * 32 * MB, kr * 32 * MB / 8);
    if (e == cudaSuccess && has_scales(f))
      e = encode_2d(&m->zps, h->tiled.zps + rt0 * E * 16, static_cast<uint64_t>(KQ) * E * 2, RT,
                    static_cast<uint64_t>(KQ) * E * 16, kr * E * 2);
    if (e == cudaSuccess && has_scales(f))
      e = encode_2d(&m->scales, h->tiled.scales + rt0 * E * 16, static_cast<uint64_t>(KQ) * E * 8, RT,
                    static_cast<uint64_t>(KQ) * E * 64, kr * E * 8);
    if (e != cudaSuccess) return e;
    h->umma_maps = m;
  }
  *out = static_cast<const UmmaMaps*>(h->umma_maps.get());
  return cudaSuccess;
}

cudaError_t launch_umma(const egt_dev_packed* h, const float* x, int ldx, int M, float* y, int ldy,
                        uint8_t* ws, const LaunchCtx& ctx, int num_sms) {
  return launch_umma_multi(&h, 1, x, ldx, M, &y, ldy, ws, ctx, num_sms);
}

// One launch over nseg same-shape matrices (Q, K, V of a layer): one x
// preparation, CTAs blockIdx.x = segment * RB1 + 128-row block.
cudaError_t launch_umma_multi(const egt_dev_packed* const* hs, int nseg, const float* x, int ldx, int M,
                              float* const* ys, int ldy, uint8_t* ws, const LaunchCtx& ctx, int num_sms) {
  if (nseg < 1 || nseg > kMaxSeg) return cudaErrorInvalidValue;
  const egt_dev_packed* h = hs[0];
  const UmmaMaps* segmaps[kMaxSeg] = {};
  for (int i = 0; i < nseg; ++i) {
    const cudaError_t e = umma_maps(hs[i], &segmaps[i]);
    if (e != cudaSuccess) return e;
  }
  const UmmaPlan p = plan_umma(h, M, num_sms, nseg);
  const int KS = 2 * h->tiled.KQ;
  uint8_t* xf = ws;
  float* unsc = reinterpret_cast<float*>(ws + static_cast<size_t>(p.TT) * KS * (2 * p.T) * kStageK * 2);
  uint32_t* nonfin = reinterpret_cast<uint32_t*>(unsc + p.TT * p.T);
  float* tinv = reinterpret_cast<float*>(nonfin + p.TT * p.T);
  int xform = ctx.xform;
  float eps = ctx.eps;
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
    void* xargs[] = {const_cast<float**>(&x), &ldx, &M, &cols, &T, &ks, &xf, &unsc, &nonfin, &tinv, &xform, &eps};
    cudaError_t e = cudaLaunchKernelExC(&xc, reinterpret_cast<void*>(&umma_xprep_kernel), xargs);
    if (e != cudaSuccess) return e;
    ++launch_counter();
  }
  UmmaArgs a;
  a.nseg = nseg;
  a.RB1 = (h->tiled.RT + 7) / 8;
  for (int i = 0; i < nseg; ++i) {
    a.tm[i][0] = segmaps[i]->vals;
    a.tm[i][1] = segmaps[i]->meta;
    a.tm[i][2] = segmaps[i]->zps;
    a.tm[i][3] = segmaps[i]->scales;
    a.vals[i] = hs[i]->tiled.vals;
    a.meta[i] = hs[i]->tiled.meta;
    a.scales[i] = hs[i]->tiled.scales;
    a.zps[i] = hs[i]->tiled.zps;
    a.rt_begin[i] = hs[i]->tiled.rt_begin;
    a.y[i] = ys[i];
  }
  a.KQ = h->tiled.KQ;
  a.RT = h->tiled.RT;
  a.rows = static_cast<int>(h->rows);
  a.SS = h->tiled.SS;
  a.E = h->tiled.E;
  a.xf = xf;
  a.unsc = unsc;
  a.tinv = xform == EGT_INPUT_RMSNORM ? tinv : nullptr;
  a.nonfin = nonfin;
  a.x = x;
  a.ldx = ldx;
  a.cols = static_cast<int>(h->cols);
  a.M = M;
  a.T = p.T;
  a.N = 2 * p.T;
  a.TTpad = p.TT * p.T;
  a.KS = KS;
  a.KQC = p.KQC;
  a.S = p.S;
  // x multicast over row-block pairs: measured no faster (A/B at the 7B
  // shapes, M = 272: within 2 %) -- the L2 x reads are not what bounds the
  // kernel; kept as an option (EGT_UMMA_MCAST=1)
  static const bool mcast = getenv("EGT_UMMA_MCAST") != nullptr;
  a.mcast = mcast && p.S == 1 && p.TT > 1 && (nseg * a.RB1) % 2 == 0 ? 1 : 0;
  // split-K partials pushed by bulk copies (default; EGT_UMMA_PULL=1: the
  // DSMEM-load reduction): 4096^2 at M = 80 23.2 -> 20.2 us, the verify pass
  // at 64 nodes 6.22 -> 5.98 ms (tools/umma_probe.py, verify_probe.py)
  static const bool pull = getenv("EGT_UMMA_PULL") != nullptr;
  a.push = pull ? 0 : 1;
  a.ldy = ldy;
  a.res = ctx.res;
  a.ldr = ctx.ldr;
  a.out_silu = ctx.out_silu;
  a.partial = ctx.partial;
  a.counters = ctx.counters;
  a.pad14 = h->tiled.pad14;
  a.raw_rt_bytes = raw_rt_bytes(h->format, h->tiled.E);
  a.trace = umma_trace_buffer();
  static const int udbg = getenv("EGT_UMMA_DBG") ? atoi(getenv("EGT_UMMA_DBG")) : 0;
  a.dbg = udbg;
  void* fn = pick_umma(h->format);
  cudaFuncAttributes fa{};
  cudaError_t err = cudaFuncGetAttributes(&fa, fn);
  if (err != cudaSuccess) return err;
  const size_t budget = 227 * 1024 - fa.sharedSizeBytes;  // dynamic + static shared memory per block
  const size_t x_bytes = static_cast<size_t>(a.N) * kStageK * 2;
  const bool sparse_path = h->format != I4_DENSE && getenv("EGT_UMMA_DENSE") == nullptr;
  // ring slots are k-quads: two A stages (8 / 16 KB each), two x stages
  const size_t a_bytes = 2 * (sparse_path ? 8192 : 16384), xu_bytes = 2 * x_bytes;
  const size_t fixed = 2048 + kNR * 8 * static_cast<size_t>(a.raw_rt_bytes);
  // split K: the x ring also holds the slice's partials, 128 x (T + 4) f32
  // push: the tile (T x 512 B) plus the receive area (S shares of per groups x 2 KB)
  const size_t g4 = p.T / 4, per = (g4 + p.S - 1) / p.S;
  const size_t push_bytes = static_cast<size_t>(p.T) * 512 + (p.S > 1 ? p.S * per * 2048 : 0);
  const size_t pull_bytes = p.S > 1 ? 512 * static_cast<size_t>(p.T + 4) : 0;
  static const int na_env = getenv("EGT_UMMA_NA") ? atoi(getenv("EGT_UMMA_NA")) : 0;
  const long room = static_cast<long>(budget) - static_cast<long>(fixed);
  a.NA = room > 0 ? static_cast<int>(std::min<long>(kMaxNA, room / static_cast<long>(a_bytes + xu_bytes))) : 0;
  if (na_env > 0) a.NA = std::min(a.NA, na_env);
  a.NX = a.NA;  // one ring
  if (a.push && static_cast<size_t>(a.NX) * xu_bytes < push_bytes) a.push = 0;  // no room: pull
  const int nx_min = static_cast<int>(((a.push ? push_bytes : pull_bytes) + xu_bytes - 1) / xu_bytes);
  if (a.NA < std::max(2, nx_min)) return cudaErrorInvalidConfiguration;
  const size_t smem = fixed + a.NA * a_bytes + a.NX * xu_bytes;
  err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nseg * a.RB1, p.TT, p.S);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx.stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;  // the split-K slices of a row block (or row-block pairs)
  attr[0].val.clusterDim.x = a.mcast ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = p.S;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 2 : 1;
  void* args[] = {&a};
  err = cudaLaunchKernelExC(&cfg, fn, args);
  if (err == cudaSuccess) ++launch_counter();
  return err;
}

}  // namespace egt_impl
