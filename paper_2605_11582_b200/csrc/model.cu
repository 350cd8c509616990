// The multi-token pass of prefix-tree verification on the device: the
// reference's forward_impl (model.cpp:118-202) over packed layers.
//   x = embedding[token] + positions[pos]                    (model.cpp:141-143)
//   per layer: a = rmsnorm(x); q,k,v = a W^T (SparseGemv, M rows)
//              per head: s = (q k^T) * scale, masked softmax, empty row -> 0
//              x += o Wo^T; b = rmsnorm(x); x += silu(b ff1^T) ff2^T
//   logits = rmsnorm(x) head^T
// The linear layers are the tensor-core SpGEMM of spmm_tiled.cu (any of the
// mixed-dispatch formats); the rest are small f32 kernels here.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "egt_b200.h"
#include "handle.h"
#include "model.h"

namespace egt_impl {
void set_last_error(const std::string& msg);
}

namespace {

using egt_impl::launch_counter;

constexpr float kNormEps = 1e-6f;  // model.cpp:27

__global__ void embed_kernel(const int* tok, const int* pos, const float* emb, const float* ptab,
                             float* x, int M, int d) {
  const int i = blockIdx.x;
  for (int c = threadIdx.x; c < d; c += blockDim.x)
    x[static_cast<size_t>(i) * d + c] = emb[static_cast<size_t>(tok[i]) * d + c] + ptab[static_cast<size_t>(pos[i]) * d + c];
}

// rmsnorm (model.cpp:57-67): y = x / sqrt(mean(x^2) + eps), one block per row.
__global__ void rmsnorm_kernel(const float* x, float* y, int d) {
  const float* xr = x + static_cast<size_t>(blockIdx.x) * d;
  float ss = 0.f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) ss = fmaf(xr[c], xr[c], ss);
  __shared__ float red[32];
  ss = egt_dev::warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = egt_dev::warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / static_cast<float>(d) + kNormEps);
  float* yr = y + static_cast<size_t>(blockIdx.x) * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) yr[c] = xr[c] * inv;
}

// rmsnorm for rows of d % 4 == 0, d <= 4 * 4 * blockDim: one read of x
// (float4 in registers), then the scaled write.
__global__ void __launch_bounds__(1024) rmsnorm4_kernel(const float* x, float* y, int d) {
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(blockIdx.x) * d);
  float4* yr = reinterpret_cast<float4*>(y + static_cast<size_t>(blockIdx.x) * d);
  const int n4 = d / 4;
  float4 vals[4];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    vals[i] = c < n4 ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    ss = fmaf(vals[i].x, vals[i].x, ss);
    ss = fmaf(vals[i].y, vals[i].y, ss);
    ss = fmaf(vals[i].z, vals[i].z, ss);
    ss = fmaf(vals[i].w, vals[i].w, ss);
  }
  __shared__ float red[32];
  ss = egt_dev::warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = egt_dev::warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / static_cast<float>(d) + kNormEps);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < n4) yr[c] = make_float4(vals[i].x * inv, vals[i].y * inv, vals[i].z * inv, vals[i].w * inv);
  }
}

// Batched f32 GEMM tile kernel for attention: C[b](i,j) = alpha * sum_k A[b](i,k) * B'[b](k,j)
// with B' = B^T (BT: B is [n x K] row-major) or B (B is [K x n]).
template <bool BT>
__global__ void attn_gemm_kernel(const float* A, int lda, size_t sa, const float* B, int ldb, size_t sb,
                                 float* C, int ldc, size_t sc, int m, int n, int K, float alpha) {
  __shared__ float As[16][17];
  __shared__ float Bs[16][17];
  const int b = blockIdx.z;
  const int ty = threadIdx.y, tx = threadIdx.x;
  const int i = blockIdx.y * 16 + ty, j = blockIdx.x * 16 + tx;
  A += b * sa;
  B += b * sb;
  C += b * sc;
  float acc = 0.f;
  for (int k0 = 0; k0 < K; k0 += 16) {
    const int ka = k0 + tx, kb = k0 + ty;
    As[ty][tx] = (i < m && ka < K) ? A[static_cast<size_t>(i) * lda + ka] : 0.f;
    if (BT)
      Bs[ty][tx] = (blockIdx.x * 16 + ty < n && k0 + tx < K) ? B[static_cast<size_t>(blockIdx.x * 16 + ty) * ldb + k0 + tx] : 0.f;
    else
      Bs[ty][tx] = (kb < K && j < n) ? B[static_cast<size_t>(kb) * ldb + j] : 0.f;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) acc = fmaf(As[ty][kk], BT ? Bs[tx][kk] : Bs[kk][tx], acc);
    __syncthreads();
  }
  if (i < m && j < n) C[static_cast<size_t>(i) * ldc + j] = acc * alpha;
}

// Masked softmax of one score row per warp (model.cpp:169-182); a query row
// with no visible key becomes all zeros (model.cpp:173).  mask: bit q*M+k.
__global__ void masked_softmax_kernel(float* S, const uint8_t* mask, int M, int H) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M * H) return;
  const int q = row % M;
  float* s = S + static_cast<size_t>(row) * M;
  auto vis = [&](int k) {
    const size_t bit = static_cast<size_t>(q) * M + k;
    return (mask[bit >> 3] >> (bit & 7)) & 1;
  };
  float m = -INFINITY;
  for (int k = lane; k < M; k += 32)
    if (vis(k)) m = fmaxf(m, s[k]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (!isfinite(m)) {
    for (int k = lane; k < M; k += 32) s[k] = 0.f;
    return;
  }
  float z = 0.f;
  for (int k = lane; k < M; k += 32) {
    const float e = vis(k) ? expf(s[k] - m) : 0.f;
    s[k] = e;
    z += e;
  }
  z = egt_dev::warp_sum(z);
  for (int k = lane; k < M; k += 32) s[k] = s[k] / z;
}

// Fused masked attention for one head and 16 query rows (model.cpp:161-184:
// s = (q k^T) * scale, masked softmax with an empty row -> 0, o = p V), so the
// M x M scores never leave shared memory.  Block (query tile, head), 256
// threads; smem: q tile [16][dh + 4] and scores [16][M].
constexpr int kAttnRows = 16;
__global__ void __launch_bounds__(256) fused_attention_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                              const float* __restrict__ v, float* __restrict__ o,
                                                              const uint8_t* __restrict__ mask, int M, int d, int dh,
                                                              float scale) {
  extern __shared__ float sm[];
  const int ldq = dh + 4;
  float* qs = sm;                          // [16][dh + 4]
  float* ps = sm + kAttnRows * ldq;        // [16][M]
  const int q0 = blockIdx.x * kAttnRows, h = blockIdx.y, tid = threadIdx.x;
  const int nr = min(kAttnRows, M - q0);
  const size_t hoff = static_cast<size_t>(h) * dh;
  for (int i = tid; i < kAttnRows * dh; i += blockDim.x) {
    const int r = i / dh, e = i % dh;
    qs[r * ldq + e] = r < nr ? q[static_cast<size_t>(q0 + r) * d + hoff + e] : 0.f;
  }
  __syncthreads();
  // scores: thread -> (key j, row r), 16 consecutive threads share key j
  for (int idx = tid; idx < kAttnRows * M; idx += blockDim.x) {
    const int r = idx % kAttnRows, j = idx / kAttnRows;
    float acc = 0.f;
    if (r < nr) {
      const float4* kr = reinterpret_cast<const float4*>(k + static_cast<size_t>(j) * d + hoff);
      const float4* qr = reinterpret_cast<const float4*>(qs + r * ldq);
      for (int e = 0; e < dh / 4; ++e) {
        const float4 a = qr[e], b = __ldg(kr + e);
        acc = fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, acc))));
      }
    }
    const size_t bit = static_cast<size_t>(q0 + r) * M + j;
    const bool vis = r < nr && ((mask[bit >> 3] >> (bit & 7)) & 1);
    ps[r * M + j] = vis ? acc * scale : -INFINITY;
  }
  __syncthreads();
  // softmax: two rows per warp
  const int lane = tid & 31, warp = tid >> 5;
  for (int r = warp; r < kAttnRows; r += blockDim.x >> 5) {
    float* pr = ps + r * M;
    float m = -INFINITY;
    for (int j = lane; j < M; j += 32) m = fmaxf(m, pr[j]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (!isfinite(m)) {  // no visible key: zero attention output (model.cpp:173)
      for (int j = lane; j < M; j += 32) pr[j] = 0.f;
      continue;
    }
    float z = 0.f;
    for (int j = lane; j < M; j += 32) {
      const float e = pr[j] == -INFINITY ? 0.f : expf(pr[j] - m);
      pr[j] = e;
      z += e;
    }
    z = egt_dev::warp_sum(z);
    const float iz = 1.0f / z;
    for (int j = lane; j < M; j += 32) pr[j] *= iz;
  }
  __syncthreads();
  // o = p V: thread -> column e, rows rg*8 .. rg*8+7
  for (int c = tid; c < dh * (kAttnRows / 8); c += blockDim.x) {
    const int e = c % dh, rg = c / dh;
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    for (int j = 0; j < M; ++j) {
      const float vv = __ldg(v + static_cast<size_t>(j) * d + hoff + e);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fmaf(ps[(rg * 8 + i) * M + j], vv, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (rg * 8 + i < nr) o[static_cast<size_t>(q0 + rg * 8 + i) * d + hoff + e] = acc[i];
  }
}

// The same masked attention for 32 query rows per block, the head's keys
// and values streamed through shared memory in double-buffered chunks of 32
// rows (cp.async, zero-filled past M): scores s[r][j] (phase 1, thread = key
// of the chunk x 4 rows), the exact two-pass masked softmax per row (phase
// 2, as above), o = p V (phase 3, thread = float4 column x 4 rows).  256
// threads, two blocks per SM; smem: q [32][dh + 4], scores [32][ldp], K / V
// chunks 2 x [32][dh + 4].
// The 16-row kernel above re-read every key row from L2 per (row, key) pair
// and ran latency-bound (152 us per layer at M = 272, dh = 128).
constexpr int kAttnRows2 = 32, kAttnKeys = 32;
__host__ __device__ inline int attn2_ldp(int M) {  // +4: conflict-free A-fragment reads of the scores
  return (M + kAttnKeys - 1) / kAttnKeys * kAttnKeys + 4;
}
// resident: every key / value chunk in shared memory at once (one L2 round
// trip for K, one for V; otherwise a double-buffered ring of chunks, each a
// round trip on the critical path: measured latency-bound, 68 us per layer at
// M = 272 whatever the arithmetic)
__host__ __device__ inline size_t attn2_smem(int M, int dh, bool resident = false) {
  const int ldp = attn2_ldp(M), nchunk = (M + kAttnKeys - 1) / kAttnKeys;
  return (static_cast<size_t>(kAttnRows2) * (dh + 4) + static_cast<size_t>(kAttnRows2) * ldp +
          (resident ? nchunk : 2) * static_cast<size_t>(kAttnKeys) * (dh + 4)) * sizeof(float);
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(egt_dev::smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
// f32 = tf32 hi + tf32 lo (~21 bits); a product of two split values kept to
// three tensor-core terms (hi*hi + hi*lo + lo*hi: the dropped lo*lo is
// ~2^-22 of it), accumulated in f32
// The tf32 MMA reads the top 19 bits of each f32 register (truncation), so
// the split is a mask and an exact subtraction (cvt.rna.tf32 compiles to ~5
// instructions and made the kernel issue-bound: 69 us at M = 272).
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  const uint32_t h = __float_as_uint(x) & 0xffffe000u;
  hi = h;
  lo = __float_as_uint(x - __uint_as_float(h));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// d += A (16 x 8, rows g / g + 8, columns t / t + 4) * B (8 x 8, k t / t + 4, n g), 3xTF32
__device__ __forceinline__ void mma_3xtf32(float (&d)[4], const float (&a)[4], const float (&b)[2]) {
  uint32_t ah[4], al[4], bh[2], bl[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) tf32_split(a[i], ah[i], al[i]);
  tf32_split(b[0], bh[0], bl[0]);
  tf32_split(b[1], bh[1], bl[1]);
  mma_tf32(d, al[0], al[1], al[2], al[3], bh[0], bh[1]);
  mma_tf32(d, ah[0], ah[1], ah[2], ah[3], bl[0], bl[1]);
  mma_tf32(d, ah[0], ah[1], ah[2], ah[3], bh[0], bh[1]);
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// MMA: q k^T and p V on the tensor cores in 3xTF32 (dh % 32 == 0): warp w
// owns rows 16 (w & 1) and keys 8 (w >> 1) of a chunk (scores), rows 16 (w & 1)
// and columns dh / 4 * (w >> 1) (output).
template <bool MMA>
__global__ void __launch_bounds__(256) attention_tile_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                             const float* __restrict__ v, float* __restrict__ o,
                                                             const uint8_t* __restrict__ mask, int M, int d, int dh,
                                                             float scale, int resident) {
  extern __shared__ __align__(16) float sm[];
  const int ldq = dh + 4, ldp = attn2_ldp(M), n4 = dh / 4;
  float* qs = sm;                     // [32][dh + 4]
  float* ps = qs + kAttnRows2 * ldq;  // [32][ldp]
  float* kb = ps + kAttnRows2 * ldp;  // 2 (resident: nchunk) x [32][dh + 4]
  const int q0 = blockIdx.x * kAttnRows2, h = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = min(kAttnRows2, M - q0);
  const size_t hoff = static_cast<size_t>(h) * dh;
  const int nchunk = (M + kAttnKeys - 1) / kAttnKeys;
  // chunk c of keys (src = k) or values (src = v) into buffer c & 1 (resident: c)
  auto buf = [&](int c) { return kb + (resident ? c : (c & 1)) * kAttnKeys * ldq; };
  auto stage = [&](const float* src, int c) {
    float* dst = buf(c);
    for (int f = tid; f < kAttnKeys * n4; f += blockDim.x) {
      const int key = f / n4, e4 = f % n4, kk = c * kAttnKeys + key;
      cp_async16(dst + key * ldq + 4 * e4, src + static_cast<size_t>(kk < M ? kk : 0) * d + hoff + 4 * e4, kk < M);
    }
    cp_async_commit();
  };
  for (int c = 0; c < (resident ? nchunk : 1); ++c) stage(k, c);
  for (int f = tid; f < kAttnRows2 * n4; f += blockDim.x) {
    const int r = f / n4, e4 = f % n4;
    cp_async16(qs + r * ldq + 4 * e4, q + static_cast<size_t>(r < nr ? q0 + r : q0) * d + hoff + 4 * e4, r < nr);
  }
  cp_async_commit();
  // ---- phase 1: scores; thread -> key `lane` of the chunk, rows 4 warp .. 4 warp + 3
  for (int c = 0; c < nchunk; ++c) {
    if (!resident) {
      if (c + 1 < nchunk) stage(k, c + 1); else cp_async_commit();
      cp_async_wait1();  // chunk c (and q) landed
      __syncthreads();
    } else if (c == 0) {
      cp_async_wait0();  // every chunk and q
      __syncthreads();
    }
    const float* ks = buf(c);
    if constexpr (MMA) {
      const int g = lane >> 2, t = lane & 3, rm = 16 * (warp & 1), kn = 8 * (warp >> 1);
      float dacc[4] = {0.f, 0.f, 0.f, 0.f};
      const float* qa = qs + (rm + g) * ldq + t;
      const float* kbp = ks + (kn + g) * ldq + t;
#pragma unroll 4
      for (int e0 = 0; e0 < dh; e0 += 8) {
        const float af[4] = {qa[e0], qa[8 * ldq + e0], qa[e0 + 4], qa[8 * ldq + e0 + 4]};
        const float bf[2] = {kbp[e0], kbp[e0 + 4]};
        mma_3xtf32(dacc, af, bf);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = rm + g + 8 * (i >> 1), kk = c * kAttnKeys + kn + 2 * t + (i & 1);
        const size_t bit = static_cast<size_t>(q0 + r) * M + kk;
        const bool vis = r < nr && kk < M && ((mask[bit >> 3] >> (bit & 7)) & 1);
        ps[r * ldp + kk] = vis ? dacc[i] * scale : -INFINITY;
      }
      __syncthreads();
      continue;
    }
    float acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = 0.f;
    const float4* kr = reinterpret_cast<const float4*>(ks + lane * ldq);
#pragma unroll 4
    for (int e4 = 0; e4 < n4; ++e4) {
      const float4 b = kr[e4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 a = *reinterpret_cast<const float4*>(qs + (4 * warp + i) * ldq + 4 * e4);
        acc[i] = fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, acc[i]))));
      }
    }
    const int kk = c * kAttnKeys + lane;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = 4 * warp + i;
      const size_t bit = static_cast<size_t>(q0 + r) * M + kk;
      const bool vis = r < nr && kk < M && ((mask[bit >> 3] >> (bit & 7)) & 1);
      ps[r * ldp + kk] = vis ? acc[i] * scale : -INFINITY;
    }
    __syncthreads();  // buffer c & 1 free for chunk c + 2
  }
  // values stream in while the softmax runs (the keys' last reads are
  // behind the loop's final barrier)
  for (int c = 0; c < (resident ? nchunk : 1); ++c) stage(v, c);
  // ---- phase 2: masked softmax, one warp per row (an empty row -> 0)
  for (int r = warp; r < kAttnRows2; r += blockDim.x >> 5) {
    float* pr = ps + r * ldp;
    float m = -INFINITY;
    for (int j = lane; j < M; j += 32) m = fmaxf(m, pr[j]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (!isfinite(m)) {  // no visible key: zero attention output (model.cpp:173)
      for (int j = lane; j < ldp; j += 32) pr[j] = 0.f;
      continue;
    }
    float z = 0.f;
    for (int j = lane; j < M; j += 32) {
      const float e = pr[j] == -INFINITY ? 0.f : expf(pr[j] - m);
      pr[j] = e;
      z += e;
    }
    z = egt_dev::warp_sum(z);
    const float iz = 1.0f / z;
    for (int j = lane; j < ldp; j += 32) pr[j] = j < M ? pr[j] * iz : 0.f;
  }
  // ---- phase 3: o = p V; thread -> float4 column e4, rows 4 rg .. 4 rg + 3
  const int items = (kAttnRows2 / 4) * n4;
  const int e4 = tid % n4, rg = tid / n4;
  float4 acc[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  float oacc[4][4];  // MMA: n-tiles of 8 columns x (rows g / g + 8, columns 2t / 2t + 1)
#pragma unroll
  for (int i = 0; i < 4; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  for (int c = 0; c < nchunk; ++c) {
    if (!resident) {
      if (c + 1 < nchunk) stage(v, c + 1); else cp_async_commit();
      cp_async_wait1();
      __syncthreads();  // chunk c landed; scores final
    } else if (c == 0) {
      cp_async_wait0();
      __syncthreads();
    }
    if constexpr (MMA) {
      const int g = lane >> 2, t = lane & 3, rm = 16 * (warp & 1), cn = (dh / 4) * (warp >> 1);
      const float* vs = buf(c);
      const float* pa = ps + (rm + g) * ldp + c * kAttnKeys + t;
#pragma unroll
      for (int k0 = 0; k0 < kAttnKeys; k0 += 8) {
        const float af[4] = {pa[k0], pa[8 * ldp + k0], pa[k0 + 4], pa[8 * ldp + k0 + 4]};
        uint32_t ah[4], al[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) tf32_split(af[i], ah[i], al[i]);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          if (8 * nt < dh / 4) {
            const float* vb = vs + (k0 + t) * ldq + cn + 8 * nt + g;
            uint32_t bh0, bl0, bh1, bl1;
            tf32_split(vb[0], bh0, bl0);
            tf32_split(vb[4 * ldq], bh1, bl1);
            mma_tf32(oacc[nt], al[0], al[1], al[2], al[3], bh0, bh1);
            mma_tf32(oacc[nt], ah[0], ah[1], ah[2], ah[3], bl0, bl1);
            mma_tf32(oacc[nt], ah[0], ah[1], ah[2], ah[3], bh0, bh1);
          }
        }
      }
    } else if (tid < items) {
      const float* vs = buf(c);
      const float* pc = ps + (4 * rg) * ldp + c * kAttnKeys;
#pragma unroll 4
      for (int j = 0; j < kAttnKeys; ++j) {  // keys past M: zero values and zero p
        const float4 vv = *reinterpret_cast<const float4*>(vs + j * ldq + 4 * e4);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float p = pc[i * ldp + j];
          acc[i].x = fmaf(p, vv.x, acc[i].x);
          acc[i].y = fmaf(p, vv.y, acc[i].y);
          acc[i].z = fmaf(p, vv.z, acc[i].z);
          acc[i].w = fmaf(p, vv.w, acc[i].w);
        }
      }
    }
    __syncthreads();
  }
  if constexpr (MMA) {
    const int g = lane >> 2, t = lane & 3, rm = 16 * (warp & 1), cn = (dh / 4) * (warp >> 1);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      if (8 * nt >= dh / 4) break;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int r = rm + g + 8 * hh;
        if (r < nr)
          *reinterpret_cast<float2*>(o + static_cast<size_t>(q0 + r) * d + hoff + cn + 8 * nt + 2 * t) =
              make_float2(oacc[nt][2 * hh], oacc[nt][2 * hh + 1]);
      }
    }
  } else if (tid < items) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (4 * rg + i < nr)
        reinterpret_cast<float4*>(o + static_cast<size_t>(q0 + 4 * rg + i) * d + hoff)[e4] = acc[i];
  }
}

// KV pool: the keys / values of committed rows persist
// across the constrained beam steps; a row is written once and shared by
// every beam whose prefix contains it (beams re-rank by list, never copy).
// store: pool[l][rows[i]] <- k / v row i of this pass.
__global__ void kv_store_kernel(const float* __restrict__ k, const float* __restrict__ v, float* kp, float* vp,
                                const uint32_t* __restrict__ rows, int M, int d) {
  const int i = blockIdx.x;
  if (i >= M) return;
  const size_t dst = static_cast<size_t>(rows[i]) * d, src = static_cast<size_t>(i) * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    kp[dst + c] = k[src + c];
    vp[dst + c] = v[src + c];
  }
}

// One query row per block x head: keys / values = pool rows key_rows[
// key_ptr[i] .. key_ptr[i+1]) (its committed prefix, in position order) then
// its own row of this pass -- model.cpp:161-184's masked softmax over exactly
// the causal prefix of that row.  Scores in shared memory.
__global__ void __launch_bounds__(128) kv_attention_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                           const float* __restrict__ v, const float* __restrict__ kp,
                                                           const float* __restrict__ vp,
                                                           const uint32_t* __restrict__ key_ptr,
                                                           const uint32_t* __restrict__ key_rows, float* o, int d,
                                                           int dh, float scale) {
  extern __shared__ float sc[];  // [n keys]
  const int i = blockIdx.x, h = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t k0 = key_ptr[i], n = key_ptr[i + 1] - k0 + 1;
  const size_t hoff = static_cast<size_t>(h) * dh;
  const float* qr = q + static_cast<size_t>(i) * d + hoff;
  // scores: a warp per key, lanes over the head dimension
  for (uint32_t j = warp; j < n; j += blockDim.x >> 5) {
    const float* kr = j + 1 < n ? kp + static_cast<size_t>(key_rows[k0 + j]) * d + hoff
                                : k + static_cast<size_t>(i) * d + hoff;
    float acc = 0.f;
    for (int e = lane; e < dh; e += 32) acc = fmaf(qr[e], kr[e], acc);
    acc = egt_dev::warp_sum(acc);
    if (lane == 0) sc[j] = acc * scale;
  }
  __syncthreads();
  __shared__ float red[4];
  float m = -INFINITY;
  for (uint32_t j = tid; j < n; j += blockDim.x) m = fmaxf(m, sc[j]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  float z = 0.f;
  for (uint32_t j = tid; j < n; j += blockDim.x) {
    const float e = expf(sc[j] - m);
    sc[j] = e;
    z += e;
  }
  z = egt_dev::warp_sum(z);
  if (lane == 0) red[warp] = z;
  __syncthreads();
  const float iz = 1.0f / (red[0] + red[1] + red[2] + red[3]);
  // o = p V: thread per head dimension
  for (int e = tid; e < dh; e += blockDim.x) {
    float acc = 0.f;
    for (uint32_t j = 0; j < n; ++j) {
      const float* vr = j + 1 < n ? vp + static_cast<size_t>(key_rows[k0 + j]) * d + hoff
                                  : v + static_cast<size_t>(i) * d + hoff;
      acc = fmaf(sc[j] * iz, vr[e], acc);
    }
    o[static_cast<size_t>(i) * d + hoff + e] = acc;
  }
}

__global__ void silu_kernel(float* f, size_t n) {  // model.cpp:80-84
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float v = f[i];
    f[i] = v * (1.0f / (1.0f + expf(-v)));
  }
}

__global__ void add_kernel(float* x, const float* t, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    x[i] = x[i] + t[i];
}

__global__ void gather_kernel(const float* src, uint64_t ld, const uint32_t* idx, uint32_t n, float* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[static_cast<uint64_t>(idx[i]) * ld + idx[n + i]];
}

egt_status fail(egt_status s, const std::string& m) {
  egt_impl::set_last_error(m);
  return s;
}

#define MCUDA(expr)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess) return fail(EGT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

unsigned grid_for(size_t n) { return static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 4096)); }

}  // namespace

namespace {

// The prefix-tree mask straight from the compact encoding (SURVEY 8(f) row
// 4): block per row q; committed rows see their beam's committed tokens up to
// themselves (left-padded, pad rows see nothing), node rows see their beam's
// committed block plus their ancestors and themselves (build_tree_mask,
// decode.cpp:240-299).  mask: u32 words, bit q*M+k LSB-first, zeroed.
__global__ void tree_mask_kernel(uint32_t* mask, int M, int nb, int lmax, const uint32_t* committed,
                                 const int32_t* parent, const uint32_t* beam) {
  extern __shared__ uint8_t anc[];  // [n_nodes] ancestor-or-self flags of this row's node
  const int q = blockIdx.x, F = nb * lmax, nn = M - F;
  int lo = 0, hi = 0;  // committed key range [lo, hi) visible to row q
  bool node = q >= F;
  if (!node) {
    const int b = q / lmax, first = b * lmax + (lmax - static_cast<int>(committed[b]));
    if (q >= first) lo = first, hi = q + 1;
  } else {
    const int f = q - F, b = static_cast<int>(beam[f]);
    lo = b * lmax + (lmax - static_cast<int>(committed[b]));
    hi = (b + 1) * lmax;
    for (int i = threadIdx.x; i < nn; i += blockDim.x) anc[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int p = f; p >= 0; p = parent[p]) anc[p] = 1;
    __syncthreads();
  }
  for (int k = threadIdx.x; k < M; k += blockDim.x) {
    const bool vis = (k >= lo && k < hi) || (node && k >= F && anc[k - F]);
    if (vis) {
      const uint64_t bit = static_cast<uint64_t>(q) * M + k;
      atomicOr(mask + (bit >> 5), 1u << (bit & 31));
    }
  }
}

// KV-pool pass: rows of this pass are stored at pool rows out_rows; with
// key lists (key_ptr != null) the attention of row i reads the pool rows
// key_rows[key_ptr[i] .. key_ptr[i+1]) then its own row (no M x M mask).
struct KvPass {
  egt_kv_pool* pool = nullptr;
  const uint32_t* out_rows = nullptr;  // host [M]
  const uint32_t* key_ptr = nullptr;   // host [M + 1] or null
  const uint32_t* key_rows = nullptr;  // host [key_ptr[M]]
};

egt_status forward_core(const egt_model* m, const int32_t* tokens, const int32_t* positions,
                        const uint8_t* mask_bits, const egt_tree_view* tree, uint32_t M, float* logits,
                        void* stream, const KvPass* kv = nullptr) {
  if (!m || !tokens || !positions || !logits) return fail(EGT_EINVAL, "forward: null argument");
  const egt_model_config& c = m->cfg;
  if (M == 0) return fail(EGT_EINVAL, "forward: empty token sequence");  // model.cpp:123
  for (uint32_t i = 0; i < M; ++i) {                                        // model.cpp:128-135
    if (tokens[i] < 0 || static_cast<uint32_t>(tokens[i]) >= c.vocab_size)
      return fail(EGT_EINVAL, "forward: token out of range");
    if (positions[i] < 0 || static_cast<uint32_t>(positions[i]) >= c.max_positions)
      return fail(EGT_EINVAL, "forward: position out of range");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t d = c.d_model, dff = c.d_ff, H = c.n_heads, dh = d / H;
  const size_t Md = M * d;
  const size_t mask_bytes = (static_cast<size_t>(M) * M + 31) / 32 * 4;
  const size_t tree_ints = tree ? tree->n_beams + 2ull * tree->n_nodes : 0;
  const bool gather = kv && kv->key_ptr;
  const size_t kv_ints = kv ? M + (gather ? M + 1ull + kv->key_ptr[M] : 0) : 0;
  const size_t floats = 6 * Md + M * dff + (gather ? 0 : H * static_cast<size_t>(M) * M);
  char* scratch = nullptr;
  {
    // keep the stream-ordered pool's memory across passes: with the default
    // release threshold (0) every synchronisation returns it and the next
    // pass maps it again (measured: verify passes jittering 6.8 -> 11 ms)
    static bool pool_kept = false;
    if (!pool_kept) {
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      pool_kept = true;
    }
  }
  MCUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                        floats * sizeof(float) + 2 * M * sizeof(int) + mask_bytes + tree_ints * 4 + kv_ints * 4 + 64,
                        s));
  float* x = reinterpret_cast<float*>(scratch);
  float* a = x + Md;
  float* q = a + Md;
  float* k = q + Md;
  float* v = k + Md;
  float* o = v + Md;
  float* f1 = o + Md;
  float* S = f1 + M * dff;
  int* dtok = reinterpret_cast<int*>(S + (gather ? 0 : H * static_cast<size_t>(M) * M));
  int* dpos = dtok + M;
  uint8_t* dmask = reinterpret_cast<uint8_t*>(dpos + M);
  egt_status st = EGT_OK;
  auto lin = [&](const egt_dev_packed* h, const float* in, float* outp, uint32_t flags) {
    if (st == EGT_OK) st = egt_spmv_ex(h, in, outp, M, h->cols, h->rows, flags, stream);
  };
  cudaMemcpyAsync(dtok, tokens, M * sizeof(int), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dpos, positions, M * sizeof(int), cudaMemcpyHostToDevice, s);
  if (tree) {
    uint32_t* dcommit = reinterpret_cast<uint32_t*>(dmask + mask_bytes);
    int32_t* dparent = reinterpret_cast<int32_t*>(dcommit + tree->n_beams);
    uint32_t* dbeam = reinterpret_cast<uint32_t*>(dparent + tree->n_nodes);
    cudaMemsetAsync(dmask, 0, mask_bytes, s);
    if (tree->n_beams) cudaMemcpyAsync(dcommit, tree->committed_len, tree->n_beams * 4ull, cudaMemcpyHostToDevice, s);
    if (tree->n_nodes) {
      cudaMemcpyAsync(dparent, tree->parent, tree->n_nodes * 4ull, cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(dbeam, tree->beam, tree->n_nodes * 4ull, cudaMemcpyHostToDevice, s);
    }
    tree_mask_kernel<<<M, 256, tree->n_nodes, s>>>(reinterpret_cast<uint32_t*>(dmask), static_cast<int>(M),
                                                   static_cast<int>(tree->n_beams), static_cast<int>(tree->padded_len),
                                                   dcommit, dparent, dbeam);
    ++launch_counter();
  } else if (mask_bits) {
    cudaMemcpyAsync(dmask, mask_bits, (static_cast<size_t>(M) * M + 7) / 8, cudaMemcpyHostToDevice, s);
  }
  uint32_t *d_out_rows = nullptr, *d_key_ptr = nullptr, *d_key_rows = nullptr;
  if (kv) {
    d_out_rows = reinterpret_cast<uint32_t*>(dmask + mask_bytes) + tree_ints;
    cudaMemcpyAsync(d_out_rows, kv->out_rows, M * 4ull, cudaMemcpyHostToDevice, s);
    if (gather) {
      d_key_ptr = d_out_rows + M;
      d_key_rows = d_key_ptr + M + 1;
      cudaMemcpyAsync(d_key_ptr, kv->key_ptr, (M + 1ull) * 4, cudaMemcpyHostToDevice, s);
      if (kv->key_ptr[M]) cudaMemcpyAsync(d_key_rows, kv->key_rows, kv->key_ptr[M] * 4ull, cudaMemcpyHostToDevice, s);
    }
  }
  embed_kernel<<<M, 256, 0, s>>>(dtok, dpos, m->emb, m->pos, x, static_cast<int>(M), static_cast<int>(d));
  ++launch_counter();
  auto rmsnorm = [&](const float* in, float* outp) {
    if (d % 4 == 0 && d <= 16 * 1024)
      rmsnorm4_kernel<<<M, static_cast<unsigned>(std::min<size_t>(1024, (d / 4 + 31) / 32 * 32)), 0, s>>>(
          in, outp, static_cast<int>(d));
    else
      rmsnorm_kernel<<<M, 256, 0, s>>>(in, outp, static_cast<int>(d));
  };
  const float att_scale = 1.0f / std::sqrt(static_cast<float>(dh));  // model.cpp:139
  // fused attention while the 16-row score tile fits in shared memory
  const size_t attn_smem = (kAttnRows * (dh + 4) + static_cast<size_t>(kAttnRows) * M) * sizeof(float);
  static const bool no_fused = getenv("EGT_UNFUSED_ATTENTION") != nullptr;
  const bool fused_attn = !no_fused && dh % 4 == 0 && attn_smem <= 200 * 1024;
  if (fused_attn && attn_smem > 48 * 1024)
    MCUDA(cudaFuncSetAttribute(fused_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(attn_smem)));
  // the 64-row staged kernel where its tiles fit (dh <= 128)
  static const bool old_attn = getenv("EGT_ATTN16") != nullptr;
  const bool attn_res = attn2_smem(static_cast<int>(M), static_cast<int>(dh), true) <= 200 * 1024;
  const size_t attn2 = attn2_smem(static_cast<int>(M), static_cast<int>(dh), attn_res);
  const bool tile_attn = !no_fused && !old_attn && dh % 4 == 0 && dh / 4 <= 256 / (kAttnRows2 / 4) &&
                         attn2 <= 200 * 1024;
  static const bool no_attn_mma = getenv("EGT_ATTN_NO_MMA") != nullptr;  // tuning: CUDA-core phases
  const bool attn_mma = !no_attn_mma && dh % 32 == 0 && dh <= 128;
  if (tile_attn && attn2 > 48 * 1024) {
    MCUDA(cudaFuncSetAttribute(attention_tile_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(attn2)));
    MCUDA(cudaFuncSetAttribute(attention_tile_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(attn2)));
  }
  const dim3 tb(16, 16);
  for (uint32_t l = 0; l < c.n_layers && st == EGT_OK; ++l) {
    const egt_dev_packed* const* w = m->layers.data() + 6 * l;
    // on the tcgen05 path the rmsnorm of Q/K/V's and ff1's input is folded
    // into the x preparation (one pass for the row's sum of squares and range)
    static const bool no_fold = getenv("EGT_NO_RMSNORM_FOLD") != nullptr;  // tuning
    static const bool no_multi = getenv("EGT_NO_QKV_MULTI") != nullptr;  // tuning: three launches
    const bool fold = !no_fold && !no_multi && M > 1 && egt_impl::umma_eligible(w[0], static_cast<int>(M)) &&
                      egt_impl::umma_eligible(w[4], static_cast<int>(M));
    if (!fold) {
      rmsnorm(x, a);
      ++launch_counter();
    }
    if (M > 1 && !no_multi) {  // one tcgen05 launch over Q, K, V when the tokens take that path
      const egt_dev_packed* qkv[3] = {w[0], w[1], w[2]};
      float* outs[3] = {q, k, v};
      if (st == EGT_OK)
        st = egt_spmm_multi(qkv, 3, fold ? x : a, static_cast<uint32_t>(M), w[0]->cols, outs, w[0]->rows,
                            fold ? EGT_INPUT_RMSNORM : EGT_INPUT_NONE, kNormEps, stream);
    } else {
      lin(w[0], a, q, 0);
      lin(w[1], a, k, EGT_SPMV_INDEPENDENT);  // K and V read `a`, not the previous product
      lin(w[2], a, v, EGT_SPMV_INDEPENDENT);
    }
    if (kv) {  // this pass's keys / values into the pool (the rows later passes attend to)
      const size_t lo = static_cast<size_t>(l) * kv->pool->capacity * d;
      kv_store_kernel<<<M, 256, 0, s>>>(k, v, kv->pool->k + lo, kv->pool->v + lo, d_out_rows, static_cast<int>(M),
                                        static_cast<int>(d));
      ++launch_counter();
    }
    // scores per head: S[h] = (q_h k_h^T) * scale
    if (gather) {
      const size_t lo = static_cast<size_t>(l) * kv->pool->capacity * d;
      kv_attention_kernel<<<dim3(M, H), 128, (c.max_positions + 1) * sizeof(float), s>>>(
          q, k, v, kv->pool->k + lo, kv->pool->v + lo, d_key_ptr, d_key_rows, o, static_cast<int>(d),
          static_cast<int>(dh), att_scale);
      ++launch_counter();
    } else if (tile_attn) {
      if (attn_mma)
        attention_tile_kernel<true><<<dim3((M + kAttnRows2 - 1) / kAttnRows2, H), 256, attn2, s>>>(
            q, k, v, o, dmask, static_cast<int>(M), static_cast<int>(d), static_cast<int>(dh), att_scale, attn_res);
      else
        attention_tile_kernel<false><<<dim3((M + kAttnRows2 - 1) / kAttnRows2, H), 256, attn2, s>>>(
            q, k, v, o, dmask, static_cast<int>(M), static_cast<int>(d), static_cast<int>(dh), att_scale, attn_res);
      ++launch_counter();
    } else if (fused_attn) {
      fused_attention_kernel<<<dim3((M + kAttnRows - 1) / kAttnRows, H), 256, attn_smem, s>>>(
          q, k, v, o, dmask, static_cast<int>(M), static_cast<int>(d), static_cast<int>(dh), att_scale);
      ++launch_counter();
    } else {
    attn_gemm_kernel<true><<<dim3((M + 15) / 16, (M + 15) / 16, H), tb, 0, s>>>(
        q, static_cast<int>(d), dh, k, static_cast<int>(d), dh, S, static_cast<int>(M),
        static_cast<size_t>(M) * M, static_cast<int>(M), static_cast<int>(M), static_cast<int>(dh), att_scale);
    masked_softmax_kernel<<<(M * H + 7) / 8, 256, 0, s>>>(S, dmask, static_cast<int>(M), static_cast<int>(H));
    attn_gemm_kernel<false><<<dim3((dh + 15) / 16, (M + 15) / 16, H), tb, 0, s>>>(
        S, static_cast<int>(M), static_cast<size_t>(M) * M, v, static_cast<int>(d), dh, o, static_cast<int>(d),
        dh, static_cast<int>(M), static_cast<int>(dh), static_cast<int>(M), 1.0f);
    launch_counter() += 3;
    }
    // x += o Wo^T; f = silu(rmsnorm(x) ff1^T); x += f ff2^T -- the residual
    // adds and the silu in the products' epilogues where the path allows
    auto fused = [&](const egt_dev_packed* h, const float* in, float* outp, const float* res, uint32_t flags,
                     uint32_t input = EGT_INPUT_NONE) {
      if (st == EGT_OK)
        st = egt_spmv_fused(h, in, outp, M, h->cols, h->rows, res, res ? static_cast<uint32_t>(d) : 0,
                            input, kNormEps, flags, nullptr, stream);
    };
    const bool glue = w[3]->path == EGT_PATH_TILED && w[4]->path == EGT_PATH_TILED && w[5]->path == EGT_PATH_TILED;
    if (glue) {
      fused(w[3], o, x, x, 0);
      if (fold) {
        fused(w[4], x, f1, nullptr, EGT_SPMV_OUTPUT_SILU, EGT_INPUT_RMSNORM);
      } else {
        rmsnorm(x, a);
        ++launch_counter();
        fused(w[4], a, f1, nullptr, EGT_SPMV_OUTPUT_SILU);
      }
      fused(w[5], f1, x, x, 0);
    } else {
      lin(w[3], o, a, 0);  // a <- o Wo^T
      add_kernel<<<grid_for(Md), 256, 0, s>>>(x, a, Md);
      rmsnorm(x, a);
      launch_counter() += 2;
      lin(w[4], a, f1, 0);
      silu_kernel<<<grid_for(M * dff), 256, 0, s>>>(f1, M * dff);
      ++launch_counter();
      lin(w[5], f1, a, 0);
      add_kernel<<<grid_for(Md), 256, 0, s>>>(x, a, Md);
      ++launch_counter();
    }
  }
  if (st == EGT_OK) {
    rmsnorm(x, a);
    ++launch_counter();
    lin(m->head, a, logits, 0);
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(scratch, s);
  if (st != EGT_OK) return st;
  if (e != cudaSuccess) return fail(EGT_ECUDA, std::string("forward: ") + cudaGetErrorString(e));
  return EGT_OK;
}
}  // namespace

extern "C" {

egt_status egt_model_create(const egt_model_config* cfg, const float* embedding,
                            const egt_dev_packed* const* layers, const egt_dev_packed* head,
                            void* stream, egt_model** out) {
  if (!cfg || !embedding || !layers || !head || !out) return fail(EGT_EINVAL, "model: null argument");
  *out = nullptr;
  const egt_model_config& c = *cfg;  // ModelConfig::validate (model.hpp:41-42)
  if (!c.vocab_size || !c.d_model || !c.n_layers || !c.n_heads || !c.d_ff || !c.max_positions)
    return fail(EGT_EINVAL, "model config: every dimension must be positive");
  if (c.d_model % c.n_heads != 0) return fail(EGT_EINVAL, "model config: d_model must be divisible by n_heads");
  const uint32_t d = c.d_model;
  for (uint32_t l = 0; l < c.n_layers; ++l) {
    const uint32_t shape[6][2] = {{d, d}, {d, d}, {d, d}, {d, d}, {c.d_ff, d}, {d, c.d_ff}};
    for (int j = 0; j < 6; ++j) {
      const egt_dev_packed* h = layers[6 * l + j];
      if (!h || h->rows != shape[j][0] || h->cols != shape[j][1])
        return fail(EGT_EINVAL, "model: layer " + std::to_string(l) + " matrix " + std::to_string(j) +
                                    " has the wrong shape");
    }
  }
  if (head->rows != c.vocab_size || head->cols != d) return fail(EGT_EINVAL, "model: head has the wrong shape");
  auto m = new egt_model();
  m->cfg = c;
  m->layers.assign(layers, layers + 6 * c.n_layers);
  m->head = head;
  cudaGetDevice(&m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // sinusoidal_positions (model.cpp:44-54): double math, stored f32
  std::vector<float> ptab(static_cast<size_t>(c.max_positions) * d);
  for (uint32_t p = 0; p < c.max_positions; ++p)
    for (uint32_t i = 0; i < d; ++i) {
      const double expo = static_cast<double>(2 * (i / 2)) / static_cast<double>(d);
      const double angle = static_cast<double>(p) / std::pow(10000.0, expo);
      ptab[static_cast<size_t>(p) * d + i] = static_cast<float>(i % 2 == 0 ? std::sin(angle) : std::cos(angle));
    }
  const size_t eb = static_cast<size_t>(c.vocab_size) * d * sizeof(float);
  const size_t pb = ptab.size() * sizeof(float);
  if (cudaMalloc(&m->emb, eb) != cudaSuccess || cudaMalloc(&m->pos, pb) != cudaSuccess) {
    cudaFree(m->emb);
    delete m;
    return fail(EGT_ECUDA, "model: device allocation failed");
  }
  cudaMemcpyAsync(m->emb, embedding, eb, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(m->pos, ptab.data(), pb, cudaMemcpyHostToDevice, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    cudaFree(m->emb);
    cudaFree(m->pos);
    delete m;
    return fail(EGT_ECUDA, "model: upload failed");
  }
  *out = m;
  return EGT_OK;
}

egt_status egt_model_query(const egt_model* m, egt_model_config* cfg) {
  if (!m || !cfg) return fail(EGT_EINVAL, "model: null argument");
  *cfg = m->cfg;
  return EGT_OK;
}

egt_status egt_model_destroy(egt_model* m) {
  if (m) {
    cudaFree(m->emb);
    cudaFree(m->pos);
    delete m;
  }
  return EGT_OK;
}


egt_status egt_forward(const egt_model* m, const int32_t* tokens, const int32_t* positions,
                       const uint8_t* mask_bits, uint32_t M, float* logits, void* stream) {
  if (!mask_bits) return fail(EGT_EINVAL, "forward: null argument");
  return forward_core(m, tokens, positions, mask_bits, nullptr, M, logits, stream);
}

egt_status egt_forward_tree(const egt_model* m, const int32_t* tokens, const int32_t* positions,
                            const egt_tree_view* t, float* logits, void* stream) {
  if (!t || (t->n_beams && !t->committed_len) || (t->n_nodes && (!t->parent || !t->beam)))
    return fail(EGT_EINVAL, "forward: null argument");
  const uint64_t M64 = static_cast<uint64_t>(t->n_beams) * t->padded_len + t->n_nodes;
  if (M64 == 0 || M64 > 65536) return fail(EGT_EINVAL, "forward: tree rows must be 1..65536");
  for (uint32_t b = 0; b < t->n_beams; ++b)
    if (t->committed_len[b] > t->padded_len) return fail(EGT_EINVAL, "decode: committed length above the padded length");
  for (uint32_t f = 0; f < t->n_nodes; ++f) {  // build_tree_mask's checks (decode.cpp:278-281)
    if (t->beam[f] >= t->n_beams) return fail(EGT_EINVAL, "decode: flattened node references a missing beam");
    const int32_t p = t->parent[f];
    if (p >= 0 && (static_cast<uint32_t>(p) >= f || t->beam[p] != t->beam[f]))
      return fail(EGT_EINVAL, "decode: flattened parent does not precede its child");
  }
  return forward_core(m, tokens, positions, nullptr, t, static_cast<uint32_t>(M64), logits, stream);
}


// One released pool's buffers are kept for the next create (a decode creates
// and destroys its pool per call; cudaMalloc / cudaFree of the keys and values
// -- tens of MB, cudaFree synchronising the device -- measured several ms per
// 7B beam decode).
namespace {
struct KvCache {
  std::mutex mu;
  float* k = nullptr;
  float* v = nullptr;
  size_t floats = 0;
  int device = -1;
};
KvCache& kv_cache() {
  static KvCache c;
  return c;
}
}  // namespace

egt_status egt_kv_pool_create(const egt_model* m, uint32_t capacity, egt_kv_pool** out) {
  if (!m || !out || capacity == 0) return fail(EGT_EINVAL, "kv pool: null argument or zero capacity");
  *out = nullptr;
  const size_t floats = static_cast<size_t>(m->cfg.n_layers) * capacity * m->cfg.d_model;
  auto p = new egt_kv_pool();
  p->capacity = capacity;
  p->d = m->cfg.d_model;
  p->layers = m->cfg.n_layers;
  p->floats = floats;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    KvCache& c = kv_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    if (c.k && c.device == dev && c.floats >= floats) {
      p->k = c.k;
      p->v = c.v;
      p->floats = c.floats;
      c.k = c.v = nullptr;
      c.floats = 0;
      *out = p;
      return EGT_OK;
    }
  }
  if (cudaMalloc(&p->k, floats * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&p->v, floats * sizeof(float)) != cudaSuccess) {
    cudaFree(p->k);
    delete p;
    return fail(EGT_ECUDA, "kv pool: device allocation failed");
  }
  *out = p;
  return EGT_OK;
}

egt_status egt_kv_pool_destroy(egt_kv_pool* p) {
  if (p) {
    int dev = 0;
    cudaGetDevice(&dev);
    KvCache& c = kv_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    if (p->floats > c.floats || !c.k) {  // keep the larger pair
      if (c.k) {
        cudaFree(c.k);
        cudaFree(c.v);
      }
      c.k = p->k;
      c.v = p->v;
      c.floats = p->floats;
      c.device = dev;
    } else {
      cudaFree(p->k);
      cudaFree(p->v);
    }
    delete p;
  }
  return EGT_OK;
}

egt_status egt_forward_kv(const egt_model* m, egt_kv_pool* pool, const int32_t* tokens, const int32_t* positions,
                          uint32_t M, const uint8_t* mask_bits, const uint32_t* out_rows, const uint32_t* key_ptr,
                          const uint32_t* key_rows, float* logits, void* stream) {
  if (!m || !pool || !out_rows || (!mask_bits && !key_ptr)) return fail(EGT_EINVAL, "forward kv: null argument");
  if (pool->d != m->cfg.d_model || pool->layers != m->cfg.n_layers)
    return fail(EGT_EINVAL, "forward kv: pool built for another model");
  for (uint32_t i = 0; i < M; ++i) {
    if (out_rows[i] >= pool->capacity) return fail(EGT_EINVAL, "forward kv: pool row out of range");
    if (key_ptr) {
      if (key_ptr[i + 1] < key_ptr[i]) return fail(EGT_EINVAL, "forward kv: key lists must be ascending ranges");
      if (key_ptr[i + 1] - key_ptr[i] >= m->cfg.max_positions)
        return fail(EGT_EINVAL, "forward kv: prefix longer than max_positions");
      for (uint32_t j = key_ptr[i]; j < key_ptr[i + 1]; ++j)
        if (key_rows[j] >= pool->capacity) return fail(EGT_EINVAL, "forward kv: pool row out of range");
    }
  }
  KvPass kv{pool, out_rows, key_ptr, key_rows};
  return forward_core(m, tokens, positions, key_ptr ? nullptr : mask_bits, nullptr, M, logits, stream, &kv);
}

egt_status egt_gather(const float* src, uint64_t ld, const uint32_t* rows, const uint32_t* cols,
                      uint32_t n, float* out, void* stream) {
  if (n == 0) return EGT_OK;
  if (!src || !rows || !cols || !out) return fail(EGT_EINVAL, "gather: null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<uint32_t> idx(2 * static_cast<size_t>(n));
  std::memcpy(idx.data(), rows, n * sizeof(uint32_t));
  std::memcpy(idx.data() + n, cols, n * sizeof(uint32_t));
  char* buf = nullptr;
  MCUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), idx.size() * 4 + n * 4, s));
  uint32_t* didx = reinterpret_cast<uint32_t*>(buf);
  float* dout = reinterpret_cast<float*>(didx + idx.size());
  cudaMemcpyAsync(didx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, s);
  gather_kernel<<<(n + 255) / 256, 256, 0, s>>>(src, ld, didx, n, dout);
  ++launch_counter();
  cudaMemcpyAsync(out, dout, n * 4, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(buf, s);
  MCUDA(cudaStreamSynchronize(s));
  return EGT_OK;
}

}  // extern "C"
