// Microbenchmark: cycles per tcgen05.mma (kind::f16, M = 128, cta_group::1)
// issued back to back by one thread on fixed shared-memory operands, for
// dense / 2:4-sparse and several N.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o /tmp/umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t row_bytes) {
  const uint64_t layout = row_bytes == 128 ? 2ull : 4ull;
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(((8 * row_bytes) >> 4) & 0x3FFFu) << 32) |
         (1ull << 46) | (layout << 61);
}
__global__ void k(int N, int sparse, int iters, long long* out, int nacc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(sa(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {  // metadata: (0,1) everywhere
    // (TMEM lane access: warp 1 -> lanes 32..63; metadata only needs to be valid-ish)
  }
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24) | (sparse ? (1u << 2) : 0u);
    const uint32_t a = sa(base), b = sa(base + 32768);
    const uint64_t ad = desc_sw(a, sparse ? 64 : 128), bd = desc_sw(b, 128);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)((i % nacc) * (N < 128 ? 64 : 0));
      if (sparse)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n"
                     "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, p;\n}\n" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(tmem + 256), "r"(idesc), "r"(1));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(1));
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(sa(&bar)));
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sa(&bar)));
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// TMEM -> register throughput: nw warps each load `cols` columns (x8 loads,
// all in flight, one wait) `iters` times.
__global__ void ld(int cols, int iters, long long* out) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(sa(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = slot + ((uint32_t)(32 * ((threadIdx.x >> 5) & 3)) << 16);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < cols; c += 32) {
      uint32_t r[32];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(r[8*q]), "=r"(r[8*q+1]), "=r"(r[8*q+2]), "=r"(r[8*q+3]), "=r"(r[8*q+4]), "=r"(r[8*q+5]),
                       "=r"(r[8*q+6]), "=r"(r[8*q+7])
                     : "r"(tmem + (uint32_t)(c + 8 * q)));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int q = 0; q < 32; ++q) acc += __uint_as_float(r[q]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.f) out[1] = 1;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(slot));
}
int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int nacc : {1, 4})
  for (int sparse = 0; sparse < 2; ++sparse)
    for (int N : {16, 48, 64, 128, 256}) {
      const int iters = 256;
      if (nacc > 1 && N >= 128) continue;
      k<<<1, 128, 80 * 1024>>>(N, sparse, iters, d, nacc);
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      cudaError_t e = cudaGetLastError();
      printf("acc x%d %s N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", nacc, sparse ? "sparse" : "dense ", N,
             (double)h[0] / iters, (double)h[1] / iters, cudaGetErrorString(e));
    }
  for (int nw : {4, 8, 16})
    for (int cols : {64, 256}) {
      ld<<<1, 32 * nw>>>(cols, 64, d);
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      const double bytes = 64.0 * cols * 4 * 32 * nw;  // iters x cols x 4 B x threads
      printf("tcgen05.ld: %2d warps x %3d cols: %.1f B/cycle (%s)\n", nw, cols, bytes / h[0],
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
