// Device helpers shared by the SparseGemv kernels (sm_100a only).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "egt_b200 is built for sm_100a only"
#endif

namespace egt_dev {

constexpr int kWarp = 32;

// Streamed, read-once weight loads: no L1 allocation, and an L2 evict-first
// policy so the packed stream does not push x / partial sums out of L2.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg_stream_v4(const void* ptr, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ uint2 ldg_stream_v2(const void* ptr, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;\n"
               : "=r"(r.x), "=r"(r.y)
               : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t ldg_stream_u32(const void* ptr, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;\n"
               : "=r"(r)
               : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t ldg_stream_u16(const void* ptr, uint64_t pol) {
  uint16_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;\n"
               : "=h"(r)
               : "l"(ptr), "l"(pol));
  return r;
}

// Programmatic dependent launch: weights do not depend on the previous
// kernel, x does.  Everything before pdl_wait() may overlap the producer.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// INT4 nibble pair -> half2 {1024 + lo, 1024 + hi}: the nibbles at bits
// [0,4) and [16,20) of v land in the fp16 mantissas under exponent 0x64.
__device__ __forceinline__ uint32_t nib2_magic(uint32_t v) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(v), "r"(0x000F000Fu), "r"(0x64006400u));
  return r;  // (v & mask) | magic
}

// INT4 nibble pair at bits [4,8) and [20,24) -> half2 {1024 + 16 lo, 1024 + 16 hi}.
__device__ __forceinline__ uint32_t nib16_magic(uint32_t v) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(v), "r"(0x00F000F0u), "r"(0x64006400u));
  return r;
}

__device__ __forceinline__ uint32_t hsub2_u32(uint32_t a, uint32_t b) {
  __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

// half2 {1024 + z0, 1024 + z1} for two zero points.
__device__ __forceinline__ uint32_t zp_magic(uint32_t z0, uint32_t z1) {
  return (0x6400u | z0) | ((0x6400u | z1) << 16);
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// D[16x8] (+)= A[16x32, 2:4 sparse] * B[32x8], f16 inputs, f32 accumulate.
// Metadata register e is read from lanes {0,1} (sel 0) or {2,3} (sel 1) of
// each quad (measured on B200, tests/test_gpu_spmv.py::test_effective_matrix_probe):
// lane 2*sel + hh covers groups [4hh, 4hh+4) (columns 16hh..16hh+15), row g in
// bits [0,16) and row g+8 in bits [16,32); nibble q4 = group 4hh+q4, with
// bits[1:0] the first kept index and [3:2] the second.
template <int kSel>
__device__ __forceinline__ void mma_sp_16832(float (&d)[4], const uint32_t (&a)[4],
                                             const uint32_t (&b)[4], uint32_t e) {
  asm volatile(
      "mma.sp::ordered_metadata.sync.aligned.m16n8k32.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9,%10,%11}, {%0,%1,%2,%3}, %12, %13;\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]),
        "r"(e), "n"(kSel));
}

// Dense D[16x8] (+)= A[16x16] * B[16x8], f16 inputs, f32 accumulate.
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace egt_dev

namespace egt_dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mbarrier + bulk-copy (TMA engine, non-tensor) primitives.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Polling wait (mbarrier.test_wait never suspends the thread): for waits
// that are usually short, where try_wait's suspend/wake-up latency would sit
// on the critical path.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0,
// both addresses 16-byte aligned), L2 evict-first.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// global -> shared bulk copy without a cache-policy operand.
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Fused all-gather wait (one thread): ctrl[0] counts this rank's completed
// gathers; every rank's arrival counter flags[g] must reach ctrl[0] + 1.
// Relaxed system-scope polling (peers add over NVLink), one acq_rel fence
// once all have arrived; bounded by 2 s of globaltimer, after which ctrl[2]
// records the timeout instead of hanging.
__device__ __forceinline__ void peer_wait_all(const uint32_t* flags, int n, uint32_t* ctrl) {
  const uint32_t target = ctrl[0] + 1u;
  unsigned long long t0 = 0;
  for (int g = 0; g < n; ++g) {
    while (true) {
      uint32_t v;
      asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + g) : "memory");
      if (static_cast<int32_t>(v - target) >= 0) break;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      if (t - t0 > 2000000000ull) {
        ctrl[2] = 1u;
        g = n;
        break;
      }
      __nanosleep(32);
    }
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  ctrl[0] = target;
}

}  // namespace egt_dev
