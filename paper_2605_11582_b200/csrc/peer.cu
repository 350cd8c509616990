// Peer buffers and groups for the row-sharded SparseGemv with a fused
// all-gather.  The reference has no multi-GPU path (spmv,
// packed.cpp:211-220, runs the whole matrix in one process); this replaces
// "local spmv + ncclAllGather of the y slices" with one kernel whose
// epilogue stores every y row into every rank's buffer over NVLink (CUDA IPC
// mappings of the peers' buffers) and whose last CTA exchanges arrival
// counters (spmm_tiled.cu, peer_complete).
#include "device_common.cuh"
#include "egt_b200.h"
#include "handle.h"

#include <cstdlib>
#include <cstring>
#include <string>

namespace egt_impl {
void set_last_error(const std::string& m);
}

namespace {
using namespace egt_impl;

egt_status pfail(egt_status s, const std::string& m) {
  set_last_error(m);
  return s;
}

#define PCUDA(expr)                                                                 \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) return pfail(EGT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct PeerSignal {
  uint32_t* flags[kMaxPeers];
  uint32_t* own_flags;
  uint32_t* ctrl;
  int n, rank, signal, wait;
};

__global__ void peer_signal_kernel(const PeerSignal p) {
  if (threadIdx.x != 0) return;
  // after the shard product on this stream (a plain stream-ordered launch)
  if (p.signal) {
    __threadfence_system();
    for (int g = 0; g < p.n; ++g) atomicAdd_system(p.flags[g] + p.rank, 1u);
  }
  if (p.wait) egt_dev::peer_wait_all(p.own_flags, p.n, p.ctrl);
}

}  // namespace

namespace egt_impl {
cudaError_t launch_peer_signal(const egt_peer_group* g, bool signal, bool wait, cudaStream_t s) {
  static const bool force = getenv("EGT_DEBUG_MODE") && atoi(getenv("EGT_DEBUG_MODE")) == 14;
  if (g->world == 1 && !force) return cudaSuccess;  // one rank: nothing to exchange (as in the kernel)
  PeerSignal p{};
  for (uint32_t i = 0; i < g->world; ++i) p.flags[i] = g->flags[i];
  p.own_flags = g->flags[g->rank];
  p.ctrl = g->ctrl;
  p.n = static_cast<int>(g->world);
  p.rank = static_cast<int>(g->rank);
  p.signal = signal ? 1 : 0;
  p.wait = wait ? 1 : 0;
  peer_signal_kernel<<<1, 32, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++launch_counter();
  return e;
}
}  // namespace egt_impl

extern "C" {

egt_status egt_peer_buffer_alloc(size_t y_floats, void** buf, egt_ipc_handle* handle) {
  if (!buf) return pfail(EGT_EINVAL, "peer buffer: null output");
  void* p = nullptr;
  const size_t bytes = EGT_PEER_CTRL_BYTES + y_floats * sizeof(float);
  PCUDA(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && handle) {
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, p);
    if (e == cudaSuccess) {
      static_assert(sizeof(h) == sizeof(handle->bytes), "CUDA IPC handle is 64 bytes");
      std::memcpy(handle->bytes, &h, sizeof(h));
    }
  }
  if (e != cudaSuccess) {
    cudaFree(p);
    return pfail(EGT_ECUDA, std::string("peer buffer: ") + cudaGetErrorString(e));
  }
  *buf = p;
  return EGT_OK;
}

egt_status egt_peer_buffer_free(void* buf) {
  if (buf) PCUDA(cudaFree(buf));
  return EGT_OK;
}

egt_status egt_peer_buffer_open(const egt_ipc_handle* handle, void** buf) {
  if (!handle || !buf) return pfail(EGT_EINVAL, "peer buffer: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle->bytes, sizeof(h));
  PCUDA(cudaIpcOpenMemHandle(buf, h, cudaIpcMemLazyEnablePeerAccess));
  return EGT_OK;
}

egt_status egt_peer_buffer_close(void* buf) {
  if (buf) PCUDA(cudaIpcCloseMemHandle(buf));
  return EGT_OK;
}

egt_status egt_peer_group_create(uint32_t world, uint32_t rank, void* const* bufs, egt_peer_group** out) {
  if (!out || !bufs) return pfail(EGT_EINVAL, "peer group: null argument");
  if (world == 0 || world > EGT_MAX_PEERS || rank >= world)
    return pfail(EGT_EINVAL, "peer group: world must be 1..8 and rank below it");
  for (uint32_t i = 0; i < world; ++i)
    if (!bufs[i]) return pfail(EGT_EINVAL, "peer group: null buffer");
  auto* g = new egt_peer_group;
  g->world = world;
  g->rank = rank;
  for (uint32_t i = 0; i < world; ++i) {
    g->flags[i] = static_cast<uint32_t*>(bufs[i]);
    g->y[i] = reinterpret_cast<float*>(static_cast<uint8_t*>(bufs[i]) + EGT_PEER_CTRL_BYTES);
  }
  g->ctrl = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(bufs[rank]) + 256);
  *out = g;
  return EGT_OK;
}

egt_status egt_peer_group_destroy(egt_peer_group* g) {
  delete g;
  return EGT_OK;
}

float* egt_peer_group_y(const egt_peer_group* g) { return g ? g->y[g->rank] : nullptr; }

egt_status egt_peer_wait(egt_peer_group* g, void* stream) {
  if (!g) return pfail(EGT_EINVAL, "peer wait: null group");
  PCUDA(launch_peer_signal(g, false, true, static_cast<cudaStream_t>(stream)));
  return EGT_OK;
}

egt_status egt_peer_group_check(egt_peer_group* g) {
  if (!g) return pfail(EGT_EINVAL, "peer group: null group");
  PCUDA(cudaDeviceSynchronize());
  uint32_t err = 0;
  PCUDA(cudaMemcpy(&err, g->ctrl + 2, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) return pfail(EGT_EINTERNAL, "peer wait timed out: a rank's slice never arrived");
  return EGT_OK;
}

}  // extern "C"
