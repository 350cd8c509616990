// Internal device-handle representation shared by the C-ABI and the kernels.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <mutex>

#include "tiled_format.h"

namespace egt_impl {
constexpr int kMaxPeers = 8;  // ranks of one NVSwitch node

struct DevStorage {
  int device = 0;
  void* base = nullptr;
  size_t bytes = 0;
  ~DevStorage();
};

// Raw (reference-order) stream, used by the general CUDA-core path and as
// the source of the upload-time re-tiling.
struct RawStream {
  const uint16_t* words = nullptr;       // index words
  const uint8_t* codes = nullptr;        // nibble-packed codes (INT4 sparse)
  const uint8_t* dense_codes = nullptr;  // one code per byte (dense INT4)
  const __half* values = nullptr;        // FP16 values (sparse FP)
  const uint32_t* group_sizes = nullptr;
  const uint32_t* group_offsets = nullptr;
  const float* scales = nullptr;
  const uint8_t* zps = nullptr;
  uint64_t n_scales = 0;
  uint32_t row_begin = 0;  // first row of this handle within the stream
};

// Fragment-tiled stream (tiled_format.h), used by the tensor-core path.
struct TiledStream {
  const uint8_t* vals = nullptr;
  const uint8_t* meta = nullptr;
  const float* scales = nullptr;
  const uint8_t* zps = nullptr;
  int KQ = 0;        // k-quads per row tile (storage)
  int rt_begin = 0;  // first row tile of this handle
  int RT = 0;        // row tiles covered by this handle
  int SS = 4;        // k-tiles per scale entry
  int E = 1;         // scale entries per k-quad (4 / SS)
  int pad14 = 0;     // INT4 1:4 stored as 2:4 (each kept entry paired with a zero-valued one)
};

struct TiledSchedule {
  int RB = 1;  // row tiles per CTA
  int WK = 1;  // warps per row tile (split of the CTA's k-quads)
  int KC = 1;  // k-quads per CTA
  int S = 1;   // K splits (CTAs along K, reduced by the last arriver)
  int NT = 1;  // mma n-tiles (4 tokens each) per CTA
  int NB = 1;  // n-blocks (CTAs along tokens)
  int nw = 8;   // consumer warps per CTA (+1 producer warp)
  int NST = 1;  // shared-memory stages in flight
  int CH = 1;   // k-quads per stage (chunk of a row tile)
  int grid_x = 1, grid_y = 1, grid_z = 1;
  size_t smem = 0;
};

}  // namespace egt_impl

struct egt_dev_packed {
  std::shared_ptr<egt_impl::DevStorage> store;
  uint32_t rows = 0, cols = 0;
  uint8_t n = 2, m = 4, kind = 1, format = 0, path = 0;
  // general path, INT4 2:4 with every row's group size a power of two >= 16
  // (or one group per row) and cols % 16 == 0: the grouped-stream kernel
  uint8_t grouped_ok = 0;
  egt_impl::RawStream raw;
  egt_impl::TiledStream tiled;
  uint64_t nnz = 0;
  uint64_t algorithmic_bytes = 0;
  uint64_t device_bytes = 0;
  // Launch plans keyed by M (logically const: a plan depends only on shape).
  mutable std::mutex plan_mu;
  mutable std::map<int, egt_impl::TiledSchedule> plans;
  mutable std::shared_ptr<void> umma_maps;  // TMA tensor maps of the tcgen05 path (umma_spmm.cu)
};

// Row-shard peer group (fused all-gather): every rank's buffer in rank order;
// each is [512-byte control block | y].  Control block: u32 arrival counters
// [0, 8), then at byte 256 this rank's [sequence, done, error].
struct egt_peer_group {
  uint32_t world = 0, rank = 0;
  uint32_t* flags[egt_impl::kMaxPeers] = {};
  float* y[egt_impl::kMaxPeers] = {};
  uint32_t* ctrl = nullptr;
};

namespace egt_impl {
// GPU compression (compress.cu): importance_scores, prune_nm, the exact-N
// check, and quantize + pack into the reference's stream layout.
cudaError_t launch_importance(const float* w, const float* xn, const float* g, uint32_t rows, uint32_t cols,
                              float* out, cudaStream_t s);
cudaError_t launch_prune_nm(const float* scores, uint32_t rows, uint32_t cols, int n, uint8_t* mask,
                            cudaStream_t s);
cudaError_t launch_check_nm(const uint8_t* mask, uint32_t rows, uint32_t cols, int n,
                            unsigned long long* first_bad, cudaStream_t s);
cudaError_t launch_quantize_pack(const float* w, const uint8_t* mask, uint32_t rows, uint32_t cols, int n,
                                 const uint32_t* gs, const uint32_t* goff, float* scales, uint8_t* zps,
                                 uint8_t* codes_tmp, uint8_t* value_bytes, uint16_t* words, cudaStream_t s);
// Dense f32 GEMV (the dense-FP baseline arm, bench_spmv's dense-fp).
cudaError_t launch_gemv_f32(const float* w, const float* x, float* y, uint32_t rows, uint32_t cols, cudaStream_t s);
// Signal this rank's (empty) slice and optionally wait for every peer's.
cudaError_t launch_peer_signal(const egt_peer_group* g, bool signal, bool wait, cudaStream_t s);
}  // namespace egt_impl

namespace egt_impl {

// Per-call launch context.
struct LaunchCtx {
  cudaStream_t stream = nullptr;
  bool pdl = true;
  float* partial = nullptr;      // split-K partial sums
  uint32_t* counters = nullptr;  // split-K arrival counters (self-resetting)
  int xform = 0;                 // EGT_INPUT_* applied to x while staging
  int out_silu = 0;              // EGT_SPMV_OUTPUT_SILU: y = silu(...)
  float eps = 1e-6f;
  const float* res = nullptr;    // y = res + product (may alias y)
  int ldr = 0;
  const egt_dev_packed* l2_next = nullptr;  // weights to prefetch into L2 meanwhile
  int nseg = 0;                             // > 1: one launch over several same-shape matrices
  const egt_dev_packed* segs[3] = {nullptr, nullptr, nullptr};
  float* seg_y[3] = {nullptr, nullptr, nullptr};
  int npeer = 0;                  // > 0: row shard, y rows stored into every peer (fused all-gather)
  int peer_rank = 0, peer_row0 = 0, peer_wait = 1;
  float* peer_y[kMaxPeers] = {};
  uint32_t* peer_flag[kMaxPeers] = {};
  uint32_t* peer_ctrl = nullptr;
};

TiledSchedule plan_tiled(const egt_dev_packed* h, int M, int num_sms, bool indep);
TiledSchedule plan_tiled_rt(const egt_dev_packed* h, int RT, int M, int num_sms, bool indep);
void force_plan(int RB, int S, int nw, int NST, int CH);  // tuning hook (0 = automatic)
bool plan_forced();
size_t tiled_workspace_floats(const egt_dev_packed* h, const TiledSchedule& sc, int M);

cudaError_t launch_tiled(const egt_dev_packed* h, const TiledSchedule& sc, const float* x, int ldx,
                         int M, float* y, int ldy, const LaunchCtx& ctx, bool indep);
// Many-token products (M > 16): x fragments in global memory (xf_ws of
// wide_workspace_bytes), weight-streaming CTAs per 16-token block (spmm_wide.cu).
// Many-token products on tcgen05 / TMEM (umma_spmm.cu): INT4 2:4 (and 1:4
// stored as 2:4), dense INT4 and FP16 2:4 layers with 64/128-column scale
// groups; ws = umma_workspace_bytes (x stages + per-token range), split-K
// partials / counters in ctx.
bool umma_eligible(const egt_dev_packed* h, int M);
unsigned long long* umma_trace_buffer();  // EGT_UMMA_TRACE (tuning)
size_t umma_workspace_bytes(const egt_dev_packed* h, int M);
size_t umma_partial_floats(const egt_dev_packed* h, int M, int num_sms);
size_t umma_counters(const egt_dev_packed* h, int M, int num_sms);
cudaError_t launch_umma(const egt_dev_packed* h, const float* x, int ldx, int M, float* y, int ldy,
                        uint8_t* ws, const LaunchCtx& ctx, int num_sms);
// nseg (<= 3) same-shape matrices over the same x in one launch (no residual)
cudaError_t launch_umma_multi(const egt_dev_packed* const* hs, int nseg, const float* x, int ldx, int M,
                              float* const* ys, int ldy, uint8_t* ws, const LaunchCtx& ctx, int num_sms);
size_t wide_workspace_bytes(const egt_dev_packed* h, int M);
cudaError_t launch_wide(const egt_dev_packed* h, const float* x, int ldx, int M, float* y, int ldy,
                        uint32_t* xf_ws, const LaunchCtx& ctx, int num_sms);
// Reference-order INT4 2:4 stream with power-of-two groups >= 16 (the
// reference's default g_fine = 16), M <= 4, fused input / epilogue
// (stream_kernels.cu); false when the shape is not covered.
bool grouped_stream_ok(const egt_dev_packed* h, int M);
cudaError_t launch_grouped_stream(const egt_dev_packed* h, const float* x, int ldx, int M, float* y, int ldy,
                                  const LaunchCtx& ctx);
cudaError_t launch_general(const egt_dev_packed* h, const float* x, int ldx, int M, float* y,
                           int ldy, const LaunchCtx& ctx);

// Upload-time kernels; the raw arrays live on the device.
cudaError_t launch_validate_offsets(const uint16_t* words, uint32_t rows, uint32_t cols, int n,
                                    uint32_t* err_flag, cudaStream_t s);
cudaError_t launch_validate_groups(const uint32_t* gsizes, const uint32_t* goffs, uint32_t rows,
                                   uint32_t cols, uint64_t n_scales, uint32_t* err_flag,
                                   cudaStream_t s);
cudaError_t launch_f32_to_f16(const float* src, __half* dst, uint64_t n, bool check, uint32_t* err, cudaStream_t s);
cudaError_t launch_relayout(const RawStream& raw, int format, uint32_t rows, uint32_t cols,
                            const TiledStream& dst_shape, uint8_t* vals, uint8_t* meta,
                            float* scales, uint8_t* zps, cudaStream_t s);  // dst_shape.pad14: raw is 1:4
cudaError_t launch_dequant(const egt_dev_packed* h, float* w, uint8_t* mask, cudaStream_t s);

uint64_t& launch_counter();
unsigned long long* tiled_trace_buffer();  // EGT_TILED_TRACE tuning stamps (or null)

}  // namespace egt_impl
