// KV-cached batch-1 decode loop on the device: the
// reference recomputes the whole prefix every step (decode.cpp:122-190 calls
// forward over the block-diagonal causal prefix); here each step runs the
// token at position t through the stack against a KV cache, which is the
// same arithmetic (the query at t attends to keys 0..t, model.cpp:161-184)
// with every linear layer an M = 1 SparseGemv.
//
// One step, for the token at position t (both live in device memory, so the
// step is position-independent and captured ONCE as a CUDA graph):
//   h = emb[token] + pos[t]                                (model.cpp:141-143)
//   per layer: q,k,v = W rmsnorm(h)      (egt_spmv_fused, rmsnorm staged in)
//              k,v -> cache[t]; o = softmax(q K^T * scale) V   (per head)
//              h = h + Wo o              (residual epilogue)
//              f = Wff1 rmsnorm(h); h = h + Wff2 silu(f)
//   logits = head rmsnorm(h)                               (model.cpp:194-195)
//   next = prompt[t+1] while inside the prompt, else argmax(logits)
//          (greedy, ties -> lowest id); t += 1
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "device_common.cuh"
#include "egt_b200.h"
#include "handle.h"
#include "model.h"

namespace egt_impl {
void set_last_error(const std::string& msg);
}

struct egt_decoder {
  const egt_model* m = nullptr;
  uint32_t max_len = 0;
  cudaStream_t s = nullptr;
  char* mem = nullptr;
  float *kc = nullptr, *vc = nullptr;  // [L][max_len][d]
  float *h = nullptr, *q = nullptr, *k = nullptr, *v = nullptr, *o = nullptr, *f = nullptr, *logits = nullptr;
  int32_t* state = nullptr;   // [0] t, [1] token at t, [2] prompt length
  int32_t* prompt = nullptr;  // [max_len]
  int32_t* out = nullptr;     // [max_len] token at each position
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  uint32_t host_t = 0;  // positions run so far (host mirror of state[0])
};

namespace {

using egt_impl::launch_counter;
constexpr float kNormEps = 1e-6f;  // model.cpp:27

egt_status dfail(egt_status s, const std::string& m) {
  egt_impl::set_last_error(m);
  return s;
}

__global__ void dec_embed_kernel(const int32_t* state, const float* emb, const float* ptab, float* h, int d,
                                 int32_t* out, int max_len) {
  egt_dev::pdl_launch_dependents();  // the first Q product may prefetch its weights
  const int t = state[0], tok = state[1];
  if (t >= max_len) return;  // replay past the cache: no-op (the host also refuses)
  if (threadIdx.x == 0 && blockIdx.x == 0) out[t] = tok;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d; c += gridDim.x * blockDim.x)
    h[c] = emb[static_cast<size_t>(tok) * d + c] + ptab[static_cast<size_t>(t) * d + c];
}

// One block per head: append k,v at row t, scores over keys 0..t (warp per
// key, coalesced 4 floats per lane), softmax (max-subtracted, model.cpp:
// 169-182), o = p V (thread per head dimension, two key halves).
constexpr int kKvPre = 64;  // cached keys / values staged into shared memory before the PDL wait

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

template <int DH>
__global__ void __launch_bounds__(256) dec_attention_kernel(const int32_t* state, const float* q, const float* k,
                                                            const float* v, float* kc, float* vc, float* o, int d,
                                                            float scale, int sc_cap, int max_len) {
  extern __shared__ __align__(16) float smx[];
  float* sc = smx;                      // [t + 1] scores (sc_cap floats)
  float* kp = smx + sc_cap;             // [kKvPre][DH] cached keys
  float* vp = kp + kKvPre * DH;         // [kKvPre][DH] cached values
  __shared__ float red[8];
  __shared__ __align__(16) float qs[DH];
  __shared__ float part[8][DH];
  // launched with programmatic serialization: let the O product start
  // streaming its weights now.  Cache rows [0, t) were written by earlier
  // steps (complete: every kernel before this one's predecessor has
  // finished), so they are staged while the Q/K/V product still runs; q, k,
  // v (row t) only after the wait.
  egt_dev::pdl_launch_dependents();
  const int t = state[0], n = t + 1;
  if (t >= max_len) return;  // past the cache rows / score buffer: no-op
  const int hh = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t base = static_cast<size_t>(hh) * DH;
  const int npre = min(t, kKvPre);
  for (int idx = tid; idx < npre * (DH / 4); idx += blockDim.x) {
    const int i = idx / (DH / 4), e4 = (idx % (DH / 4)) * 4;
    cp_async16(kp + i * DH + e4, kc + static_cast<size_t>(i) * d + base + e4);
    cp_async16(vp + i * DH + e4, vc + static_cast<size_t>(i) * d + base + e4);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  egt_dev::pdl_wait();
  for (int i = tid; i < DH; i += blockDim.x) {
    kc[static_cast<size_t>(t) * d + base + i] = k[base + i];
    vc[static_cast<size_t>(t) * d + base + i] = v[base + i];
    qs[i] = q[base + i];
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  // scores: a thread per key, the key's head slice as float4 loads (all of a
  // thread's loads in flight together); row t was just written by this block
  static_assert(DH % 4 == 0, "head dimension multiple of 4");
  for (int i = tid; i < n; i += blockDim.x) {
    const float4* kr = reinterpret_cast<const float4*>(i < npre ? kp + i * DH : kc + static_cast<size_t>(i) * d + base);
    float dot = 0.f;
#pragma unroll
    for (int e = 0; e < DH / 4; ++e) {
      const float4 kv = kr[e];
      const float4 qv = reinterpret_cast<const float4*>(qs)[e];
      dot = fmaf(qv.x, kv.x, fmaf(qv.y, kv.y, fmaf(qv.z, kv.z, fmaf(qv.w, kv.w, dot))));
    }
    sc[i] = dot * scale;
  }
  __syncthreads();
  float mx = -INFINITY;
  for (int i = tid; i < n; i += blockDim.x) mx = fmaxf(mx, sc[i]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float z = 0.f;
  for (int i = tid; i < n; i += blockDim.x) {
    const float e = expf(sc[i] - mx);
    sc[i] = e;
    z += e;
  }
  z = egt_dev::warp_sum(z);
  if (lane == 0) red[warp] = z;
  __syncthreads();
  z = 0.f;
  for (int w = 0; w < 8; ++w) z += red[w];
  // o = sum_i p_i v_i: warp w takes keys w, w + 8, ..., lane l dims
  // [l*PER, (l+1)*PER); four keys in flight; then the 8 warp partials
  constexpr int PER = DH >= 32 ? DH / 32 : 1;
  const bool on = lane * PER < DH;
  float acc[PER];
#pragma unroll
  for (int e = 0; e < PER; ++e) acc[e] = 0.f;
  if (on) {
    int i = warp;
    for (; i + 24 < n; i += 32) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float p_ = sc[i + 8 * r];
        const int ii = i + 8 * r;
        const float* vr = (ii < npre ? vp + ii * DH : vc + static_cast<size_t>(ii) * d + base) + lane * PER;
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[e] = fmaf(p_, vr[e], acc[e]);
      }
    }
    for (; i < n; i += 8) {
      const float p_ = sc[i];
      const float* vr = (i < npre ? vp + i * DH : vc + static_cast<size_t>(i) * d + base) + lane * PER;
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[e] = fmaf(p_, vr[e], acc[e]);
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) part[warp][lane * PER + e] = acc[e];
  }
  __syncthreads();
  for (int dim = tid; dim < DH; dim += blockDim.x) {
    float sum = 0.f;
    for (int w = 0; w < 8; ++w) sum += part[w][dim];
    o[base + dim] = sum / z;
  }
}

// next token: the prompt's while t + 1 is inside it, else argmax (ties ->
// lowest id); advances t.
__global__ void __launch_bounds__(1024) dec_next_kernel(int32_t* state, const int32_t* prompt, const float* logits,
                                                        int vocab, int max_len) {
  __shared__ float bv[32];
  __shared__ int bi[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int i = tid; i < vocab; i += blockDim.x) {
    const float v = logits[i];
    if (v > best) {  // strided scan: the first (lowest) index wins ties
      best = v;
      idx = i;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, off);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
    if (ov > best || (ov == best && oi < idx)) {
      best = ov;
      idx = oi;
    }
  }
  if (lane == 0) {
    bv[warp] = best;
    bi[warp] = idx;
  }
  __syncthreads();
  if (tid == 0) {
    best = bv[0];
    idx = bi[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (bv[w] > best || (bv[w] == best && bi[w] < idx)) {
        best = bv[w];
        idx = bi[w];
      }
    const int t = state[0];
    if (t < max_len) {  // never advance past the cache
      state[1] = t + 1 < state[2] ? prompt[t + 1] : idx;
      state[0] = t + 1;
    }
  }
}

#define DCUDA(expr)                                                                    \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) return dfail(EGT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// The launches of one step on d->s (captured into the graph).
egt_status enqueue_step(egt_decoder* dd) {
  const egt_model* m = dd->m;
  const egt_model_config& c = m->cfg;
  const uint32_t d = c.d_model, H = c.n_heads, dh = d / H;
  cudaStream_t s = dd->s;
  dec_embed_kernel<<<(d + 255) / 256, 256, 0, s>>>(dd->state, m->emb, m->pos, dd->h, static_cast<int>(d), dd->out,
                                                    static_cast<int>(dd->max_len));
  ++launch_counter();
  const float scale = 1.0f / std::sqrt(static_cast<float>(dh));  // model.cpp:139
  egt_status st = EGT_OK;
  // optional (EGT_DECODE_L2PF=1): each product prefetches the next product's
  // weights into L2 (measured slower on B200: 538 vs 576 tok/s, so off)
  const bool l2pf = getenv("EGT_DECODE_L2PF") != nullptr;
  auto lin = [&](const egt_dev_packed* w, const float* x, float* y, const float* res, uint32_t input,
                 uint32_t flags, const egt_dev_packed* next) {
    if (st == EGT_OK)
      st = egt_spmv_fused(w, x, y, 1, w->cols, w->rows, res, w->rows, input, kNormEps, flags, l2pf ? next : nullptr, s);
  };
  const int sc_cap = static_cast<int>((dd->max_len + 3) / 4 * 4);
  const size_t attn_smem = (static_cast<size_t>(sc_cap) + 2ull * kKvPre * dh) * sizeof(float);
  for (uint32_t l = 0; l < c.n_layers && st == EGT_OK; ++l) {
    const egt_dev_packed* const* w = m->layers.data() + 6 * l;
    const bool qkv_fused = getenv("EGT_DECODE_NO_QKV") == nullptr && w[0]->format == w[1]->format &&
                           w[1]->format == w[2]->format && w[0]->tiled.SS == w[1]->tiled.SS &&
                           w[1]->tiled.SS == w[2]->tiled.SS && w[0]->rows % 16 == 0;
    const egt_dev_packed* next_q = l + 1 < c.n_layers ? m->layers[6 * (l + 1)] : m->head;
    if (qkv_fused) {  // Q, K, V in one launch: one staging of rmsnorm(h), one wait
      float* ys[3] = {dd->q, dd->k, dd->v};
      if (st == EGT_OK) st = egt_spmv_fused_multi(w, 3, dd->h, ys, EGT_INPUT_RMSNORM, kNormEps, 0, s);
    } else {
      lin(w[0], dd->h, dd->q, nullptr, EGT_INPUT_RMSNORM, 0, w[1]);
      lin(w[1], dd->h, dd->k, nullptr, EGT_INPUT_RMSNORM, EGT_SPMV_INDEPENDENT, w[2]);
      lin(w[2], dd->h, dd->v, nullptr, EGT_INPUT_RMSNORM, EGT_SPMV_INDEPENDENT, w[3]);
    }
    float* kc = dd->kc + static_cast<size_t>(l) * dd->max_len * d;
    float* vc = dd->vc + static_cast<size_t>(l) * dd->max_len * d;
    {
      void* fn = dh == 16 ? reinterpret_cast<void*>(&dec_attention_kernel<16>)
               : dh == 32 ? reinterpret_cast<void*>(&dec_attention_kernel<32>)
               : dh == 64 ? reinterpret_cast<void*>(&dec_attention_kernel<64>)
                          : reinterpret_cast<void*>(&dec_attention_kernel<128>);
      if (attn_smem > 48 * 1024) DCUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                          static_cast<int>(attn_smem)));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(H);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = attn_smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      const int32_t* st_ = dd->state;
      const float *q_ = dd->q, *k_ = dd->k, *v_ = dd->v;
      float* o_ = dd->o;
      int d_ = static_cast<int>(d);
      float sc_ = scale;
      int cap_ = sc_cap;
      int ml_ = static_cast<int>(dd->max_len);
      void* args[] = {&st_, &q_, &k_, &v_, &kc, &vc, &o_, &d_, &sc_, &cap_, &ml_};
      DCUDA(cudaLaunchKernelExC(&cfg, fn, args));
    }
    ++launch_counter();
    lin(w[3], dd->o, dd->h, dd->h, EGT_INPUT_NONE, 0, w[4]);
    lin(w[4], dd->h, dd->f, nullptr, EGT_INPUT_RMSNORM, EGT_SPMV_OUTPUT_SILU, w[5]);  // f = silu(ff1 b)
    lin(w[5], dd->f, dd->h, dd->h, EGT_INPUT_NONE, 0, next_q);
  }
  lin(m->head, dd->h, dd->logits, nullptr, EGT_INPUT_RMSNORM, 0, m->layers[0]);
  if (st != EGT_OK) return st;
  dec_next_kernel<<<1, 1024, 0, s>>>(dd->state, dd->prompt, dd->logits, static_cast<int>(c.vocab_size),
                                     static_cast<int>(dd->max_len));
  ++launch_counter();
  DCUDA(cudaGetLastError());
  return EGT_OK;
}

}  // namespace

extern "C" {

egt_status egt_decoder_create(const egt_model* m, uint32_t max_len, egt_decoder** out) {
  if (!m || !out || max_len == 0) return dfail(EGT_EINVAL, "decoder: null argument");
  *out = nullptr;
  const egt_model_config& c = m->cfg;
  if (max_len > c.max_positions) return dfail(EGT_EINVAL, "decoder: max_len exceeds max_positions");
  if (max_len > 8192) return dfail(EGT_EINVAL, "decoder: max_len above 8192");
  const uint32_t d = c.d_model, dh = d / c.n_heads;
  if (dh != 16 && dh != 32 && dh != 64 && dh != 128)
    return dfail(EGT_EINVAL, "decoder: head dimension must be 16, 32, 64 or 128");
  for (const egt_dev_packed* w : m->layers)
    if (w->path != EGT_PATH_TILED) return dfail(EGT_EINVAL, "decoder: every layer must be on the tiled path");
  if (m->head->path != EGT_PATH_TILED) return dfail(EGT_EINVAL, "decoder: head must be on the tiled path");
  auto dd = new egt_decoder();
  dd->m = m;
  dd->max_len = max_len;
  const size_t cache = static_cast<size_t>(c.n_layers) * max_len * d;
  const size_t floats = 2 * cache + 5 * static_cast<size_t>(d) + c.d_ff + c.vocab_size;
  const size_t bytes = floats * 4 + (3 + 2 * static_cast<size_t>(max_len)) * 4 + 256;
  cudaError_t e = cudaStreamCreateWithFlags(&dd->s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&dd->mem, bytes);
  if (e == cudaSuccess) e = cudaMemsetAsync(dd->mem, 0, bytes, dd->s);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&dd->ev_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&dd->ev_out, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    egt_decoder_destroy(dd);
    return dfail(EGT_ECUDA, std::string("decoder: allocation failed: ") + cudaGetErrorString(e));
  }
  float* p = reinterpret_cast<float*>(dd->mem);
  dd->kc = p;
  dd->vc = p + cache;
  p += 2 * cache;
  dd->h = p;
  dd->q = p + d;
  dd->k = p + 2 * d;
  dd->v = p + 3 * d;
  dd->o = p + 4 * d;
  dd->f = p + 5 * d;
  dd->logits = dd->f + c.d_ff;
  dd->state = reinterpret_cast<int32_t*>(dd->logits + c.vocab_size);
  dd->prompt = dd->state + 3;
  dd->out = dd->prompt + max_len;
  // one eager step (state t = 0, token 0) allocates the product workspaces
  // outside the capture; the graph is captured afterwards
  egt_status st = enqueue_step(dd);
  if (st == EGT_OK) {
    cudaGraph_t g = nullptr;
    e = cudaStreamBeginCapture(dd->s, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      st = enqueue_step(dd);
      e = cudaStreamEndCapture(dd->s, &g);
    }
    if (st == EGT_OK && e == cudaSuccess) e = cudaGraphInstantiate(&dd->exec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (st == EGT_OK && e != cudaSuccess) st = dfail(EGT_ECUDA, std::string("decoder: graph capture failed: ") + cudaGetErrorString(e));
  }
  if (st == EGT_OK && cudaStreamSynchronize(dd->s) != cudaSuccess) st = dfail(EGT_ECUDA, "decoder: warm-up step failed");
  if (st != EGT_OK) {
    egt_decoder_destroy(dd);
    return st;
  }
  *out = dd;
  return EGT_OK;
}

egt_status egt_decoder_start(egt_decoder* dd, const int32_t* prompt, uint32_t prompt_len, void* stream) {
  if (!dd || !prompt || prompt_len == 0) return dfail(EGT_EINVAL, "decoder: empty prompt");
  if (prompt_len > dd->max_len) return dfail(EGT_EINVAL, "decoder: prompt longer than max_len");
  for (uint32_t i = 0; i < prompt_len; ++i)
    if (prompt[i] < 0 || static_cast<uint32_t>(prompt[i]) >= dd->m->cfg.vocab_size)
      return dfail(EGT_EINVAL, "decoder: token out of range");
  cudaStream_t us = static_cast<cudaStream_t>(stream);
  const int32_t st[3] = {0, prompt[0], static_cast<int32_t>(prompt_len)};
  DCUDA(cudaEventRecord(dd->ev_in, us));
  DCUDA(cudaStreamWaitEvent(dd->s, dd->ev_in, 0));
  DCUDA(cudaMemcpyAsync(dd->state, st, sizeof(st), cudaMemcpyHostToDevice, dd->s));
  DCUDA(cudaMemcpyAsync(dd->prompt, prompt, prompt_len * sizeof(int32_t), cudaMemcpyHostToDevice, dd->s));
  DCUDA(cudaStreamSynchronize(dd->s));  // the host buffers may be reused on return
  dd->host_t = 0;
  return EGT_OK;
}

egt_status egt_decoder_step(egt_decoder* dd, uint32_t n_steps, void* stream) {
  if (!dd) return dfail(EGT_EINVAL, "decoder: null decoder");
  if (static_cast<uint64_t>(dd->host_t) + n_steps > dd->max_len)
    return dfail(EGT_EINVAL, "decoder: step past max_len");
  dd->host_t += n_steps;
  cudaStream_t us = static_cast<cudaStream_t>(stream);
  DCUDA(cudaEventRecord(dd->ev_in, us));
  DCUDA(cudaStreamWaitEvent(dd->s, dd->ev_in, 0));
  for (uint32_t i = 0; i < n_steps; ++i) DCUDA(cudaGraphLaunch(dd->exec, dd->s));
  DCUDA(cudaEventRecord(dd->ev_out, dd->s));
  DCUDA(cudaStreamWaitEvent(us, dd->ev_out, 0));
  return EGT_OK;
}

egt_status egt_decoder_read(const egt_decoder* dd, int32_t* tokens_host, uint32_t n, uint32_t* position,
                            float* logits_dev, void* stream) {
  if (!dd) return dfail(EGT_EINVAL, "decoder: null decoder");
  cudaStream_t us = static_cast<cudaStream_t>(stream);
  int32_t st[3];
  DCUDA(cudaMemcpyAsync(st, dd->state, sizeof(st), cudaMemcpyDeviceToHost, us));
  if (logits_dev)
    DCUDA(cudaMemcpyAsync(logits_dev, dd->logits, dd->m->cfg.vocab_size * sizeof(float), cudaMemcpyDeviceToDevice, us));
  DCUDA(cudaStreamSynchronize(us));
  const uint32_t t = static_cast<uint32_t>(st[0]);
  if (tokens_host && n) {
    // positions [0, t) were run; the token at position t is pending
    const uint32_t ran = std::min(std::min(n, t), dd->max_len);
    if (ran) DCUDA(cudaMemcpy(tokens_host, dd->out, ran * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (t < n) tokens_host[t] = st[1];
  }
  if (position) *position = t;
  return EGT_OK;
}

egt_status egt_decoder_destroy(egt_decoder* dd) {
  if (dd) {
    if (dd->s) cudaStreamSynchronize(dd->s);
    if (dd->exec) cudaGraphExecDestroy(dd->exec);
    if (dd->ev_in) cudaEventDestroy(dd->ev_in);
    if (dd->ev_out) cudaEventDestroy(dd->ev_out);
    cudaFree(dd->mem);
    if (dd->s) cudaStreamDestroy(dd->s);
    delete dd;
  }
  return EGT_OK;
}

}  // extern "C"
