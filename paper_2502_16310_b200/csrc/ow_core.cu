// Context, error state, scratch slots and readback for libowb200.
#include <stdlib.h>
#include <stdarg.h>
#include <string.h>

#include "ow_common.cuh"

static thread_local char g_err[1024] = "";

void ow_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* ow_last_error(void) { return g_err; }

extern "C" int ow_version(void) { return 10000; }  // 1.0.0

extern "C" int64_t ow_launch_count(ow_ctx* ctx) { return ctx ? ctx->launches : 0; }

extern "C" int ow_ctx_create(int device, ow_ctx** out) {
  if (!out) {
    ow_set_error("ow_ctx_create: null out pointer");
    return OW_ERR_INVALID;
  }
  OW_CUDA(cudaSetDevice(device));
  ow_ctx* c = (ow_ctx*)calloc(1, sizeof(ow_ctx));
  if (!c) {
    ow_set_error("ow_ctx_create: out of host memory");
    return OW_ERR_INTERNAL;
  }
  c->device = device;
  c->prep_key = -1;
  cudaError_t e = cudaMallocHost((void**)&c->h_pinned, OW_PINNED_WORDS * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc((void**)&c->d_small, 64 * sizeof(int64_t));
  // (the readbacks copy contiguous runs of these words, spare ones included:
  // defined from the start, compute-sanitizer initcheck stays clean)
  if (e == cudaSuccess) e = cudaMemset(c->d_small, 0, 64 * sizeof(int64_t));
  if (e != cudaSuccess) {
    ow_set_error("ow_ctx_create: %s", cudaGetErrorString(e));
    free(c);
    return OW_ERR_INTERNAL;
  }
  *out = c;
  return OW_OK;
}

extern "C" int ow_ctx_destroy(ow_ctx* c) {
  if (!c) return OW_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int i = 0; i < SLOT_COUNT; ++i)
    if (c->slot_ptr[i]) cudaFree(c->slot_ptr[i]);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (int i = 0; i < 4; ++i) {
    if (c->loop_exec[i]) cudaGraphExecDestroy(c->loop_exec[i]);
    free(c->loop_key[i]);
    free(c->eager_key[i]);
  }
  if (c->capture_stream) cudaStreamDestroy(c->capture_stream);
  if (c->d_graph_epoch) cudaFree(c->d_graph_epoch);
  for (int i = 0; i < 2; ++i)
    if (c->copy_ev[i]) cudaEventDestroy(c->copy_ev[i]);
  if (c->stage_events) {
    cudaEvent_t* ev = (cudaEvent_t*)c->stage_events;  // StageEvents starts with its event table
    for (int i = 0; i < OW_MAX_PASSES * 5; ++i)
      if (ev[i]) cudaEventDestroy(ev[i]);
    free(c->stage_events);
  }
  if (c->prof) {
    for (int i = 0; i < PROF_N; ++i)
      for (int k = 0; k < PROF_MAX; ++k)
        for (int j = 0; j < 2; ++j)
          if (c->prof->ev[i][k][j]) cudaEventDestroy(c->prof->ev[i][k][j]);
    free(c->prof);
  }
  ow_g2g_release(c);
  cudaFreeHost(c->h_pinned);
  cudaFree(c->d_small);
  free(c);
  return OW_OK;
}

int ow_slot(ow_ctx* ctx, int slot, size_t bytes, cudaStream_t s, void** out) {
  if (bytes == 0) bytes = 16;
  if (ctx->slot_bytes[slot] < bytes && ctx->capturing) {  // (a graph must not own scratch: run eagerly)
    ctx->capture_failed = true;
    ow_set_error("graph capture: scratch slot %d would grow", slot);
    return OW_ERR_INTERNAL;
  }
  if (ctx->slot_bytes[slot] < bytes) {
    size_t want = bytes + bytes / 4 + 256;
    if (ctx->slot_ptr[slot]) OW_CUDA(cudaFreeAsync(ctx->slot_ptr[slot], s));
    ctx->slot_ptr[slot] = nullptr;
    ctx->slot_bytes[slot] = 0;
    OW_CUDA(cudaMallocAsync(&ctx->slot_ptr[slot], want, s));
    ctx->slot_bytes[slot] = want;
  }
  *out = ctx->slot_ptr[slot];
  return OW_OK;
}

void ow_prof_mark(ow_ctx* ctx, int id, int end, cudaStream_t s) {
  ow_prof* p = ctx->prof;
  int k = p->n[id];
  if (k >= PROF_MAX) return;
  cudaEvent_t* e = &p->ev[id][k][end];
  if (!*e) cudaEventCreate(e);
  cudaEventRecord(*e, s);
  if (end) p->n[id] = k + 1;
}

extern "C" int ow_profile(ow_ctx* ctx, int enable) {
  if (!ctx->prof) {
    ctx->prof = (ow_prof*)calloc(1, sizeof(ow_prof));
    if (!ctx->prof) {
      ow_set_error("ow_profile: out of host memory");
      return OW_ERR_INTERNAL;
    }
  }
  ctx->prof->enabled = enable;
  for (int i = 0; i < PROF_N; ++i) ctx->prof->n[i] = 0;
  return OW_OK;
}

extern "C" int ow_profile_read(ow_ctx* ctx, int id, double* total_ms, int64_t* launches) {
  *total_ms = 0.0;
  *launches = 0;
  if (!ctx->prof || id < 0 || id >= PROF_N) return OW_OK;
  ow_prof* p = ctx->prof;
  for (int k = 0; k < p->n[id]; ++k) {
    OW_CUDA(cudaEventSynchronize(p->ev[id][k][1]));
    float ms = 0.0f;
    OW_CUDA(cudaEventElapsedTime(&ms, p->ev[id][k][0], p->ev[id][k][1]));
    *total_ms += ms;
  }
  *launches = p->n[id];
  return OW_OK;
}

int ow_readback(ow_ctx* ctx, const int64_t* d_src, int n, int64_t* h_dst, cudaStream_t s) {
  OW_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_src, n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  OW_CUDA(cudaStreamSynchronize(s));
  memcpy(h_dst, ctx->h_pinned, n * sizeof(int64_t));
  return OW_OK;
}

bool ow_pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("OW_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// ---------------------------------------------------------------------------
// memset as a kernel: it joins the programmatic-dependent-launch chain of the
// kernels around it (a cudaMemsetAsync node breaks the overlap and costs a
// launch bubble in the level loop)
// ---------------------------------------------------------------------------
namespace {
__global__ void k_fill(uint32_t* __restrict__ w, int64_t n_words, uint8_t* __restrict__ tail, int n_tail, uint32_t v) {
  ow_pdl_wait();
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  // 16-byte stores for the aligned body (w is 4-byte aligned; the head up to
  // 16-byte alignment and the remainder word by word)
  const int64_t head = (int64_t)(((16 - ((uintptr_t)w & 15u)) & 15u) >> 2);
  const int64_t h = head < n_words ? head : n_words;
  const int64_t n4 = (n_words - h) >> 2;
  uint4* w4 = reinterpret_cast<uint4*>(w + h);
  const uint4 v4 = make_uint4(v, v, v, v);
  for (int64_t i = i0; i < n4; i += stride) w4[i] = v4;
  for (int64_t i = i0; i < h; i += stride) w[i] = v;
  for (int64_t i = h + 4 * n4 + i0; i < n_words; i += stride) w[i] = v;
  if (i0 < n_tail) tail[i0] = (uint8_t)v;
}
}  // namespace

int ow_fill_async(ow_ctx* ctx, void* p, int value, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return OW_OK;
  if (((uintptr_t)p & 3u) != 0) {
    OW_CUDA(cudaMemsetAsync(p, value, bytes, s));
    return OW_OK;
  }
  const uint32_t b = (uint32_t)(value & 0xFF);
  const int64_t n_words = (int64_t)(bytes >> 2);
  const int n_tail = (int)(bytes & 3u);
  ow_launch(k_fill, ow_blocks(n_words > 0 ? (n_words + 3) / 4 : 1, 256, 8 * OW_SMS), 256, 0, s, (uint32_t*)p, n_words,
            (uint8_t*)p + 4 * n_words, n_tail, b | b << 8 | b << 16 | b << 24);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}
