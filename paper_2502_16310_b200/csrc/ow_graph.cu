// CUDA graph of the fused pass's device-resident level loop.
//
// The loop (bins emission, per level: leaves, marking, propagation, refine
// sweeps; the deepest level's leaves and the driver summary) is ~50 short
// dependent kernels with no host round trip.  Launched one by one, the host
// cannot keep ahead of the GPU (a launch costs about as much host time as
// the kernel takes on the device), so the GPU idles between kernels.  A pass
// whose host-side inputs (pointers, sizes, parameters, scratch slots) equal
// the previous pass's is captured once (cudaStreamBeginCapture) and replayed
// with one cudaGraphLaunch afterwards.
//
// Scans inside a graph cannot take their look-back epoch from a host counter
// (a replay would reuse the baked epochs over status words the previous
// replay tagged): they read a device epoch base that the graph's first
// kernel increments, and use a status array of their own (SLOT_SCAN_STATUS_G);
// epoch = base * 64 + the scan's site in the pass.  When the 16-bit epoch
// field would wrap, that first kernel clears the array.
#include <string.h>

#include <chrono>
#include <functional>

#include "ow_scan.cuh"

namespace {
constexpr int MAX_SITES = (int)ow::GRAPH_SITES;  // scans per captured pass
constexpr int64_t BASE_MAX = (65535 / MAX_SITES) - 1;

__global__ void k_graph_begin(unsigned long long* base, unsigned long long* status, int64_t n_words) {
  __shared__ int s_clear;
  if (threadIdx.x == 0) {
    unsigned long long b = *base + 1;
    s_clear = b > (unsigned long long)BASE_MAX;
    if (s_clear) b = 1;
    *base = b;
  }
  __syncthreads();
  if (s_clear)
    for (int64_t i = threadIdx.x; i < n_words; i += blockDim.x) status[i] = 0ull;
}
}  // namespace

void loop_key_slots(GraphKey* k, const ow_ctx* ctx);

void make_loop_key(GraphKey* k, const ow_ctx* ctx, const ow_forest* f, const float* d_coords, int64_t n_faces,
                   const ow_grid* grid, const ow_nearwall_params* p, const int32_t* ids, const int32_t* counts,
                   const int32_t* offsets, int64_t E, const void* stats, const void* drv) {
  memset(k, 0, sizeof(*k));  // (padding included: keys compare with memcmp)
  k->f = *f;
  if (grid) k->g = *grid;
  k->p = *p;
  k->coords = d_coords;
  k->n_faces = n_faces;
  k->ids = ids;
  k->counts = counts;
  k->offsets = offsets;
  k->E = E;
  k->stats = stats;
  k->drv = drv;
  k->dev = ctx->dev_pass ? 1 : 0;
  loop_key_slots(k, ctx);
}

// scratch slots the captured loop never touches (the lattice stage and the
// cell-face links run after it): left out of the key, so their growth after
// the loop does not defeat the capture of the next pass
static bool slot_outside_loop(int i) {
  switch (i) {
    case SLOT_SCAN_STATUS_G:  // (allocated by the capture itself)
    case SLOT_LINK_CNT: case SLOT_LINK_OFF: case SLOT_LINK_CELLOFF: case SLOT_LINK_LEAVES:
    case SLOT_LAT_BCOUNT: case SLOT_LAT_BOFFS: case SLOT_LAT_LEAVES: case SLOT_LAT_RANK: case SLOT_LAT_POS:
    case SLOT_LAT_HAS: case SLOT_LAT_CEN: case SLOT_LAT_REC: case SLOT_LAT_ROWS: case SLOT_LAT_ROWOFF:
    case SLOT_LAT_TILEROW: case SLOT_LAT_HITS: case SLOT_LAT_HITDIR: case SLOT_LAT_TILEHITS: case SLOT_LAT_IHITS:
    case SLOT_LAT_IHITDIR: case SLOT_LAT_BMASK: case SLOT_LAT_HCOUNT: case SLOT_LAT_HOFFS: case SLOT_LAT_RFLAGS:
    case SLOT_LAT_QPACK: case SLOT_LAT_GRID: case SLOT_MISC:
      return true;
    default:
      return false;
  }
}

void loop_key_slots(GraphKey* k, const ow_ctx* ctx) {
  for (int i = 0; i < SLOT_COUNT; ++i) {
    const bool out = slot_outside_loop(i);
    k->slot_ptr[i] = out ? nullptr : ctx->slot_ptr[i];
    k->slot_bytes[i] = out ? 0 : ctx->slot_bytes[i];
  }
}

// Runs body() for the loop: replays a cached graph whose key matches
// (returns -1: nothing ran on the host), captures and launches a new graph
// when the key matches a recent eager pass's, else runs body() eagerly
// (returns its status).  Never leaves a stream in capture mode.
int ow_loop_graph(ow_ctx* ctx, bool ok, const GraphKey* key, cudaStream_t* ps, const std::function<int()>& body) {
  constexpr int NG = 4;
  const cudaStream_t s = *ps;
  static const bool disabled = getenv("OW_NO_GRAPHS") != nullptr;
  if (!ok || disabled) return body();
  for (int i = 0; i < NG; ++i) {
    if (!ctx->loop_key[i]) ctx->loop_key[i] = (GraphKey*)calloc(1, sizeof(GraphKey));
    if (!ctx->eager_key[i]) ctx->eager_key[i] = (GraphKey*)calloc(1, sizeof(GraphKey));
    if (!ctx->loop_key[i] || !ctx->eager_key[i]) return body();
  }
  for (int i = 0; i < NG; ++i)
    if (ctx->loop_exec[i] && memcmp(ctx->loop_key[i], key, sizeof(GraphKey)) == 0) {
      static const bool timed = getenv("OW_TIME_GRAPH") != nullptr;
      const auto t0 = std::chrono::steady_clock::now();
      OW_CUDA(cudaGraphLaunch(ctx->loop_exec[i], s));
      if (timed) {
        static double acc = 0.0;
        static int n = 0;
        acc += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        if (++n % 20 == 0) fprintf(stderr, "graph launch: %.1f us host (mean of 20, %lld kernels)\n", acc / 20,
                                   (long long)ctx->loop_launches[i]);
        if (n % 20 == 0) acc = 0.0;
      }
      ctx->launches += ctx->loop_launches[i];
      ctx->prep_key = -1;  // (the face-prep cache is not tracked across replays)
      return -1;
    }
  int ek = -1;
  for (int i = 0; i < NG; ++i)
    if (memcmp(ctx->eager_key[i], key, sizeof(GraphKey)) == 0) ek = i;
  if (ek < 0) {
    // first pass with these inputs: run eagerly (it sizes every scratch slot);
    // the key is recorded with the slots as this pass left them, so the next
    // pass with the same inputs is captured even when this one grew scratch
    if (getenv("OW_DEBUG_GRAPH")) fprintf(stderr, "ow graph: eager pass (dev=%d)\n", key->dev);
    const int e = ctx->eager_next;
    *ctx->eager_key[e] = *key;
    ctx->eager_next = (e + 1) % NG;
    const int st = body();
    loop_key_slots(ctx->eager_key[e], ctx);
    return st;
  }
  // second pass with the same inputs: capture the loop, then launch it
  memset(ctx->eager_key[ek], 0, sizeof(GraphKey));  // (one capture attempt per eager pass)
  static const bool dbg = getenv("OW_DEBUG_GRAPH") != nullptr;
  if (dbg) fprintf(stderr, "ow graph: capture attempt (dev=%d)\n", key->dev);
  if (!ctx->d_graph_epoch) {
    OW_CUDA(cudaMalloc((void**)&ctx->d_graph_epoch, 64));
    OW_CUDA(cudaMemsetAsync(ctx->d_graph_epoch, 0, 64, s));
  }
  const int64_t words = (ctx->slot_bytes[SLOT_SCAN_STATUS] / 8 > 4096 ? ctx->slot_bytes[SLOT_SCAN_STATUS] / 8 : 4096);
  if (ctx->slot_bytes[SLOT_SCAN_STATUS_G] < 8 * (size_t)words) {
    void* pg;
    OW_TRY(ow_slot(ctx, SLOT_SCAN_STATUS_G, 8 * (size_t)words, s, &pg));
    OW_CUDA(cudaMemsetAsync(pg, 0, ctx->slot_bytes[SLOT_SCAN_STATUS_G], s));
  }
  cudaGraph_t graph = nullptr;
  ctx->prep_key = -1;  // the face payload kernel must be part of the graph
  if (!ctx->capture_stream) OW_CUDA(cudaStreamCreateWithFlags(&ctx->capture_stream, cudaStreamNonBlocking));
  const int64_t launches0 = ctx->launches;
  // record on the private stream (the body launches on *ps); the graph is
  // then launched on the caller's stream, ordered after its earlier work
  OW_CUDA(cudaStreamBeginCapture(ctx->capture_stream, cudaStreamCaptureModeThreadLocal));
  *ps = ctx->capture_stream;
  ctx->capturing = true;
  ctx->capture_failed = false;
  ctx->graph_site = 0;
  ow_launch(k_graph_begin, 1, 256, 0, ctx->capture_stream, ctx->d_graph_epoch,
            (unsigned long long*)ctx->slot_ptr[SLOT_SCAN_STATUS_G], (int64_t)(ctx->slot_bytes[SLOT_SCAN_STATUS_G] / 8));
  OW_LAUNCHED(ctx);
  const int st = body();
  ctx->capturing = false;
  *ps = s;
  const cudaError_t ce = cudaStreamEndCapture(ctx->capture_stream, &graph);
  cudaGetLastError();
  const bool good = st == OW_OK && ce == cudaSuccess && graph && !ctx->capture_failed &&
                    ctx->graph_site <= MAX_SITES;
  if (!good) {
    if (dbg) fprintf(stderr, "ow graph: capture failed (%s)\n", ow_last_error());
    if (graph) cudaGraphDestroy(graph);
    ctx->launches = launches0;
    if (st != OW_OK && !ctx->capture_failed) return st;
    return body();  // (scratch had to grow, or too many scan sites: eager)
  }
  const int v = ctx->loop_next;
  cudaGraphExec_t exec = nullptr;
  cudaError_t e = cudaErrorUnknown;
  if (ctx->loop_exec[v]) {  // the victim's executable takes the new graph in place when it can
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(ctx->loop_exec[v], graph, &info) == cudaSuccess) {
      exec = ctx->loop_exec[v];
      e = cudaSuccess;
    } else {
      cudaGetLastError();
      cudaGraphExecDestroy(ctx->loop_exec[v]);
      ctx->loop_exec[v] = nullptr;
    }
  }
  if (!exec) e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->launches = launches0;
    return body();
  }
  cudaGraphUpload(exec, s);  // (device-side resources staged once: lower launch latency)
  cudaGetLastError();
  ctx->loop_exec[v] = exec;
  *ctx->loop_key[v] = *key;
  ctx->loop_launches[v] = ctx->launches - launches0;
  ctx->loop_next = (v + 1) % NG;
  OW_CUDA(cudaGraphLaunch(exec, s));
  ctx->prep_key = -1;
  return OW_OK;
}
