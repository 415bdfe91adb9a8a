// Device-side exchange between the ranks of one node over peer memory
// (multi-GPU).  One process per GPU; every rank owns one
// symmetric buffer (cudaMalloc) whose CUDA IPC handle the others map
// (cudaIpcOpenMemHandle, peer access over NVLink / NVSwitch, or the same
// device when ranks share a GPU).  An exchange is two stream-ordered kernels
// and no host round trip:
//
//   put : the rank stores its own slice of an array straight into every
//         peer's buffer (P2P stores), then the last CTA releases its epoch
//         into each peer's flag word for this rank (st.release.sys);
//   get : CTAs acquire every peer's flag (ld.acquire.sys spin, bounded by a
//         timeout that raises an error word instead of hanging the GPU) and
//         copy the other ranks' slices from the local buffer into the array.
//
// Ranks' slices partition the array, so after the exchange every rank holds
// the whole array (an all-gather of disjoint ranges).  Two data areas
// alternate by epoch parity: a fast rank's next put cannot land in an area a
// slow rank is still reading (it needs that rank's next put first).
//
// Users: the native level loop (marks of each rank's leaf slice + marking
// statistics) and the lattice stage (flag words of each rank's finest-leaf
// slice, q rows of its boundary cells) in ow_geometry_to_grid.
#include <string.h>

#include "ow_scan.cuh"

namespace {

constexpr int HDR_FLAG_STRIDE = 16;            // int64 words between two flag words (128 B)
constexpr size_t HDR_STATS = 8 * 128;          // byte offset of the per-rank stats slots (2 parities x 8 x 64 B)
constexpr size_t HDR_BYTES = 4096;             // header bytes before the two data areas
constexpr unsigned long long TIMEOUT_NS = 60ull * 1000000000ull;

struct Peers {
  uint8_t* p[OW_COMM_MAX];
};

__device__ __forceinline__ void st_release_sys(int64_t* a, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* a) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// thread 0 of each CTA waits for every peer's epoch; the CTA follows
__device__ __forceinline__ bool wait_peers(const uint8_t* local, int world, int rank, int64_t epoch, int64_t* err) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = 1;
    const int64_t* flags = reinterpret_cast<const int64_t*>(local);
    const unsigned long long t0 = globaltimer();
    for (int r = 0; r < world && ok; ++r) {
      if (r == rank) continue;
      while (ld_acquire_sys(flags + r * HDR_FLAG_STRIDE) < epoch) {
        if (globaltimer() - t0 > TIMEOUT_NS || ld_acquire_sys(err) != 0) {
          atomicExch(reinterpret_cast<unsigned long long*>(err), 1ull);
          ok = 0;
          break;
        }
        __nanosleep(256);
      }
    }
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// the last CTA to finish its stores releases the epoch to every peer
__device__ __forceinline__ void signal_peers(Peers P, int world, int rank, int64_t epoch, unsigned* counter) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      __threadfence_system();
      for (int r = 0; r < world; ++r)
        if (r != rank) st_release_sys(reinterpret_cast<int64_t*>(P.p[r]) + rank * HDR_FLAG_STRIDE, epoch);
      *counter = 0u;  // (the next put starts after this kernel)
    }
  }
}

// 32-bit words [lo, hi) of src -> the same words of every peer's area
__global__ void k_xput_u32(Peers P, int world, int rank, size_t area, const uint32_t* __restrict__ src,
                           const int64_t* range, int64_t h_lo, int64_t h_hi, int64_t epoch, unsigned* counter) {
  ow_pdl_wait();
  const int64_t lo = range ? range[0] : h_lo, hi = range ? range[1] : h_hi;
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = src[i];
    for (int r = 0; r < world; ++r)
      if (r != rank) reinterpret_cast<uint32_t*>(P.p[r] + area)[i] = v;
  }
  signal_peers(P, world, rank, epoch, counter);
}

// every word of [0, n) outside [lo, hi) from the local area into dst
__global__ void k_xget_u32(const uint8_t* local, int world, int rank, size_t area, uint32_t* dst, const int64_t* range,
                           int64_t h_lo, int64_t h_hi, const int64_t* d_n, int64_t h_n, int64_t epoch, int64_t* err) {
  ow_pdl_wait();
  if (!wait_peers(local, world, rank, epoch, err)) return;
  const int64_t lo = range ? range[0] : h_lo, hi = range ? range[1] : h_hi, n = d_n ? *d_n : h_n;
  const uint32_t* a = reinterpret_cast<const uint32_t*>(local + area);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (i < lo || i >= hi) dst[i] = a[i];
}

// marks of the leaves at positions [lo, hi) (byte per position) + the
// rank's marking statistics -> every peer
__global__ void k_xput_marks(Peers P, int world, int rank, size_t area, const int32_t* __restrict__ leaves,
                             const int8_t* __restrict__ marks, const int64_t* slice, const unsigned long long* stats,
                             int n_stats, int64_t epoch, unsigned* counter) {
  const size_t slots = HDR_STATS + 512 * (size_t)(epoch & 1);
  ow_pdl_wait();
  const int64_t lo = slice[0], hi = slice[1];
  // interior words are written whole; the (at most two) edge words byte by
  // byte: the bytes next to the slice belong to other ranks' concurrent puts
  const int64_t w0 = (lo + 3) >> 2, w1 = hi >> 2;
  for (int64_t w = w0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < w1; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v |= (uint32_t)(uint8_t)marks[leaves[4 * w + k]] << (8 * k);
    for (int r = 0; r < world; ++r)
      if (r != rank) reinterpret_cast<uint32_t*>(P.p[r] + area)[w] = v;
  }
  if (blockIdx.x == 0) {
    for (int64_t i = lo + threadIdx.x; i < hi && i < 4 * w0; i += blockDim.x) {
      const int8_t v = marks[leaves[i]];
      for (int r = 0; r < world; ++r)
        if (r != rank) reinterpret_cast<int8_t*>(P.p[r] + area)[i] = v;
    }
    for (int64_t i = (4 * w1 > lo ? 4 * w1 : lo) + threadIdx.x; i < hi; i += blockDim.x) {
      const int8_t v = marks[leaves[i]];
      for (int r = 0; r < world; ++r)
        if (r != rank) reinterpret_cast<int8_t*>(P.p[r] + area)[i] = v;
    }
    if (threadIdx.x < n_stats)
      for (int r = 0; r < world; ++r)  // own slot too: the get sums every slot
        reinterpret_cast<unsigned long long*>(P.p[r] + slots + 64 * rank)[threadIdx.x] = stats[threadIdx.x];
  }
  signal_peers(P, world, rank, epoch, counter);
}

__global__ void k_xget_marks(const uint8_t* local, int world, int rank, size_t area, const int32_t* __restrict__ leaves,
                             int8_t* marks, const int64_t* slice, const int64_t* d_n, unsigned long long* stats,
                             int n_stats, int64_t epoch, int64_t* err) {
  ow_pdl_wait();
  if (!wait_peers(local, world, rank, epoch, err)) return;
  const int64_t lo = slice[0], hi = slice[1], n = *d_n;
  const int8_t* a = reinterpret_cast<const int8_t*>(local + area);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (i < lo || i >= hi) marks[leaves[i]] = a[i];
  if (blockIdx.x == 0 && threadIdx.x < n_stats) {
    unsigned long long sum = 0;
    for (int r = 0; r < world; ++r)
      sum += reinterpret_cast<const unsigned long long*>(local + HDR_STATS + 512 * (size_t)(epoch & 1) + 64 * r)[threadIdx.x];
    stats[threadIdx.x] = sum;
  }
}

Peers peers_of(const ow_comm* c) {
  Peers P;
  memset(&P, 0, sizeof(P));
  for (int r = 0; r < c->world; ++r) P.p[r] = c->peer[r];
  return P;
}

unsigned xgrid(int64_t n) { return (unsigned)ow_blocks(n, 256, 2 * OW_SMS); }

}  // namespace

size_t ow_comm_area(const ow_comm* c, int64_t epoch) { return HDR_BYTES + (size_t)(epoch & 1) * c->area_bytes; }

int ow_comm_check(ow_comm* c, int64_t bytes, const char* what) {
  if (bytes > c->area_bytes) {
    ow_set_error("multi-GPU exchange: %s needs %lld bytes, the exchange buffer holds %lld (create the ow_comm "
                 "with more room)", what, (long long)bytes, (long long)c->area_bytes);
    return OW_ERR_CAPACITY;
  }
  return OW_OK;
}

int ow_comm_allgather_words(ow_ctx* ctx, ow_comm* c, uint32_t* d_data, const int64_t* d_range, int64_t lo, int64_t hi,
                            const int64_t* d_n, int64_t n, cudaStream_t s) {
  if (c->world <= 1) return OW_OK;
  const int64_t bound = d_n ? n : n;  // n bounds the array either way
  OW_TRY(ow_comm_check(c, 4 * bound, "an all-gather"));
  const int64_t epoch = ++c->epoch;
  const size_t area = ow_comm_area(c, epoch);
  ow_launch(k_xput_u32, xgrid(d_range ? n : hi - lo), 256, 0, s, peers_of(c), c->world, c->rank, area,
            (const uint32_t*)d_data, d_range, lo, hi, epoch, c->d_counter);
  ow_launch(k_xget_u32, xgrid(n), 256, 0, s, (const uint8_t*)c->local, c->world, c->rank, area, d_data, d_range, lo,
            hi, d_n, n, epoch, c->d_err);
  ctx->launches += 2;
  OW_CHECK_LAUNCH();
  return OW_OK;
}

int ow_comm_exchange_marks(ow_ctx* ctx, ow_comm* c, const int32_t* d_leaves, int8_t* d_marks, const int64_t* d_slice,
                           const int64_t* d_n, int64_t n_bound, unsigned long long* d_stats, int n_stats,
                           cudaStream_t s) {
  OW_TRY(ow_comm_check(c, n_bound + 8, "the marks of a level"));
  const int64_t epoch = ++c->epoch;
  const size_t area = ow_comm_area(c, epoch);
  ow_launch(k_xput_marks, xgrid(n_bound / 4 + 1), 256, 0, s, peers_of(c), c->world, c->rank, area, d_leaves,
            (const int8_t*)d_marks, d_slice, (const unsigned long long*)d_stats, n_stats, epoch, c->d_counter);
  ow_launch(k_xget_marks, xgrid(n_bound), 256, 0, s, (const uint8_t*)c->local, c->world, c->rank, area, d_leaves,
            d_marks, d_slice, d_n, d_stats, n_stats, epoch, c->d_err);
  ctx->launches += 2;
  OW_CHECK_LAUNCH();
  return OW_OK;
}

extern "C" int ow_comm_create(int device, int32_t rank, int32_t world, int64_t area_bytes, ow_comm** out,
                              void* handle) {
  if (!out || !handle || world < 1 || world > OW_COMM_MAX || rank < 0 || rank >= world || area_bytes < 0) {
    ow_set_error("ow_comm_create: bad rank %d / world %d (at most %d ranks) or size", rank, world, OW_COMM_MAX);
    return OW_ERR_INVALID;
  }
  OW_CUDA(cudaSetDevice(device));
  ow_comm* c = (ow_comm*)calloc(1, sizeof(ow_comm));
  if (!c) {
    ow_set_error("ow_comm_create: out of host memory");
    return OW_ERR_INTERNAL;
  }
  c->device = device;
  c->rank = rank;
  c->world = world;
  c->area_bytes = (area_bytes + 255) & ~int64_t(255);
  const size_t total = HDR_BYTES + 2 * (size_t)c->area_bytes;
  cudaError_t e = cudaMalloc(&c->local, total);
  if (e == cudaSuccess) e = cudaMemset(c->local, 0, HDR_BYTES);
  if (e == cudaSuccess) e = cudaMalloc((void**)&c->d_err, 64);
  if (e == cudaSuccess) e = cudaMemset(c->d_err, 0, 64);
  if (e == cudaSuccess) c->d_counter = (unsigned*)(c->d_err + 4);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, c->local);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    ow_set_error("ow_comm_create: %s", cudaGetErrorString(e));
    if (c->local) cudaFree(c->local);
    if (c->d_err) cudaFree(c->d_err);
    free(c);
    return OW_ERR_INTERNAL;
  }
  memcpy(handle, &h, sizeof(h));
  c->peer[rank] = (uint8_t*)c->local;
  *out = c;
  return OW_OK;
}

extern "C" int ow_comm_open(ow_comm* c, const void* handles) {
  OW_CUDA(cudaSetDevice(c->device));
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank || c->peer[r]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const uint8_t*)handles + sizeof(cudaIpcMemHandle_t) * r, sizeof(h));
    void* p = nullptr;
    OW_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->peer[r] = (uint8_t*)p;
  }
  c->open = 1;
  return OW_OK;
}

// first device error word (1: a peer did not arrive within the timeout)
extern "C" int ow_comm_status(ow_comm* c, int64_t* out) {
  OW_CUDA(cudaSetDevice(c->device));
  OW_CUDA(cudaMemcpy(out, c->d_err, sizeof(int64_t), cudaMemcpyDeviceToHost));
  return OW_OK;
}

// all-gather of disjoint word ranges: this rank's [lo, hi) of the n words at
// d_data reach every rank, and every rank's array ends up whole (tests and
// user code; the level loop uses the same kernels)
extern "C" int ow_comm_allgather_u32(ow_ctx* ctx, ow_comm* c, uint32_t* d_data, int64_t lo, int64_t hi, int64_t n,
                                     void* stream) {
  if (!c->open || lo < 0 || hi < lo || hi > n) {
    ow_set_error("ow_comm_allgather_u32: unopened comm or bad range [%lld, %lld) of %lld", (long long)lo,
                 (long long)hi, (long long)n);
    return OW_ERR_INVALID;
  }
  return ow_comm_allgather_words(ctx, c, d_data, nullptr, lo, hi, nullptr, n, (cudaStream_t)stream);
}

extern "C" int ow_comm_destroy(ow_comm* c) {
  if (!c) return OW_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < c->world; ++r)
    if (r != c->rank && c->peer[r]) cudaIpcCloseMemHandle(c->peer[r]);
  cudaFree(c->local);
  cudaFree(c->d_err);
  free(c);
  return OW_OK;
}
