// Single-pass exclusive scan with decoupled look-back, and a stable LSD radix
// sort of (u32 key, i32 value) pairs built on it.  Both are generic over
// functors so compaction / ranking / CSR offsets fuse into the scan pass.
#pragma once

#include "ow_common.cuh"

namespace ow {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;
// Status words carry an epoch so the array never needs clearing between
// scans: [63:62] flag (1 aggregate, 2 inclusive prefix), [61:46] epoch,
// [45:0] value (sums < 2^46).  The tile-ticket counter is reset by the last
// tile to finish.
constexpr unsigned long long ST_AGG = 1ull << 62;
constexpr unsigned long long ST_INC = 2ull << 62;
constexpr unsigned long long ST_VAL = (1ull << 46) - 1;
constexpr int ST_EPOCH_SHIFT = 46;

__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Load: int64_t operator()(int64_t i) const      (non-negative values)
// Store: void operator()(int64_t i, int64_t exclusive_prefix, int64_t value) const
template <class Load, class Store>
__global__ void __launch_bounds__(SCAN_THREADS)
k_scan(Load load, Store store, int64_t n, int64_t n_tiles, unsigned long long* status, unsigned int* tile_ctr,
       int64_t* total_out, unsigned long long epoch) {
  __shared__ int s_tile;
  __shared__ int64_t s_warp[SCAN_THREADS / 32];
  __shared__ int64_t s_prefix;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS];
  int64_t sum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + k;
    v[k] = (i < n) ? load(i) : 0;
    sum += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = (lane < SCAN_THREADS / 32) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < SCAN_THREADS / 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < SCAN_THREADS / 32) s_warp[lane] = w;
  }
  __syncthreads();
  const int64_t agg = s_warp[SCAN_THREADS / 32 - 1];
  const int64_t thread_excl = (warp ? s_warp[warp - 1] : 0) + x - sum;
  const unsigned long long tag = epoch << ST_EPOCH_SHIFT;
  if (warp == 0) {
    // decoupled look-back, one warp: publish the aggregate, then inspect a
    // window of 32 predecessors per step (lane k reads tile p - k) until an
    // inclusive prefix appears; each step costs one round of parallel loads
    int64_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) st_status(&status[0], ST_INC | tag | (unsigned long long)agg);
    } else {
      if (lane == 0) st_status(&status[tile], ST_AGG | tag | (unsigned long long)agg);
      int64_t p = tile - 1;  // newest predecessor of the current window
      while (true) {
        const int64_t q = p - lane;
        unsigned long long st = 0;
        bool ready = true;
        if (q >= 0) {
          st = ld_status(&status[q]);
          ready = ((st & ~(3ull << 62)) >> ST_EPOCH_SHIFT) == epoch;
        }
        if (!__all_sync(0xffffffffu, ready)) continue;  // some predecessor not yet published
        const bool inc = q >= 0 && (st >> 62) == 2;
        const unsigned im = __ballot_sync(0xffffffffu, inc);
        // lanes up to (and including) the nearest inclusive one contribute
        const int stop = im ? __ffs(im) - 1 : 31;
        int64_t val = (q >= 0 && lane <= stop) ? (int64_t)(st & ST_VAL) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        if (im || p - 31 < 0) break;
        p -= 32;
      }
      if (lane == 0) st_status(&status[tile], ST_INC | tag | (unsigned long long)(prefix + agg));
    }
    if (lane == 0) {
      s_prefix = prefix;
      if (tile == n_tiles - 1 && total_out) *total_out = prefix + agg;
    }
  }
  __syncthreads();
  int64_t run = s_prefix + thread_excl;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + k;
    if (i < n) store(i, run, v[k]);
    run += v[k];
  }
  if (threadIdx.x == 0) {  // last tile out resets the ticket counters for the next scan
    __threadfence();
    if (atomicAdd(tile_ctr + 1, 1u) == (unsigned)(n_tiles - 1)) {
      tile_ctr[0] = 0;
      tile_ctr[1] = 0;
    }
  }
}

// Exclusive scan of load(0..n-1); *d_total (device) receives the sum.
template <class Load, class Store>
int scan(ow_ctx* ctx, Load load, Store store, int64_t n, int64_t* d_total, cudaStream_t s) {
  if (n <= 0) {
    if (d_total) OW_CUDA(cudaMemsetAsync(d_total, 0, sizeof(int64_t), s));
    return OW_OK;
  }
  int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  const size_t need = 8 * (size_t)(tiles + 1);
  void* old = ctx->slot_ptr[SLOT_SCAN_STATUS];
  const size_t old_bytes = ctx->slot_bytes[SLOT_SCAN_STATUS];
  void* p;
  OW_TRY(ow_slot(ctx, SLOT_SCAN_STATUS, need, s, &p));
  if (p != old || ctx->slot_bytes[SLOT_SCAN_STATUS] != old_bytes || ctx->scan_epoch >= 65535) {
    // fresh (or wrapped) status array: clear once, epochs restart at 1
    OW_CUDA(cudaMemsetAsync(p, 0, ctx->slot_bytes[SLOT_SCAN_STATUS], s));
    ctx->scan_epoch = 0;
  }
  const unsigned long long epoch = (unsigned long long)(++ctx->scan_epoch);
  unsigned long long* status = (unsigned long long*)p + 1;  // word 0: ticket counters
  k_scan<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(load, store, n, tiles, status, (unsigned int*)p, d_total, epoch);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

// ---- common functors --------------------------------------------------------
template <class T>
struct LoadArr {
  const T* a;
  __device__ int64_t operator()(int64_t i) const { return (int64_t)a[i]; }
};
template <class T>
struct StoreExcl {  // out[i] = exclusive prefix
  T* out;
  __device__ void operator()(int64_t i, int64_t e, int64_t) const { out[i] = (T)e; }
};

// ---- stable LSD radix sort of (key, value) ----------------------------------
constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
constexpr int RS_BITS = 8;
constexpr int RS_DIGITS = 1 << RS_BITS;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_WARP_ITEMS = RS_TILE / RS_WARPS;  // 512 contiguous items per warp

static __global__ void __launch_bounds__(RS_THREADS)
k_radix_hist(const uint32_t* keys, int64_t n, int shift, int64_t n_tiles, int32_t* hist) {
  __shared__ int h[RS_DIGITS];
  for (int d = threadIdx.x; d < RS_DIGITS; d += RS_THREADS) h[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
  for (int k = 0; k < RS_ITEMS; ++k) {
    int64_t i = base + (int64_t)k * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & (RS_DIGITS - 1)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < RS_DIGITS; d += RS_THREADS) hist[(int64_t)d * n_tiles + blockIdx.x] = h[d];
}

static __global__ void __launch_bounds__(RS_THREADS)
k_radix_scatter(const uint32_t* keys, const int32_t* vals, int64_t n, int shift, int64_t n_tiles,
                const int32_t* hist_excl, uint32_t* keys_out, int32_t* vals_out) {
  __shared__ int cnt[RS_WARPS][RS_DIGITS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = lane; d < RS_DIGITS; d += 32) cnt[warp][d] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE + (int64_t)warp * RS_WARP_ITEMS;
  uint32_t kk[RS_ITEMS];
  int32_t vv[RS_ITEMS];
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    int64_t i = base + r * 32 + lane;
    bool ok = i < n;
    kk[r] = ok ? keys[i] : 0u;
    vv[r] = ok ? vals[i] : 0;
    int d = ok ? (int)((kk[r] >> shift) & (RS_DIGITS - 1)) : RS_DIGITS;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    if (ok && lane == __ffs(peers) - 1) cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < RS_DIGITS; d += RS_THREADS) {
    int run = hist_excl[(int64_t)d * n_tiles + blockIdx.x];
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      int c = cnt[w][d];
      cnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    int64_t i = base + r * 32 + lane;
    bool ok = i < n;
    int d = ok ? (int)((kk[r] >> shift) & (RS_DIGITS - 1)) : RS_DIGITS;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    if (ok) {
      int pos = cnt[warp][d] + __popc(peers & lanemask_lt());
      keys_out[pos] = kk[r];
      vals_out[pos] = vv[r];
    }
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
}

// Sort n pairs by the low `key_bits` bits of key, stably.  Input in (k0, v0);
// the sorted result pointer pair is returned through (*rk, *rv), which is
// either (k0, v0) or (k1, v1).
inline int radix_sort_pairs(ow_ctx* ctx, uint32_t* k0, int32_t* v0, uint32_t* k1, int32_t* v1, int64_t n,
                            int key_bits, uint32_t** rk, int32_t** rv, cudaStream_t s) {
  *rk = k0;
  *rv = v0;
  if (n <= 1 || key_bits <= 0) return OW_OK;
  int64_t tiles = (n + RS_TILE - 1) / RS_TILE;
  void* hp;
  OW_TRY(ow_slot(ctx, SLOT_RADIX_HIST, sizeof(int32_t) * RS_DIGITS * (size_t)tiles, s, &hp));
  int32_t* hist = (int32_t*)hp;
  uint32_t *ki = k0, *ko = k1;
  int32_t *vi = v0, *vo = v1;
  for (int shift = 0; shift < key_bits; shift += RS_BITS) {
    k_radix_hist<<<(unsigned)tiles, RS_THREADS, 0, s>>>(ki, n, shift, tiles, hist);
    OW_LAUNCHED(ctx);
    OW_CHECK_LAUNCH();
    OW_TRY(scan(ctx, LoadArr<int32_t>{hist}, StoreExcl<int32_t>{hist}, RS_DIGITS * tiles, nullptr, s));
    k_radix_scatter<<<(unsigned)tiles, RS_THREADS, 0, s>>>(ki, vi, n, shift, tiles, hist, ko, vo);
    OW_LAUNCHED(ctx);
    OW_CHECK_LAUNCH();
    uint32_t* tk = ki; ki = ko; ko = tk;
    int32_t* tv = vi; vi = vo; vo = tv;
  }
  *rk = ki;
  *rv = vi;
  return OW_OK;
}

}  // namespace ow
