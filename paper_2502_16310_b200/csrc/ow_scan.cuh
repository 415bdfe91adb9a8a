// Single-pass exclusive scan with decoupled look-back, and a stable LSD radix
// sort of (u32 key, i32 value) pairs built on it.  Both are generic over
// functors so compaction / ranking / CSR offsets fuse into the scan pass.
#pragma once

#include "ow_common.cuh"

namespace ow {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;
constexpr int64_t SCAN_MAX_CHUNKS = 8 * OW_SMS;  // one wave of 256-thread CTAs
// Status words carry an epoch so the array never needs clearing between
// scans: [63:62] flag (1 aggregate, 2 inclusive prefix), [61:46] epoch,
// [45:0] value (sums < 2^46).  Tiles are blockIdx order: CTAs dispatch in
// index order, so every predecessor a tile waits on is already running.
constexpr unsigned long long ST_AGG = 1ull << 62;
constexpr unsigned long long ST_INC = 2ull << 62;
constexpr unsigned long long ST_VAL = (1ull << 46) - 1;
constexpr int ST_EPOCH_SHIFT = 46;
constexpr unsigned long long GRAPH_SITES = 64;  // scans per captured pass (ow_graph.cu: epoch = base * 64 + site)

__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Load: int64_t operator()(int64_t i) const      (non-negative values; may be
//       called twice per index, so it must be free of non-idempotent effects)
// Store: void operator()(int64_t i, int64_t exclusive_prefix, int64_t value) const
//
// Decoupled look-back by one warp (all lanes call it; agg is warp-uniform):
// publish this tile's aggregate, then inspect 128 predecessors per step (lane
// k, window j reads tile p - k - 32 j) until an inclusive prefix appears;
// publish the inclusive prefix and return the exclusive one.
__device__ __forceinline__ int64_t lookback(unsigned long long* status, int64_t tile, int64_t agg,
                                            unsigned long long epoch, int lane) {
  const unsigned long long tag = epoch << ST_EPOCH_SHIFT;
  int64_t prefix = 0;
  if (tile == 0) {
    if (lane == 0) st_status(&status[0], ST_INC | tag | (unsigned long long)agg);
    return 0;
  }
  if (lane == 0) st_status(&status[tile], ST_AGG | tag | (unsigned long long)agg);
  int64_t p = tile - 1;  // newest predecessor of the current window
  while (true) {
    unsigned long long st[4];
    bool ready = true;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t q = p - lane - 32 * j;
      st[j] = q >= 0 ? ld_status(&status[q]) : 0ull;
      ready &= q < 0 || ((st[j] & ~(3ull << 62)) >> ST_EPOCH_SHIFT) == epoch;
    }
    if (!__all_sync(0xffffffffu, ready)) {  // some predecessor not yet published
      __nanosleep(64);
      continue;
    }
    int jstop = 4, lstop = 31;
#pragma unroll
    for (int j = 3; j >= 0; --j) {
      const unsigned im = __ballot_sync(0xffffffffu, p - lane - 32 * j >= 0 && (st[j] >> 62) == 2);
      if (im) jstop = j, lstop = __ffs(im) - 1;
    }
    int64_t val = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (p - lane - 32 * j >= 0 && (j < jstop || (j == jstop && lane <= lstop))) val += (int64_t)(st[j] & ST_VAL);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    prefix += val;
    if (jstop < 4 || p - 127 < 0) break;
    p -= 128;
  }
  if (lane == 0) st_status(&status[tile], ST_INC | tag | (unsigned long long)(prefix + agg));
  return prefix;
}

// Chunked reduce-then-scan: each CTA takes a contiguous chunk of whole tiles
// (chunks in ticket order) and each of its warps a contiguous slice of the
// chunk.  Pass 1 sums the slices with coalesced loads (SCAN_ITEMS in flight
// per thread); the chunk aggregate is published and one warp looks back over
// 128 predecessors per step; pass 2 rescans every slice independently (warp
// scans only, no CTA barrier; the re-read hits L2) and stores.  One tile per
// CTA would make the look-back chain grow with n / SCAN_TILE and dominate:
// when tiles are cheap every tile looks back at once.
template <class Load, class Store, int ITEMS = SCAN_ITEMS>
__global__ void __launch_bounds__(SCAN_THREADS)
k_scan(Load load, Store store, int64_t n, int64_t n_chunks, int64_t chunk, unsigned long long* status,
       int64_t* total_out, unsigned long long epoch, const unsigned long long* d_epoch_base) {
  constexpr int SCAN_ITEMS = ITEMS;  // (shadows the default: small scans take 2 per thread)
  ow_pdl_wait();
  if (d_epoch_base) epoch += *d_epoch_base * GRAPH_SITES;  // inside a CUDA graph (ow_graph.cu)
  constexpr int W = SCAN_THREADS / 32;
  __shared__ int64_t s_warp[W];
  const int64_t tile = blockIdx.x;  // chunk index (CTAs dispatch in index order)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wch = chunk / W;  // slice length (a multiple of 32 * SCAN_ITEMS)
  const int64_t w0 = min(n, tile * chunk + warp * wch), w1 = min(n, w0 + wch);
  const bool one = w1 - w0 <= 32 * SCAN_ITEMS;  // single-step slice: keep the values
  int64_t v[SCAN_ITEMS];
  int64_t sum = 0;
  if (one) {
    const int64_t base = w0 + lane * SCAN_ITEMS;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) v[k] = base + k < w1 ? load(base + k) : 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) sum += v[k];
  } else {
    for (int64_t i0 = w0 + lane; i0 < w1; i0 += 32 * SCAN_ITEMS) {
#pragma unroll
      for (int k = 0; k < SCAN_ITEMS; ++k) v[k] = i0 + k * 32 < w1 ? load(i0 + k * 32) : 0;
#pragma unroll
      for (int k = 0; k < SCAN_ITEMS; ++k) sum += v[k];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) s_warp[warp] = sum;
  __syncthreads();
  if (warp == 0) {
    int64_t x = lane < W ? s_warp[lane] : 0;  // exclusive scan of the slice sums
#pragma unroll
    for (int o = 1; o < W; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const int64_t agg = __shfl_sync(0xffffffffu, x, W - 1);
    const int64_t wex = x - (lane < W ? s_warp[lane] : 0);
    const int64_t prefix = lookback(status, tile, agg, epoch, lane);
    if (lane < W) s_warp[lane] = prefix + wex;  // start of every slice
    if (lane == 0 && tile == n_chunks - 1 && total_out) *total_out = prefix + agg;
  }
  __syncthreads();
  int64_t run0 = s_warp[warp];
  for (int64_t t0 = w0; t0 < w1; t0 += 32 * SCAN_ITEMS) {
    const int64_t base = t0 + lane * SCAN_ITEMS;
    if (!one) {
#pragma unroll
      for (int k = 0; k < SCAN_ITEMS; ++k) v[k] = base + k < w1 ? load(base + k) : 0;
    }
    int64_t ts = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) ts += v[k];
    int64_t x = ts;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    int64_t run = run0 + x - ts;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
      if (base + k < w1) store(base + k, run, v[k]);
      run += v[k];
    }
    run0 += __shfl_sync(0xffffffffu, x, 31);
  }
}

// status words for `tiles` tiles (+ the ticket counters) and this scan's epoch
// (inside a graph capture: the graph's own status array and the scan's site;
// the kernel adds the device epoch base, see ow_graph.cu)
inline int scan_status(ow_ctx* ctx, int64_t tiles, cudaStream_t s, unsigned long long** status,
                       unsigned long long* epoch) {
  if (ctx->capturing) {
    if (8 * (size_t)(tiles + 1) > ctx->slot_bytes[SLOT_SCAN_STATUS_G] || ctx->graph_site + 1 >= GRAPH_SITES) {
      ctx->capture_failed = true;
      ow_set_error("graph capture: scan status array too small or too many scans");
      return OW_ERR_INTERNAL;
    }
    *epoch = (unsigned long long)(++ctx->graph_site);
    *status = (unsigned long long*)ctx->slot_ptr[SLOT_SCAN_STATUS_G] + 1;
    return OW_OK;
  }
  void* old = ctx->slot_ptr[SLOT_SCAN_STATUS];
  const size_t old_bytes = ctx->slot_bytes[SLOT_SCAN_STATUS];
  void* p;
  OW_TRY(ow_slot(ctx, SLOT_SCAN_STATUS, 8 * (size_t)(tiles + 1), s, &p));
  if (p != old || ctx->slot_bytes[SLOT_SCAN_STATUS] != old_bytes || ctx->scan_epoch >= 65535) {
    // fresh (or wrapped) status array: clear once, epochs restart at 1
    OW_CUDA(cudaMemsetAsync(p, 0, ctx->slot_bytes[SLOT_SCAN_STATUS], s));
    ctx->scan_epoch = 0;
  }
  *epoch = (unsigned long long)(++ctx->scan_epoch);
  *status = (unsigned long long*)p + 1;  // (word 0 spare)
  return OW_OK;
}

// Exclusive scan of load(0..n-1); *d_total (device) receives the sum.
template <class Load, class Store>
int scan(ow_ctx* ctx, Load load, Store store, int64_t n, int64_t* d_total, cudaStream_t s) {
  if (n <= 0) {
    if (d_total) OW_CUDA(cudaMemsetAsync(d_total, 0, sizeof(int64_t), s));
    return OW_OK;
  }
  // chunks of whole tiles, at most SCAN_MAX_CHUNKS of them (tiles of 2 elements
  // per thread below 1 M elements: 4x the CTAs in flight for small scans)
  const bool small = n <= (int64_t(1) << 20);
  const int64_t tile = (int64_t)SCAN_THREADS * (small ? 2 : SCAN_ITEMS);
  const int64_t tiles = (n + tile - 1) / tile;
  const int64_t per = (tiles + SCAN_MAX_CHUNKS - 1) / SCAN_MAX_CHUNKS;
  const int64_t chunk = per * tile;
  const int64_t n_chunks = (n + chunk - 1) / chunk;
  unsigned long long* status;
  unsigned long long epoch;
  OW_TRY(scan_status(ctx, n_chunks, s, &status, &epoch));
  const unsigned long long* base = (const unsigned long long*)(ctx->capturing ? ctx->d_graph_epoch : nullptr);
  if (small)
    ow_launch(k_scan<Load, Store, 2>, (unsigned)n_chunks, SCAN_THREADS, 0, s, load, store, n, n_chunks, chunk, status,
              d_total, epoch, base);
  else
    ow_launch(k_scan<Load, Store, SCAN_ITEMS>, (unsigned)n_chunks, SCAN_THREADS, 0, s, load, store, n, n_chunks, chunk,
              status, d_total, epoch, base);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

// ---- 0/1 scans (compactions) -----------------------------------------------
// Load returns 0 or 1.  One tile of C01_TILE elements per CTA, element i =
// base + k * 256 + threadIdx.x (coalesced), all C01_ITEMS predicates in flight
// per thread; ranks come from ballots, so values never leave registers.
constexpr int C01_ITEMS = 16;
constexpr int C01_TILE = SCAN_THREADS * C01_ITEMS;
// small compactions (the level loop's leaf / split / violator lists: up to a
// few 100 k elements) use 1 024-element tiles instead: 4x the CTAs in flight
// for the same elements, so the dependent loads of the predicates overlap
constexpr int C01_ITEMS_SMALL = 4;
constexpr int64_t C01_SMALL_MAX = int64_t(1) << 20;

template <class Load, class Store, int ITEMS = C01_ITEMS>
__global__ void __launch_bounds__(SCAN_THREADS, 6)
k_scan01(Load load, Store store, int64_t n, const int64_t* d_n, unsigned long long* status, int64_t* total_out,
         unsigned long long epoch, const unsigned long long* d_epoch_base) {
  ow_pdl_wait();
  if (d_epoch_base) epoch += *d_epoch_base * GRAPH_SITES;  // inside a CUDA graph (ow_graph.cu)
  constexpr int W = SCAN_THREADS / 32;
  constexpr int C01_TILE = SCAN_THREADS * ITEMS;
  constexpr int C01_ITEMS = ITEMS;
  static_assert(C01_ITEMS * W == 128 || C01_ITEMS * W == 32, "warp 0 holds 4 or 1 counts per lane");
  __shared__ int s_cnt[C01_ITEMS * W];  // per (item k, warp) in element order -> exclusive ranks
  __shared__ int64_t s_pre;
  const int64_t tile = blockIdx.x;
  if (d_n) {  // live length on the device: tiles past it do nothing
    const int64_t dn = *d_n;
    n = dn < n ? dn : n;
    if (tile > 0 && tile * C01_TILE >= n) return;
  }
  const int64_t last = n > 0 ? (n - 1) / C01_TILE : 0;  // writes the total
  const int64_t base = tile * C01_TILE + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // only the ballot masks are kept (few registers: many CTAs per SM hide the latency)
  bool v[C01_ITEMS];
#pragma unroll
  for (int k = 0; k < C01_ITEMS; ++k) v[k] = base + k * SCAN_THREADS < n && load(base + k * SCAN_THREADS) != 0;
  unsigned m[C01_ITEMS];
  int c = 0;
#pragma unroll
  for (int k = 0; k < C01_ITEMS; ++k) {
    m[k] = __ballot_sync(0xffffffffu, v[k]);
    if (lane == k) c = __popc(m[k]);
  }
  if (lane < C01_ITEMS) s_cnt[lane * W + warp] = c;
  __syncthreads();
  if (warp == 0) {
    int x;
    if constexpr (C01_ITEMS * W == 128) {
      const int a0 = s_cnt[4 * lane], a1 = s_cnt[4 * lane + 1], a2 = s_cnt[4 * lane + 2], a3 = s_cnt[4 * lane + 3];
      const int s4 = a0 + a1 + a2 + a3;
      x = s4;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const int ex = x - s4;
      s_cnt[4 * lane] = ex;
      s_cnt[4 * lane + 1] = ex + a0;
      s_cnt[4 * lane + 2] = ex + a0 + a1;
      s_cnt[4 * lane + 3] = ex + a0 + a1 + a2;
    } else {
      const int a0 = s_cnt[lane];
      x = a0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      s_cnt[lane] = x - a0;
    }
    const int64_t agg = __shfl_sync(0xffffffffu, x, 31);
    const int64_t prefix = lookback(status, tile, agg, epoch, lane);
    if (lane == 0) {
      s_pre = prefix;
      if (tile == last && total_out) *total_out = prefix + agg;
    }
  }
  __syncthreads();
  const int64_t pre = s_pre;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int k = 0; k < C01_ITEMS; ++k) {
    const int64_t i = base + k * SCAN_THREADS;
    if (i < n) store(i, pre + s_cnt[k * W + warp] + __popc(m[k] & lt), (int64_t)((m[k] >> lane) & 1u));
  }
}

// d_n (optional): the live length is min(n, *d_n), read on the device.
template <class Load, class Store>
int scan01(ow_ctx* ctx, Load load, Store store, int64_t n, int64_t* d_total, cudaStream_t s,
           const int64_t* d_n = nullptr) {
  if (n <= 0) {
    if (d_total) OW_CUDA(cudaMemsetAsync(d_total, 0, sizeof(int64_t), s));
    return OW_OK;
  }
  const bool small = n <= C01_SMALL_MAX;
  const int64_t tile = (int64_t)SCAN_THREADS * (small ? C01_ITEMS_SMALL : C01_ITEMS);
  const int64_t tiles = (n + tile - 1) / tile;
  unsigned long long* status;
  unsigned long long epoch;
  OW_TRY(scan_status(ctx, tiles, s, &status, &epoch));
  const unsigned long long* base = (const unsigned long long*)(ctx->capturing ? ctx->d_graph_epoch : nullptr);
  if (small)
    ow_launch(k_scan01<Load, Store, C01_ITEMS_SMALL>, (unsigned)tiles, SCAN_THREADS, 0, s, load, store, n, d_n, status,
              d_total, epoch, base);
  else
    ow_launch(k_scan01<Load, Store, C01_ITEMS>, (unsigned)tiles, SCAN_THREADS, 0, s, load, store, n, d_n, status,
              d_total, epoch, base);
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
// BITS-bit digits (8..10): keys of up to 10 bits sort in one pass, up to 20 in
// two (bin ids of every grid here).  A tile is RS_THREADS x ITEMS items; ITEMS
// (1..16) is chosen per sort so the grid covers every SM at least twice
// (C2's 25 k entries: 97 tiles of 256 instead of 7 of 4 096).
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;

template <int BITS, int ITEMS>
__global__ void __launch_bounds__(RS_THREADS)
k_radix_hist(const uint32_t* keys, int64_t n, int shift, int64_t n_tiles, int32_t* hist, const int64_t* d_n) {
  ow_pdl_wait();
  if (d_n && *d_n < n) n = *d_n;  // live length on the device (n: the buffers' bound)
  constexpr int DIG = 1 << BITS, TILE = RS_THREADS * ITEMS;
  __shared__ int h[DIG];
  for (int d = threadIdx.x; d < DIG; d += RS_THREADS) h[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * TILE;
#pragma unroll 4
  for (int k = 0; k < ITEMS; ++k) {
    int64_t i = base + (int64_t)k * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & (DIG - 1)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < DIG; d += RS_THREADS) hist[(int64_t)d * n_tiles + blockIdx.x] = h[d];
}

template <int BITS, int ITEMS>
__global__ void __launch_bounds__(RS_THREADS)
k_radix_scatter(const uint32_t* keys, const int32_t* vals, int64_t n, int shift, int64_t n_tiles,
                const int32_t* hist_excl, uint32_t* keys_out, int32_t* vals_out, const int64_t* d_n) {
  ow_pdl_wait();
  if (d_n && *d_n < n) n = *d_n;
  constexpr int DIG = 1 << BITS, TILE = RS_THREADS * ITEMS, WARP_ITEMS = TILE / RS_WARPS;
  __shared__ int cnt[RS_WARPS][DIG];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = lane; d < DIG; d += 32) cnt[warp][d] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * TILE + (int64_t)warp * WARP_ITEMS;
  uint32_t kk[ITEMS];
  int32_t vv[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    int64_t i = base + r * 32 + lane;
    bool ok = i < n;
    kk[r] = ok ? keys[i] : 0u;
    vv[r] = ok ? vals[i] : 0;
    int d = ok ? (int)((kk[r] >> shift) & (DIG - 1)) : DIG;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    if (ok && lane == __ffs(peers) - 1) cnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < DIG; d += RS_THREADS) {
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
  for (int r = 0; r < ITEMS; ++r) {
    int64_t i = base + r * 32 + lane;
    bool ok = i < n;
    int d = ok ? (int)((kk[r] >> shift) & (DIG - 1)) : DIG;
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

template <int BITS, int ITEMS>
inline int radix_pass(ow_ctx* ctx, const uint32_t* ki, const int32_t* vi, uint32_t* ko, int32_t* vo, int64_t n,
                      int shift, int64_t tiles, int32_t* hist, cudaStream_t s, const int64_t* d_n) {
  ow_launch(k_radix_hist<BITS, ITEMS>, (unsigned)tiles, RS_THREADS, 0, s, ki, n, shift, tiles, hist, d_n);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  OW_TRY(scan(ctx, LoadArr<int32_t>{hist}, StoreExcl<int32_t>{hist}, (int64_t)(1 << BITS) * tiles, nullptr, s));
  ow_launch(k_radix_scatter<BITS, ITEMS>, (unsigned)tiles, RS_THREADS, 0, s, ki, vi, n, shift, tiles, hist, ko, vo,
            d_n);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

template <int BITS>
inline int radix_pass_items(ow_ctx* ctx, int items, const uint32_t* ki, const int32_t* vi, uint32_t* ko, int32_t* vo,
                            int64_t n, int shift, int64_t tiles, int32_t* hist, cudaStream_t s,
                            const int64_t* d_n) {
  switch (items) {
    case 1: return radix_pass<BITS, 1>(ctx, ki, vi, ko, vo, n, shift, tiles, hist, s, d_n);
    case 2: return radix_pass<BITS, 2>(ctx, ki, vi, ko, vo, n, shift, tiles, hist, s, d_n);
    case 4: return radix_pass<BITS, 4>(ctx, ki, vi, ko, vo, n, shift, tiles, hist, s, d_n);
    case 8: return radix_pass<BITS, 8>(ctx, ki, vi, ko, vo, n, shift, tiles, hist, s, d_n);
    default: return radix_pass<BITS, 16>(ctx, ki, vi, ko, vo, n, shift, tiles, hist, s, d_n);
  }
}

// digit passes of a key_bits-bit sort (radix_sort_pairs)
inline int radix_passes(int key_bits) { return key_bits <= 0 ? 0 : (key_bits + 9) / 10; }

// Sort n pairs by the low `key_bits` bits of key, stably.  Input in (k0, v0);
// the sorted result pointer pair is returned through (*rk, *rv), which is
// either (k0, v0) or (k1, v1).  d_n (optional): the live length min(n, *d_n)
// is read on the device (n then only bounds the buffers and sizes the grid).
inline int radix_sort_pairs(ow_ctx* ctx, uint32_t* k0, int32_t* v0, uint32_t* k1, int32_t* v1, int64_t n,
                            int key_bits, uint32_t** rk, int32_t** rv, cudaStream_t s, const int64_t* d_n = nullptr) {
  *rk = k0;
  *rv = v0;
  if ((n <= 1 && !d_n) || n <= 0 || key_bits <= 0) return OW_OK;
  // fewest passes of 8..10-bit digits
  const int passes = radix_passes(key_bits);
  int bits = (key_bits + passes - 1) / passes;
  if (bits < 8) bits = 8;
  // items per thread: the largest power of two <= 16 that still gives >= 2
  // tiles per SM (1 for small sorts)
  int items = 16;
  while (items > 1 && (n + RS_THREADS * items - 1) / (RS_THREADS * items) < 2 * OW_SMS) items >>= 1;
  const int64_t tiles = (n + (int64_t)RS_THREADS * items - 1) / ((int64_t)RS_THREADS * items);
  void* hp;
  OW_TRY(ow_slot(ctx, SLOT_RADIX_HIST, sizeof(int32_t) * ((size_t)1 << bits) * (size_t)tiles, s, &hp));
  int32_t* hist = (int32_t*)hp;
  uint32_t *ki = k0, *ko = k1;
  int32_t *vi = v0, *vo = v1;
  for (int shift = 0; shift < key_bits; shift += bits) {
    if (bits == 8) OW_TRY(radix_pass_items<8>(ctx, items, ki, vi, ko, vo, n, shift, tiles, hist, s, d_n));
    else if (bits == 9) OW_TRY(radix_pass_items<9>(ctx, items, ki, vi, ko, vo, n, shift, tiles, hist, s, d_n));
    else OW_TRY(radix_pass_items<10>(ctx, items, ki, vi, ko, vo, n, shift, tiles, hist, s, d_n));
    uint32_t* tk = ki; ki = ko; ko = tk;
    int32_t* tv = vi; vi = vo; vo = tv;
  }
  *rk = ki;
  *rv = vi;
  return OW_OK;
}

}  // namespace ow
