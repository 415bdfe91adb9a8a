// fill_bins on sm_100a: face -> bin assignment by FP32 discretisation samples,
// CSR (ids, counts, offsets) grouped by bin, ascending face id per bin.
//
// Reference: octowall/binning.py:106-137 (discretize_face), 200-266 (fill_bins),
// 294-311 (_sample_segments_batch), 63-85 (linear_bin_indices).
//
// Pipeline (one launch each, 1 host sync between the phases):
//   count : thread per face walks its samples; faces whose +-1-padded vertex
//           AABB bin range is <= 64 bins keep a 64-bit occupancy mask in
//           registers (fast path); larger faces go to a CTA-per-face path with
//           a bitmap in global memory.  Distinct (bin, face) pairs -> counts[bin]
//           (atomics) and nb[face].
//   scan  : decoupled look-back over nb -> per-face pair offsets, entry total.
//   emit  : faces write their (bin, face) pairs in face order.
//   sort  : stable LSD radix sort by bin (8-bit digits) => ascending face per bin.
//   scan  : offsets = exclusive scan of counts.
#include "ow_scan.cuh"
#include <string.h>

namespace {

using ow::scan;

constexpr int FAST_MAX_SAMPLES = 4096;

struct Range {
  int lo[3], ext[3];
  int64_t vol;
};

template <int D>
__device__ __forceinline__ void load_face(const float* __restrict__ c, int64_t n, int64_t f, float v[3][3]) {
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int a = 0; a < D; ++a) v[j][a] = c[((int64_t)j * D + a) * n + f];
}

template <int D>
__device__ __forceinline__ Range face_range(const GridC& g, const float v[3][3], int pad) {
  Range r;
  r.vol = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float mn = v[0][a], mx = v[0][a];
#pragma unroll
    for (int j = 1; j < D; ++j) {
      mn = fminf(mn, v[j][a]);
      mx = fmaxf(mx, v[j][a]);
    }
    int lo = max(bin_axis(mn, g.min32[a], g.len32[a], g.B) - pad, 0);
    int hi = min(bin_axis(mx, g.min32[a], g.len32[a], g.B) + pad, g.B - 1);
    r.lo[a] = lo;
    r.ext[a] = hi - lo + 1;
    r.vol *= r.ext[a];
  }
  return r;
}

// number of segments ceil(|b-a| / h) with the reference's FP32 op order
template <int D>
__device__ __forceinline__ int64_t seg_count(const float* a, const float* b, float h, float* d) {
  float sq = 0.0f;
#pragma unroll
  for (int ax = 0; ax < D; ++ax) {
    d[ax] = FSUB(b[ax], a[ax]);
    sq = ax ? FADD(sq, FMUL(d[ax], d[ax])) : FMUL(d[ax], d[ax]);
  }
  return (int64_t)ceilf(FDIV(FSQRT(sq), h));
}

// p = a + (i / max(nseg,1)) * d, per component, no FMA
template <int D>
__device__ __forceinline__ void seg_point(const float* a, const float* d, int64_t i, float den, float* p) {
  float t = FDIV((float)i, den);
#pragma unroll
  for (int ax = 0; ax < D; ++ax) p[ax] = FADD(a[ax], FMUL(t, d[ax]));
}

// Visit every sample of face v (2D: v0->v1; 3D: base v0->v1, fan to v2),
// restricted to base indices [i0, i_end) stepping by `stride` (CTA sharing).
// visit(p) returns false to abort.
template <int D, class Visit>
__device__ __forceinline__ void walk_face(const float v[3][3], float h, int64_t i0, int64_t stride, Visit& visit) {
  float d1[3];
  int64_t n1 = seg_count<D>(v[0], v[1], h, d1);
  float den1 = (float)(n1 > 0 ? n1 : 1);
  for (int64_t i = i0; i <= n1; i += stride) {
    float p[3];
    seg_point<D>(v[0], d1, i, den1, p);
    if (D == 2) {
      if (!visit(p)) return;
      continue;
    }
    float d2[3];
    int64_t n2 = seg_count<D>(p, v[2], h, d2);
    float den2 = (float)(n2 > 0 ? n2 : 1);
    for (int64_t k = 0; k <= n2; ++k) {
      float q[3];
      seg_point<D>(p, d2, k, den2, q);
      if (!visit(q)) return;
    }
  }
}

template <int D>
__device__ __forceinline__ int64_t estimate_samples(const float v[3][3], float h) {
  float d[3];
  int64_t n1 = seg_count<D>(v[0], v[1], h, d);
  if (D == 2) return n1 + 1;
  int64_t a = seg_count<D>(v[0], v[2], h, d), b = seg_count<D>(v[1], v[2], h, d);
  return (n1 + 1) * (max(a, b) + 2);
}

template <int D>
struct MaskVisit {
  const GridC* g;
  Range r;
  unsigned long long mask;
  bool escaped, outside;
  __device__ bool operator()(const float* p) {
    if (outside_domain(*g, p)) {
      outside = true;
      return false;
    }
    int loc = 0, mul = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      int b = bin_axis(p[a], g->min32[a], g->len32[a], g->B) - r.lo[a];
      if (b < 0 || b >= r.ext[a]) {
        escaped = true;
        return false;
      }
      loc += b * mul;
      mul *= r.ext[a];
    }
    mask |= 1ull << loc;
    return true;
  }
};

template <int D>
__device__ __forceinline__ int64_t local_to_bin(const GridC& g, const Range& r, int loc) {
  int64_t lin = 0, mul = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    int b = loc % r.ext[a];
    loc /= r.ext[a];
    lin += (int64_t)(r.lo[a] + b) * mul;
    mul *= g.B;
  }
  return lin;
}

// small: [0] slow count, [1] first outside face (u64 min), [2] escape flag,
// [3] too-many-samples face
// (bin, face) pairs of one face by its samples (MaskVisit walk); faces whose
// padded range or sample count is too large go to the slow list
template <int D>
__device__ __forceinline__ void count_walk(const GridC& g, const float v[3][3], int64_t f, float h,
                                           unsigned long long* masks, int32_t* nb, int32_t* counts, int32_t* slow,
                                           int64_t* small) {
  Range r = face_range<D>(g, v, 1);
  bool go_slow = r.vol > 64 || estimate_samples<D>(v, h) > FAST_MAX_SAMPLES;
  if (!go_slow) {
    MaskVisit<D> mv{&g, r, 0ull, false, false};
    walk_face<D>(v, h, 0, 1, mv);
    if (mv.outside) {
      atomicMin((unsigned long long*)&small[1], (unsigned long long)f);
      masks[f] = 0;
      nb[f] = 0;
      return;
    }
    if (!mv.escaped) {
      masks[f] = mv.mask;
      nb[f] = __popcll(mv.mask);
      unsigned long long m = mv.mask;
      while (m) {
        int loc = __ffsll(m) - 1;
        m &= m - 1;
        atomicAdd(&counts[local_to_bin<D>(g, r, loc)], 1);
      }
      return;
    }
  }
  masks[f] = 0;
  nb[f] = 0;
  int idx = atomicAdd((unsigned long long*)&small[0], 1ull);
  slow[idx] = (int32_t)f;
}

// Pass 1 over all faces.  Single-bin faces (most faces of a fine mesh): every
// sample lies within 2^-16 max|x| of the vertex hull (a few roundings of hull
// coordinates), and bin_axis is monotone, so a hull widened by that much
// inside one bin and inside the domain puts every sample in that bin: no walk
// needed (then bin(min) = bin(max) = b and the padded range is [b - 1, b + 1]
// clipped).  The other faces are listed for k_count_walk, so the walks run on
// full warps instead of stalling warps of single-bin faces.
template <int D>
__global__ void __launch_bounds__(256)
k_count_fast(GridC g, const float* __restrict__ c, int64_t n, unsigned long long* masks, int32_t* nb,
             int32_t* counts, int32_t* mid, int64_t* small) {
  ow_pdl_wait();
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool one = true;
  int64_t lin = 0;
  if (f < n) {
    float v[3][3];
    load_face<D>(c, n, f, v);
    int loc = 0, mul = 1;
    int64_t lmul = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      float mn = v[0][a], mx = v[0][a];
#pragma unroll
      for (int j = 1; j < D; ++j) mn = fminf(mn, v[j][a]), mx = fmaxf(mx, v[j][a]);
      const float del = fmaxf(fabsf(mn), fabsf(mx)) * 0x1p-16f + 0x1p-100f;
      const float lo = FSUB(mn, del), hi = FADD(mx, del);
      const int b = bin_axis(lo, g.min32[a], g.len32[a], g.B);
      one &= b == bin_axis(hi, g.min32[a], g.len32[a], g.B) && (double)lo >= g.lo_tol[a] && (double)hi <= g.hi_tol[a];
      const int rlo = max(b - 1, 0), rhi = min(b + 1, g.B - 1);
      loc += (b - rlo) * mul;
      mul *= rhi - rlo + 1;
      lin += (int64_t)b * lmul;
      lmul *= g.B;
    }
    if (one) {
      masks[f] = 1ull << loc;
      nb[f] = 1;
    }
  }
  // warp-aggregated counts: consecutive faces of a fine mesh mostly share
  // their bin, so one atomic per distinct bin of the warp (north star:
  // "warp-aggregated atomic counts") instead of one per face
  {
    const bool add = f < n && one;
    const int64_t key = add ? lin : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int lane = threadIdx.x & 31;
    if (add && lane == __ffs(peers) - 1) atomicAdd(&counts[key], __popc(peers));
  }
  const bool walk = f < n && !one;
  const unsigned wm = __ballot_sync(0xffffffffu, walk);
  if (wm) {
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd((unsigned long long*)&small[6], (unsigned long long)__popc(wm));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (walk) mid[base + __popc(wm & lanemask_lt())] = (int32_t)f;
  }
}

// Pass 2: the listed faces, by their samples (count on the device)
template <int D>
__global__ void __launch_bounds__(256)
k_count_walk(GridC g, const float* __restrict__ c, int64_t n, float h, const int32_t* __restrict__ mid,
             unsigned long long* masks, int32_t* nb, int32_t* counts, int32_t* slow, int64_t* small) {
  ow_pdl_wait();
  const int64_t m = small[6];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = mid[i];
    float v[3][3];
    load_face<D>(c, n, f, v);
    count_walk<D>(g, v, f, h, masks, nb, counts, slow, small);
  }
}

struct BitVisitCtx {
  const GridC* g;
  Range r;
  unsigned* bits;
  bool outside, escaped;
};

template <int D>
struct BitVisit {
  BitVisitCtx* s;
  __device__ bool operator()(const float* p) {
    if (outside_domain(*s->g, p)) {
      s->outside = true;
      return false;
    }
    int64_t loc = 0, mul = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      int b = bin_axis(p[a], s->g->min32[a], s->g->len32[a], s->g->B) - s->r.lo[a];
      if (b < 0 || b >= s->r.ext[a]) {
        s->escaped = true;
        return false;
      }
      loc += b * mul;
      mul *= s->r.ext[a];
    }
    atomicOr(&s->bits[loc >> 5], 1u << (loc & 31));
    return true;
  }
};

// CTA per slow face: bitmap over the padded bin range in global memory.
template <int D>
__global__ void __launch_bounds__(256)
k_count_slow(GridC g, const float* __restrict__ c, int64_t n, float h, const int32_t* slow,
             const int64_t* bitoff, unsigned* bitmap, int32_t* nb, int32_t* counts, int64_t* small) {
  ow_pdl_wait();
  const int64_t f = slow[blockIdx.x];
  float v[3][3];
  load_face<D>(c, n, f, v);
  Range r = face_range<D>(g, v, 1);
  unsigned* bits = bitmap + bitoff[blockIdx.x];
  const int64_t words = (r.vol + 31) >> 5;
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) bits[w] = 0u;
  __syncthreads();
  BitVisitCtx st{&g, r, bits, false, false};
  BitVisit<D> bv{&st};
  walk_face<D>(v, h, threadIdx.x, blockDim.x, bv);
  if (st.outside) atomicMin((unsigned long long*)&small[1], (unsigned long long)f);
  if (st.escaped) atomicExch((unsigned long long*)&small[2], 1ull);
  __syncthreads();
  int local = 0;
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) {
    unsigned m = bits[w];
    local += __popc(m);
    while (m) {
      int b = __ffs(m) - 1;
      m &= m - 1;
      int64_t loc = (w << 5) + b;
      int64_t lin = 0, mul = 1, rem = loc;
      for (int a = 0; a < D; ++a) {
        lin += (int64_t)(r.lo[a] + rem % r.ext[a]) * mul;
        rem /= r.ext[a];
        mul *= g.B;
      }
      atomicAdd(&counts[lin], 1);
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  __shared__ int s_sum;
  if (threadIdx.x == 0) s_sum = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_sum, local);
  __syncthreads();
  if (threadIdx.x == 0) nb[f] = s_sum;
}

template <int D>
struct SlowVolLoad {
  GridC g;
  const float* c;
  int64_t n;
  const int32_t* slow;
  __device__ int64_t operator()(int64_t i) const {
    float v[3][3];
    load_face<D>(c, n, slow[i], v);
    Range r = face_range<D>(g, v, 1);
    return (r.vol + 31) >> 5;
  }
};

template <int D>
__global__ void k_emit_fast(GridC g, const float* __restrict__ c, int64_t n, const unsigned long long* masks,
                            const int32_t* foff, uint32_t* keys, int32_t* vals, int64_t cap) {
  ow_pdl_wait();
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  unsigned long long m = masks[f];
  if (!m) return;
  float v[3][3];
  load_face<D>(c, n, f, v);
  Range r = face_range<D>(g, v, 1);
  int64_t pos = foff[f];
  // cap: the pair buffers' length (device-sized pass: the entry count is only
  // checked on the host after the pass; entries past the buffers are dropped)
  if (pos + __popcll(m) > cap) return;
  while (m) {
    int loc = __ffsll(m) - 1;
    m &= m - 1;
    keys[pos] = (uint32_t)local_to_bin<D>(g, r, loc);
    vals[pos] = (int32_t)f;
    ++pos;
  }
}

// one warp per slow face, words in order with a warp prefix of popcounts
template <int D>
__global__ void k_emit_slow(GridC g, const float* __restrict__ c, int64_t n, const int32_t* slow,
                            const int64_t* bitoff, const unsigned* bitmap, const int32_t* foff, uint32_t* keys,
                            int32_t* vals) {
  ow_pdl_wait();
  const int64_t f = slow[blockIdx.x];
  const int lane = threadIdx.x;
  float v[3][3];
  load_face<D>(c, n, f, v);
  Range r = face_range<D>(g, v, 1);
  const unsigned* bits = bitmap + bitoff[blockIdx.x];
  const int64_t words = (r.vol + 31) >> 5;
  int64_t pos = foff[f];
  for (int64_t w0 = 0; w0 < words; w0 += 32) {
    int64_t w = w0 + lane;
    unsigned m = (w < words) ? bits[w] : 0u;
    int cnt = __popc(m), incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int64_t p = pos + incl - cnt;
    while (m) {
      int b = __ffs(m) - 1;
      m &= m - 1;
      int64_t loc = (w << 5) + b, lin = 0, mul = 1, rem = loc;
      for (int a = 0; a < D; ++a) {
        lin += (int64_t)(r.lo[a] + rem % r.ext[a]) * mul;
        rem /= r.ext[a];
        mul *= g.B;
      }
      keys[p] = (uint32_t)lin;
      vals[p] = (int32_t)f;
      ++p;
    }
    pos += __shfl_sync(0xffffffffu, incl, 31);
  }
}

__global__ void k_small_init(int64_t* small) {
  ow_pdl_wait();
  if (threadIdx.x < 8) small[threadIdx.x] = (threadIdx.x == 1 || threadIdx.x == 3) ? -1 : 0;
}

// the same and the bin counts cleared, one launch (device-sized fill_bins)
__global__ void k_bins_init(int64_t* small, int32_t* counts, int64_t n_bins) {
  ow_pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x < 8) small[threadIdx.x] = (threadIdx.x == 1 || threadIdx.x == 3) ? -1 : 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_bins; i += (int64_t)gridDim.x * blockDim.x)
    counts[i] = 0;
}

template <int D>
int fill_count(ow_ctx* ctx, const GridC& g, const float* c, int64_t n, float h, int32_t* counts, int64_t n_bins,
               int64_t* out_entries, int64_t* out_outside, cudaStream_t s) {
  void *pm, *pnb, *pfo, *psl;
  OW_TRY(ow_slot(ctx, SLOT_BIN_MASK, 8 * (size_t)n, s, &pm));
  OW_TRY(ow_slot(ctx, SLOT_BIN_NB, 4 * (size_t)n, s, &pnb));
  OW_TRY(ow_slot(ctx, SLOT_BIN_FOFF, 4 * (size_t)n, s, &pfo));
  OW_TRY(ow_slot(ctx, SLOT_BIN_SLOW, 4 * (size_t)n, s, &psl));
  int64_t* small = ctx->d_small;
  OW_TRY(ow_fill_async(ctx, counts, 0, 4 * (size_t)n_bins, s));
  ow_launch(k_small_init, 1, 32, 0, s, small);  // [1], [3] = -1 (none), rest 0
  OW_LAUNCHED(ctx);
  void* pmid;
  OW_TRY(ow_slot(ctx, SLOT_BIN_MID, 4 * (size_t)n, s, &pmid));
  ow_launch(k_count_fast<D>, ow_blocks(n, 256), 256, 0, s, g, c, n, (unsigned long long*)pm, (int32_t*)pnb, counts,
                                                   (int32_t*)pmid, small);
  ow_launch(k_count_walk<D>, ow_blocks(n, 256, 8 * OW_SMS), 256, 0, s, g, c, n, h, (const int32_t*)pmid,
                                                                (unsigned long long*)pm, (int32_t*)pnb, counts,
                                                                (int32_t*)psl, small);
  ctx->launches += 2;
  OW_CHECK_LAUNCH();
  // face offsets over the fast path's counts, read back with the slow-face
  // count in one round trip; faces with too many bins for the bitmask path
  // (rare: large faces) add a second pass and a re-scan
  OW_TRY(scan(ctx, ow::LoadArr<int32_t>{(const int32_t*)pnb}, ow::StoreExcl<int32_t>{(int32_t*)pfo}, n, small + 5, s));
  OW_PROF_END(ctx, PROF_BINS, s);  // (device work only: the readback below is host latency)
  int64_t r[6];
  if (ctx->faces_pending) {
    // fused pass: the face summary travels with this readback and is checked
    // before anything depends on valid faces (the slow path sizes bitmaps by
    // face extent); the count kernels above do bounded work on any input
    int64_t hf[6];
    OW_CUDA(cudaMemcpyAsync(ctx->h_pinned + 64, ctx->faces_pending, 6 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    OW_TRY(ow_readback(ctx, small, 6, r, s));
    memcpy(hf, ctx->h_pinned + 64, sizeof(hf));
    OW_TRY(ow_faces_settle(ctx, hf, s));
  } else {
    OW_TRY(ow_readback(ctx, small, 6, r, s));
  }
  int64_t n_slow = r[0];
  ctx->bins_slow = n_slow;
  if (n_slow > 0) {
    int64_t hs[1];
    void* po;
    OW_TRY(ow_slot(ctx, SLOT_BIN_SLOWOFF, 8 * (size_t)n_slow, s, &po));
    OW_TRY(scan(ctx, SlowVolLoad<D>{g, c, n, (const int32_t*)psl}, ow::StoreExcl<int64_t>{(int64_t*)po}, n_slow,
                small + 4, s));
    OW_TRY(ow_readback(ctx, small + 4, 1, hs, s));
    void* pb;
    OW_TRY(ow_slot(ctx, SLOT_BIN_BITMAP, 4 * (size_t)(hs[0] + 1), s, &pb));
    OW_PROF_BEGIN(ctx, PROF_BINS, s);
    ow_launch(k_count_slow<D>, (unsigned)n_slow, 256, 0, s, g, c, n, h, (const int32_t*)psl, (const int64_t*)po,
                                                     (unsigned*)pb, (int32_t*)pnb, counts, small);
    OW_LAUNCHED(ctx);
    OW_CHECK_LAUNCH();
    OW_TRY(scan(ctx, ow::LoadArr<int32_t>{(const int32_t*)pnb}, ow::StoreExcl<int32_t>{(int32_t*)pfo}, n, small + 5,
                s));
    OW_PROF_END(ctx, PROF_BINS, s);
    OW_TRY(ow_readback(ctx, small, 6, r, s));
  }
  if (r[2]) {
    ow_set_error("fill_bins: a face sample escaped its padded bin range (internal)");
    return OW_ERR_INTERNAL;
  }
  *out_outside = r[1];
  *out_entries = r[5];
  return OW_OK;
}

template <int D>
int fill_emit(ow_ctx* ctx, const GridC& g, const float* c, int64_t n, int32_t* ids, const int32_t* counts,
              int32_t* offsets, int64_t n_bins, cudaStream_t s) {
  int64_t E = ctx->bins_entries;
  void *pk0, *pv0, *pk1, *pv1;
  OW_TRY(ow_slot(ctx, SLOT_PAIR_KEY0, 4 * (size_t)E, s, &pk0));
  OW_TRY(ow_slot(ctx, SLOT_PAIR_VAL0, 4 * (size_t)E, s, &pv0));
  OW_TRY(ow_slot(ctx, SLOT_PAIR_KEY1, 4 * (size_t)E, s, &pk1));
  OW_TRY(ow_slot(ctx, SLOT_PAIR_VAL1, 4 * (size_t)E, s, &pv1));
  int bits = 0;
  while ((int64_t(1) << bits) < n_bins) ++bits;
  // the sort's last pass writes the face ids straight into `ids` (no copy):
  // an odd number of digit passes ends in the second buffer, an even one
  // (including none) in the first
  const int passes = (E <= 1 || bits <= 0) ? 0 : ow::radix_passes(bits);
  if (passes & 1) pv1 = ids;
  else pv0 = ids;
  const int32_t* foff = (const int32_t*)ctx->slot_ptr[SLOT_BIN_FOFF];
  ow_launch(k_emit_fast<D>, ow_blocks(n, 256), 256, 0, s, g, c, n, (const unsigned long long*)ctx->slot_ptr[SLOT_BIN_MASK],
                                                  foff, (uint32_t*)pk0, (int32_t*)pv0, E);
  OW_LAUNCHED(ctx);
  if (ctx->bins_slow > 0) {
    ow_launch(k_emit_slow<D>, (unsigned)ctx->bins_slow, 32, 0, s, 
        g, c, n, (const int32_t*)ctx->slot_ptr[SLOT_BIN_SLOW], (const int64_t*)ctx->slot_ptr[SLOT_BIN_SLOWOFF],
        (const unsigned*)ctx->slot_ptr[SLOT_BIN_BITMAP], foff, (uint32_t*)pk0, (int32_t*)pv0);
    OW_LAUNCHED(ctx);
  }
  OW_CHECK_LAUNCH();
  uint32_t* rk;
  int32_t* rv;
  OW_TRY(ow::radix_sort_pairs(ctx, (uint32_t*)pk0, (int32_t*)pv0, (uint32_t*)pk1, (int32_t*)pv1, E, bits, &rk, &rv, s));
  if (E > 0 && rv != ids) OW_CUDA(cudaMemcpyAsync(ids, rv, 4 * (size_t)E, cudaMemcpyDeviceToDevice, s));
  OW_TRY(scan(ctx, ow::LoadArr<int32_t>{counts}, ow::StoreExcl<int32_t>{offsets}, n_bins, nullptr, s));
  return OW_OK;
}

// offsets of the device-sized fill_bins: when the entry count outgrew the
// pair buffers (e_cap) the bins are emptied instead (counts and offsets 0), so
// nothing downstream indexes entries that were never written; the host sees
// the count after the pass and re-runs it with room
struct GuardLoad {
  const int32_t* counts;
  const int64_t* d_e;
  int64_t cap;
  __device__ int64_t operator()(int64_t i) const { return *d_e <= cap ? (int64_t)counts[i] : 0; }
};
struct GuardStore {
  int32_t* offsets;
  int32_t* counts;
  const int64_t* d_e;
  int64_t cap;
  __device__ void operator()(int64_t i, int64_t e, int64_t) const {
    offsets[i] = (int32_t)e;
    if (*d_e > cap) counts[i] = 0;
  }
};

// Device-sized fill_bins (fused pass, ow_pipeline.cu): count, face offsets,
// emission and the stable sort with the entry count left on the device
// (small[5]); e_cap bounds the pair buffers and sizes the sort's grid.  The
// host checks small[0] (slow faces: this path does not bin them), small[1]
// (a sample outside the domain), small[2] and small[5] <= e_cap after the
// pass and re-runs it on the synchronous path when one fails.
template <int D>
int fill_dev(ow_ctx* ctx, const GridC& g, const float* c, int64_t n, float h, int32_t* counts, int32_t* ids,
             int32_t* offsets, int64_t n_bins, int64_t e_cap, cudaStream_t s, bool init) {
  void *pm, *pnb, *pfo, *psl, *pmid;
  OW_TRY(ow_slot(ctx, SLOT_BIN_MASK, 8 * (size_t)n, s, &pm));
  OW_TRY(ow_slot(ctx, SLOT_BIN_NB, 4 * (size_t)n, s, &pnb));
  OW_TRY(ow_slot(ctx, SLOT_BIN_FOFF, 4 * (size_t)n, s, &pfo));
  OW_TRY(ow_slot(ctx, SLOT_BIN_SLOW, 4 * (size_t)n, s, &psl));
  OW_TRY(ow_slot(ctx, SLOT_BIN_MID, 4 * (size_t)n, s, &pmid));
  int64_t* small = ctx->d_small;
  if (init) {  // (else the caller's first kernel cleared them: k_loop_init)
    ow_launch(k_bins_init, ow_blocks(n_bins, 256, 4 * OW_SMS), 256, 0, s, small, counts, n_bins);
    OW_LAUNCHED(ctx);
  }
  ow_launch(k_count_fast<D>, ow_blocks(n, 256), 256, 0, s, g, c, n, (unsigned long long*)pm, (int32_t*)pnb, counts,
            (int32_t*)pmid, small);
  ow_launch(k_count_walk<D>, ow_blocks(n, 256, 8 * OW_SMS), 256, 0, s, g, c, n, h, (const int32_t*)pmid,
            (unsigned long long*)pm, (int32_t*)pnb, counts, (int32_t*)psl, small);
  ctx->launches += 2;
  OW_CHECK_LAUNCH();
  OW_TRY(scan(ctx, ow::LoadArr<int32_t>{(const int32_t*)pnb}, ow::StoreExcl<int32_t>{(int32_t*)pfo}, n, small + 5, s));
  void *pk0, *pv0, *pk1, *pv1;
  OW_TRY(ow_slot(ctx, SLOT_PAIR_KEY0, 4 * (size_t)e_cap, s, &pk0));
  OW_TRY(ow_slot(ctx, SLOT_PAIR_VAL0, 4 * (size_t)e_cap, s, &pv0));
  OW_TRY(ow_slot(ctx, SLOT_PAIR_KEY1, 4 * (size_t)e_cap, s, &pk1));
  OW_TRY(ow_slot(ctx, SLOT_PAIR_VAL1, 4 * (size_t)e_cap, s, &pv1));
  int bits = 0;
  while ((int64_t(1) << bits) < n_bins) ++bits;
  const int passes = bits <= 0 ? 0 : ow::radix_passes(bits);
  if (passes & 1) pv1 = ids;
  else pv0 = ids;
  ow_launch(k_emit_fast<D>, ow_blocks(n, 256), 256, 0, s, g, c, n, (const unsigned long long*)pm,
            (const int32_t*)pfo, (uint32_t*)pk0, (int32_t*)pv0, e_cap);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  uint32_t* rk;
  int32_t* rv;
  OW_TRY(ow::radix_sort_pairs(ctx, (uint32_t*)pk0, (int32_t*)pv0, (uint32_t*)pk1, (int32_t*)pv1, e_cap, bits, &rk,
                              &rv, s, small + 5));
  if (rv != ids) {
    ow_set_error("fill_bins: sort ended outside the id buffer (internal)");
    return OW_ERR_INTERNAL;
  }
  OW_TRY(scan(ctx, GuardLoad{counts, small + 5, e_cap}, GuardStore{offsets, counts, small + 5, e_cap}, n_bins, nullptr,
              s));
  ctx->bins_faces = n;
  ctx->bins_entries = -1;  // (on the device)
  ctx->bins_slow = 0;
  ctx->bins_dim = D;
  ctx->bins_B = g.B;
  ctx->bins_h = h;
  ctx->bins_coords = c;
  return OW_OK;
}

}  // namespace

int ow_fill_bins_dev(ow_ctx* ctx, const ow_grid* grid, const float* d_coords, int64_t n_faces, float spacing,
                     int32_t* d_counts, int32_t* d_ids, int32_t* d_offsets, int64_t e_cap, cudaStream_t s, bool init) {
  GridC g = make_gridc(grid);
  int64_t n_bins = 1;
  for (int a = 0; a < grid->dim; ++a) n_bins *= grid->bins_per_axis;
  OW_PROF_BEGIN(ctx, PROF_BINS, s);
  const int st = grid->dim == 2 ? fill_dev<2>(ctx, g, d_coords, n_faces, spacing, d_counts, d_ids, d_offsets, n_bins,
                                              e_cap, s, init)
                                : fill_dev<3>(ctx, g, d_coords, n_faces, spacing, d_counts, d_ids, d_offsets, n_bins,
                                              e_cap, s, init);
  OW_PROF_END(ctx, PROF_BINS, s);
  return st;
}

extern "C" int ow_fill_bins_count(ow_ctx* ctx, const ow_grid* grid, const float* d_coords, int64_t n_faces,
                                  float spacing, int32_t* d_counts, int64_t* out_entries, int64_t* out_outside,
                                  void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!grid || (grid->dim != 2 && grid->dim != 3) || grid->bins_per_axis < 1) {
    ow_set_error("fill_bins: bad grid");
    return OW_ERR_INVALID;
  }
  if (!(spacing > 0.0f)) {
    ow_set_error("spacing must be positive, got %g", (double)spacing);
    return OW_ERR_INVALID;
  }
  if (n_faces <= 0) {
    ow_set_error("cannot bin empty geometry");
    return OW_ERR_INVALID;
  }
  GridC g = make_gridc(grid);
  int64_t n_bins = 1;
  for (int a = 0; a < grid->dim; ++a) n_bins *= grid->bins_per_axis;
  if (n_bins > (int64_t(1) << 31)) {
    ow_set_error("fill_bins: too many bins (%lld)", (long long)n_bins);
    return OW_ERR_INVALID;
  }
  OW_PROF_BEGIN(ctx, PROF_BINS, s);  // (ended inside fill_count before its readbacks)
  int st = grid->dim == 2 ? fill_count<2>(ctx, g, d_coords, n_faces, spacing, d_counts, n_bins, out_entries, out_outside, s)
                          : fill_count<3>(ctx, g, d_coords, n_faces, spacing, d_counts, n_bins, out_entries, out_outside, s);
  if (st != OW_OK) return st;
  ctx->bins_faces = n_faces;
  ctx->bins_entries = *out_entries;
  ctx->bins_dim = grid->dim;
  ctx->bins_B = grid->bins_per_axis;
  ctx->bins_h = spacing;
  ctx->bins_coords = d_coords;
  return OW_OK;
}

extern "C" int ow_fill_bins_emit(ow_ctx* ctx, const ow_grid* grid, int32_t* d_ids, const int32_t* d_counts,
                                 int32_t* d_offsets, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!grid || grid->dim != ctx->bins_dim || grid->bins_per_axis != ctx->bins_B || !ctx->bins_coords) {
    ow_set_error("ow_fill_bins_emit without a matching ow_fill_bins_count");
    return OW_ERR_INVALID;
  }
  GridC g = make_gridc(grid);
  int64_t n_bins = 1;
  for (int a = 0; a < grid->dim; ++a) n_bins *= grid->bins_per_axis;
  OW_PROF_BEGIN(ctx, PROF_BINS, s);
  int st = grid->dim == 2 ? fill_emit<2>(ctx, g, ctx->bins_coords, ctx->bins_faces, d_ids, d_counts, d_offsets, n_bins, s)
                          : fill_emit<3>(ctx, g, ctx->bins_coords, ctx->bins_faces, d_ids, d_counts, d_offsets, n_bins, s);
  OW_PROF_END(ctx, PROF_BINS, s);
  return st;
}
