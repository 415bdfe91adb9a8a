// Near-wall detection on sm_100a: face prep, block marking (naive / binned),
// cell-face links, and the pairwise predicate probe.
//
// Reference: octowall/nearwall.py:31-54 (cull reach, face boxes, box cull),
// 146-214 (sphere prefilter, _scan_block), 217-311 (mark_near_wall_naive /
// _binned), 522-594 (build_cell_face_links).
//
// One CTA per leaf block.  The CTA computes its 4^D cell centres (FP64 -> one
// FP32 rounding), their bins, and the block box; then, per distinct bin of its
// cells (or once over all faces for the naive strategy), stages the bin's
// faces that pass the reference's FP64 box cull into shared memory, and
// sweeps (cell, staged face) pairs: FP32 bounding-sphere prefilter, then the
// full 130-op predicate.  The first hit ends the block (a mark is an OR).
// A pair is evaluated iff the reference evaluates it, so marks are bit-exact
// even where the predicate is ill-conditioned.
#include "ow_predicate.cuh"
#include "ow_scan.cuh"
#include <string.h>

namespace {

using ow::scan;

constexpr int MARK_THREADS = 128;

constexpr int PREP_THREADS = 128;

// Per-face terms of marking: FP32 box, bounding sphere and predicate payload.
// Records are assembled in shared memory and leave as contiguous float4 runs
// (a thread's own 112-byte payload record would be a 16-byte scatter per lane).
template <int D>
__global__ void __launch_bounds__(PREP_THREADS) k_face_prep(const float* __restrict__ c, int64_t n, float d,
                                                            double reach, float4* box, float4* sph, float4* pay) {
  ow_pdl_wait();
  constexpr int PW = D == 3 ? PAY3 : PAY2;
  __shared__ float4 s_pay[PREP_THREADS * PW];
  __shared__ float4 s_box[PREP_THREADS * 2];
  const int64_t f0 = (int64_t)blockIdx.x * PREP_THREADS;
  const int64_t f = f0 + threadIdx.x;
  const int nv = (int)min((int64_t)PREP_THREADS, n - f0);
  if (f < n) {
    float lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) {
      float mn = c[(int64_t)a * n + f], mx = mn;
      for (int j = 1; j < D; ++j) {
        float x = c[((int64_t)j * D + a) * n + f];
        mn = fminf(mn, x);
        mx = fmaxf(mx, x);
      }
      lo[a] = mn;
      hi[a] = mx;
    }
    s_box[2 * threadIdx.x] = make_float4(lo[0], lo[1], lo[2], 0.0f);
    s_box[2 * threadIdx.x + 1] = make_float4(hi[0], hi[1], hi[2], 0.0f);
    // bounding sphere: centre f32(0.5 (lo+hi)), radius^2 f32((|0.5 (hi-lo)| + reach)^2)
    double ctr[3] = {0, 0, 0}, ss = 0.0;
    for (int a = 0; a < D; ++a) {
      double l = lo[a], h = hi[a];
      ctr[a] = DMUL(0.5, DADD(l, h));
      double hh = DMUL(0.5, DSUB(h, l));
      ss = a ? DADD(ss, DMUL(hh, hh)) : DMUL(hh, hh);
    }
    double r = DADD(__dsqrt_rn(ss), reach);
    sph[f] = make_float4(__double2float_rn(ctr[0]), __double2float_rn(ctr[1]), __double2float_rn(ctr[2]),
                         __double2float_rn(DMUL(r, r)));
    face_prep_one<D>(c, n, f, d, s_pay + threadIdx.x * PW);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv * PW; i += PREP_THREADS) pay[f0 * PW + i] = s_pay[i];
  for (int i = threadIdx.x; i < nv * 2; i += PREP_THREADS) box[f0 * 2 + i] = s_box[i];
}

int prepare_faces(ow_ctx* ctx, int dim, const float* c, int64_t n, int64_t key, float d, double reach,
                  cudaStream_t s) {
  const int pw = dim == 3 ? PAY3 : PAY2;
  void *pb, *ps, *pp;
  bool fresh = ctx->prep_key != key || key < 0 || ctx->prep_faces != n || ctx->prep_dim != dim;
  size_t need_pay = sizeof(float4) * pw * (size_t)n;
  if (ctx->slot_bytes[SLOT_FACE_PREP] < need_pay || ctx->slot_bytes[SLOT_FACE_BOX] < 32 * (size_t)n ||
      ctx->slot_bytes[SLOT_FACE_SPHERE] < 16 * (size_t)n)
    fresh = true;
  if (!fresh && ctx->prep_d == d && ctx->prep_reach == reach) return OW_OK;
  OW_TRY(ow_slot(ctx, SLOT_FACE_BOX, 32 * (size_t)n, s, &pb));
  OW_TRY(ow_slot(ctx, SLOT_FACE_SPHERE, 16 * (size_t)n, s, &ps));
  OW_TRY(ow_slot(ctx, SLOT_FACE_PREP, need_pay, s, &pp));
  if (dim == 3)
    ow_launch(k_face_prep<3>, ow_blocks(n, PREP_THREADS), PREP_THREADS, 0, s, c, n, d, reach, (float4*)pb, (float4*)ps,
                                                                        (float4*)pp);
  else
    ow_launch(k_face_prep<2>, ow_blocks(n, PREP_THREADS), PREP_THREADS, 0, s, c, n, d, reach, (float4*)pb, (float4*)ps,
                                                                        (float4*)pp);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  ctx->prep_key = key;
  ctx->prep_faces = n;
  ctx->prep_dim = dim;
  ctx->prep_d = d;
  ctx->prep_reach = reach;
  return OW_OK;
}

// FP64 block-box vs face-box distance cull (nearwall.py:48-54); the sum
// follows numpy.einsum's pairing for 3 terms, (g0^2 + g2^2) + g1^2.
template <int D>
__device__ __forceinline__ bool box_ok(const double* blo, const double* bhi, float4 flo, float4 fhi, double reach2) {
  double g[3];
  const float l[3] = {flo.x, flo.y, flo.z}, h[3] = {fhi.x, fhi.y, fhi.z};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double x = fmax(DSUB((double)l[a], bhi[a]), DSUB(blo[a], (double)h[a]));
    g[a] = fmax(0.0, x);
  }
  double s = D == 3 ? DADD(DADD(DMUL(g[0], g[0]), DMUL(g[2], g[2])), DMUL(g[1], g[1]))
                    : DADD(DMUL(g[0], g[0]), DMUL(g[1], g[1]));
  return s <= reach2;
}

template <int D>
__device__ __forceinline__ bool sphere_ok(const float* p, float4 s) {
  float dx = FSUB(p[0], s.x), dy = FSUB(p[1], s.y);
  float dist = FADD(FMUL(dx, dx), FMUL(dy, dy));
  if (D == 3) {
    float dz = FSUB(p[2], s.z);
    dist = FADD(dist, FMUL(dz, dz));
  }
  return dist <= s.w;
}

struct MarkArgs {
  ForestC F;
  GridC g;
  const int32_t* leaves;
  const float4* box;
  const float4* sph;
  const float4* pay;
  const int32_t* bin_ids;
  const int32_t* bin_counts;
  const int32_t* bin_offsets;
  const float4* cbox;       // union boxes of 32-entry bin-CSR chunks
  int64_t n_faces, n_leaves;
  const int64_t* d_n;       // optional device leaf count (n_leaves is then an upper bound)
  const int64_t* d_slice;   // optional device [lo, hi) of leaf positions to mark (multi-GPU shard)
  float d;
  double reach;
  unsigned long long* out;  // [0] marked, [1] tests, [2] evaluated, [3] sphere tests, [4] box culls
  int prefilter;            // k_mark_blocks: lane-level empty-bin prefilter (OW_MARK_PREFILTER=0: off, A/B)
  int dyn;                  // k_mark_blocks: dynamic schedule over out[6] (OW_MARK_DYN, A/B)
};

// Union box of the face boxes of bin-CSR entries [32 g, 32 g + 32) (entries of
// neighbouring bins included: a larger box is still a conservative cull).  The
// FP64 box distance is monotone in the box, so a chunk whose union box fails
// the reference's cull holds no face that passes it.
template <int D>
__global__ void k_chunk_boxes(const int32_t* __restrict__ ids, int64_t n_entries, const float4* __restrict__ box,
                              float4* cbox, const int64_t* d_n) {
  ow_pdl_wait();
  if (d_n && *d_n < n_entries) n_entries = *d_n;  // entry count on the device (n_entries: its bound)
  // warp per chunk: independent loads, min / max (exact, order-free) by shuffles
  const int lane = threadIdx.x & 31;
  const int64_t n_chunks = (n_entries + 31) / 32;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < n_chunks;
       g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t e = g * 32 + lane;
    float4 lo = make_float4(INFINITY, INFINITY, INFINITY, 0.0f), hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.0f);
    if (e < n_entries) {
      const int64_t f = ids ? ids[e] : e;
      lo = box[2 * f];
      hi = box[2 * f + 1];
      lo.w = hi.w = 0.0f;
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo.x = fminf(lo.x, __shfl_xor_sync(0xffffffffu, lo.x, o));
      lo.y = fminf(lo.y, __shfl_xor_sync(0xffffffffu, lo.y, o));
      lo.z = fminf(lo.z, __shfl_xor_sync(0xffffffffu, lo.z, o));
      hi.x = fmaxf(hi.x, __shfl_xor_sync(0xffffffffu, hi.x, o));
      hi.y = fmaxf(hi.y, __shfl_xor_sync(0xffffffffu, hi.y, o));
      hi.z = fmaxf(hi.z, __shfl_xor_sync(0xffffffffu, hi.z, o));
    }
    if (lane == 0) {
      cbox[2 * g] = lo;
      cbox[2 * g + 1] = hi;
    }
  }
}

// Marking, two flat passes so no block's work is one long serial chain:
//  k_mark_blocks : warp per leaf block (runs of blocks taken from a per-pass
//                  counter; runs of several blocks are first prefiltered one
//                  block per lane, block_may_hit).  Cell centres (FP64 -> one FP32
//                  rounding) and bins, the algorithmic test count T; per
//                  distinct bin of its cells, the 32-entry bin chunks whose union
//                  box passes the reference's FP64 box cull.  The first CG
//                  surviving chunks are swept inline (most near-wall blocks hit
//                  there and stop: a mark is an OR); the rest become
//                  (block, chunk, bin) items.
//  k_mark_items  : warp per item, skipped once its block is hit.  Blocks that
//                  reach this pass are mostly undecided ones that must test
//                  every candidate, so flattening them costs no early exits.
// Per chunk: its faces passing the box cull are staged, and the (candidate
// face, cell-in-bin) pairs are swept flattened over the lanes: FP32
// bounding-sphere prefilter, then the full predicate.  Every evaluated pair
// is one the reference evaluates (same culls), so marks are bit-exact even
// where the predicate is ill-conditioned.
constexpr int MARK_WARPS = MARK_THREADS / 32;
#ifndef OW_MARK_CG
#define OW_MARK_CG 4
#endif
constexpr int CG = OW_MARK_CG;  // chunks swept inline by the block pass (levels 0-1; 8 from mark_cg8_from())

struct MarkCounts {
  unsigned long long evaluated = 0, spheres = 0, culls = 0;
};

struct MarkItems {
  int4* items;                  // (leaf position, chunk, bin, 0)
  unsigned long long* n_items;  // device counter
  int64_t cap;
  unsigned* hit;                // [n_leaves] block hit words
};

constexpr int PAIR_CAP = 256;  // sphere-passing (face, cell) pairs buffered per warp

template <int D, int CGN = CG>
struct MarkSmem {
  static constexpr int C = D == 3 ? 64 : 16;
  int cand[MARK_WARPS][32 * CGN];
  float4 sph[MARK_WARPS][32 * CGN];
  float p[MARK_WARPS][C][D];                  // cell centres of the warp's block
  unsigned short pair[MARK_WARPS][PAIR_CAP];  // face index << 6 | cell
};

// cell centres of the lane's cells into the warp's shared table
template <int D, int CGN>
__device__ __forceinline__ void share_cells(MarkSmem<D, CGN>& S, int wid, int lane, const float (*p)[3]) {
  constexpr int C = D == 3 ? 64 : 16;
  constexpr int CPL = D == 3 ? 2 : 1;
#pragma unroll
  for (int k = 0; k < CPL; ++k)
    if (lane + 32 * k < C)
#pragma unroll
      for (int a = 0; a < D; ++a) S.p[wid][lane + 32 * k][a] = p[k][a];
  __syncwarp();
}

// full predicate on the buffered pairs, 32 in parallel (their payload loads
// overlap); true on a hit
template <int D, int CGN>
__device__ __forceinline__ bool eval_pairs(const MarkArgs& A, MarkSmem<D, CGN>& S, int wid, int lane, int npairs, float r2) {
  constexpr int PW = D == 3 ? PAY3 : PAY2;
  for (int k0 = 0; k0 < npairs; k0 += 32) {
    bool h = false;
    if (k0 + lane < npairs) {
      const unsigned pr = S.pair[wid][k0 + lane];
      const int c = (int)(pr & 63u);
      float pp[3];
#pragma unroll
      for (int a = 0; a < D; ++a) pp[a] = S.p[wid][c][a];
      h = near_face<D>(A.pay + (int64_t)S.cand[wid][pr >> 6] * PW, pp, r2);
    }
    if (__any_sync(0xffffffffu, h)) return true;
  }
  return false;
}

// cell centres + bins of the lane's cells (c = lane, lane + 32), block box
template <int D, bool BINNED>
__device__ __forceinline__ void block_cells(const MarkArgs& A, int id, int lane, double* blo, double* bhi,
                                            float (*p)[3], int* bin) {
  constexpr int C = D == 3 ? 64 : 16;
  constexpr int CPL = D == 3 ? 2 : 1;
  const int L = A.F.level[id];
  double q[3];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    q[a] = block_len(A.F, a, L);
    blo[a] = DADD(A.F.dmin[a], DMUL((double)A.F.coord[a][id], q[a]));
    bhi[a] = DADD(blo[a], q[a]);
  }
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    const int c = lane + 32 * k;
    bin[k] = -1;
    if (c < C) {
      int lin = 0, mul = 1;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double u = ((double)((c >> (2 * a)) & 3) + 0.5) / 4.0;
        p[k][a] = __double2float_rn(DADD(blo[a], DMUL(u, q[a])));
        if (BINNED) {
          lin += bin_axis(p[k][a], A.g.min32[a], A.g.len32[a], A.g.B) * mul;
          mul *= A.g.B;
        }
      }
      bin[k] = lin;
    }
  }
}

// box-cull the entries of up to CG chunks gc[] (of bin range [off, off+cnt)),
// stage the survivors, then sweep them face by face: every lane tests its own
// cells (centres in registers, act = cell lies in this bin) against the
// broadcast bounding sphere, and runs the full predicate on the survivors.
// True on a hit (checked after every face: a mark is an OR).
template <int D, bool BINNED, int CGN>
__device__ __forceinline__ bool sweep_chunks(const MarkArgs& A, MarkSmem<D, CGN>& S, int wid, int lane, const int64_t* gc,
                                             int64_t off, int64_t cnt, const double* blo, const double* bhi,
                                             double reach2, float r2, const float (*p)[3], const bool* act,
                                             MarkCounts& cn) {
  constexpr int CPL = D == 3 ? 2 : 1;
  int fv[CGN];
  bool fok[CGN];
#pragma unroll
  for (int j = 0; j < CGN; ++j) {  // independent loads: the id -> box chains overlap
    const int64_t e = gc[j] * 32 + lane;
    fok[j] = gc[j] >= 0 && e >= off && e < off + cnt;
    fv[j] = fok[j] ? (BINNED ? A.bin_ids[e] : (int)e) : 0;
  }
#pragma unroll
  for (int j = 0; j < CGN; ++j)
    if (fok[j]) {
      ++cn.culls;
      fok[j] = box_ok<D>(blo, bhi, A.box[2 * (int64_t)fv[j]], A.box[2 * (int64_t)fv[j] + 1], reach2);
    }
  int nf = 0;
#pragma unroll
  for (int j = 0; j < CGN; ++j) {
    const unsigned fm = __ballot_sync(0xffffffffu, fok[j]);
    if (fok[j]) {
      const int r = nf + __popc(fm & lanemask_lt());
      S.cand[wid][r] = fv[j];
      S.sph[wid][r] = A.sph[fv[j]];
    }
    nf += __popc(fm);
  }
  if (!nf) return false;
  __syncwarp();
  // sphere prefilter over (face, own cell) with the sphere broadcast from shared
  // memory; survivors are buffered and then evaluated 32 at a time
  int npairs = 0;
  unsigned nact = 0;  // the lane's cells in this bin: sphere tests per face (counted once per exit)
#pragma unroll
  for (int k = 0; k < CPL; ++k) nact += act[k] ? 1u : 0u;
  for (int fi = 0; fi < nf; ++fi) {
    const float4 sp = S.sph[wid][fi];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const bool pass = act[k] && sphere_ok<D>(p[k], sp);
      const unsigned m = __ballot_sync(0xffffffffu, pass);
      if (pass) S.pair[wid][npairs + __popc(m & lanemask_lt())] = (unsigned short)((fi << 6) | (lane + 32 * k));
      npairs += __popc(m);
    }
    if (npairs > PAIR_CAP - 64) {  // buffer nearly full: evaluate what we have
      __syncwarp();
      cn.evaluated += lane == 0 ? npairs : 0;
      if (eval_pairs<D, CGN>(A, S, wid, lane, npairs, r2)) {
        cn.spheres += (unsigned long long)nact * (unsigned)(fi + 1);
        return true;
      }
      npairs = 0;
      __syncwarp();
    }
  }
  cn.spheres += (unsigned long long)nact * (unsigned)nf;
  __syncwarp();
  cn.evaluated += lane == 0 ? npairs : 0;
  const bool hit = eval_pairs<D, CGN>(A, S, wid, lane, npairs, r2);
  __syncwarp();
  return hit;
}

__device__ __forceinline__ void flush_counts(const MarkArgs& A, MarkCounts& cn, int lane) {
  for (int o = 16; o > 0; o >>= 1) {
    cn.evaluated += __shfl_xor_sync(0xffffffffu, cn.evaluated, o);
    cn.spheres += __shfl_xor_sync(0xffffffffu, cn.spheres, o);
    cn.culls += __shfl_xor_sync(0xffffffffu, cn.culls, o);
  }
  if (lane == 0) {
    if (cn.evaluated) atomicAdd(&A.out[2], cn.evaluated);
    if (cn.spheres) atomicAdd(&A.out[3], cn.spheres);
    if (cn.culls) atomicAdd(&A.out[4], cn.culls);
  }
}

template <int D, bool BINNED, int CGN>
__device__ __forceinline__ void mark_block(const MarkArgs& A, const MarkItems& M, MarkSmem<D, CGN>& S, int64_t pos,
                                           int lane, int wid, MarkCounts& cn, unsigned long long& t_acc,
                                           unsigned long long& marked);

// Lane-level prefilter of one leaf block (binned marking): false when every
// bin its cells fall in is empty.  Such a block adds nothing to T (its cells'
// bin counts are all 0) and has no candidate to test, so skipping it is exact.
// The cells' bins along an axis lie between the bins of its first and last
// cell centres (centres and bin_axis are monotone in the index), and those two
// centres are formed with block_cells' exact FP64 ops; a bin box of more than
// 64 bins is not scanned (the block takes the full path).
template <int D>
__device__ __forceinline__ bool block_may_hit(const MarkArgs& A, int id) {
  const int L = A.F.level[id];
  int b0[3] = {0, 0, 0}, nb[3] = {1, 1, 1};
  int total = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double q = block_len(A.F, a, L);
    const double blo = DADD(A.F.dmin[a], DMUL((double)A.F.coord[a][id], q));
    // u = (i + 0.5) / 4 for the first and last cell: 0.125 and 0.875 (exact)
    const float p0 = __double2float_rn(DADD(blo, DMUL(0.125, q)));
    const float p3 = __double2float_rn(DADD(blo, DMUL(0.875, q)));
    b0[a] = bin_axis(p0, A.g.min32[a], A.g.len32[a], A.g.B);
    nb[a] = bin_axis(p3, A.g.min32[a], A.g.len32[a], A.g.B) - b0[a] + 1;
    total *= nb[a];
  }
  if (total > 64) return true;
  int any = 0;
  for (int k = 0; k < total; ++k) {
    int r = k, lin = 0, mul = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int i = r % nb[a];
      r /= nb[a];
      lin += (b0[a] + i) * mul;
      mul *= A.g.B;
    }
    any |= __ldg(A.bin_counts + lin);
  }
  return any != 0;
}

static __device__ __forceinline__ bool mark_prefilter_on(const MarkArgs& A) { return A.prefilter != 0; }

// persistent over the level's leaves (the count may live on the device)
template <int D, bool BINNED, int MINB = 6, int CGN = CG>
__global__ void __launch_bounds__(MARK_THREADS, MINB) k_mark_blocks(MarkArgs A, MarkItems M) {
  ow_pdl_wait();
  __shared__ MarkSmem<D, CGN> S;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t lo = A.d_slice ? A.d_slice[0] : 0;
  const int64_t n = A.d_slice ? A.d_slice[1] : (A.d_n ? *A.d_n : A.n_leaves);
  // statistics accumulate per warp over its blocks: one atomic per counter
  // and warp at the end (per block they were same-address atomics from every
  // warp of the grid: 1.6 M of them at C5)
  MarkCounts cn;
  unsigned long long t_acc = 0, marked = 0;
  const int64_t G = (int64_t)gridDim.x * MARK_WARPS, gw = (int64_t)blockIdx.x * MARK_WARPS + wid;
  if (A.dyn) {
    // dynamic schedule: warps take runs of K consecutive leaf positions from a
    // per-pass counter (out[6]); the next run is reserved before the current
    // one is swept, so the atomic's round trip hides behind the work
    const int64_t total = n - lo;
    int64_t K = total / (G * 8);
    K = K < 1 ? 1 : (K > 32 ? 32 : K);
    unsigned long long nxt = 0;
    if (lane == 0) nxt = atomicAdd(&A.out[6], (unsigned long long)K);
    nxt = __shfl_sync(0xffffffffu, nxt, 0);
    while ((int64_t)nxt < total) {
      const int64_t base = lo + (int64_t)nxt;
      unsigned long long nn = 0;
      if (lane == 0) nn = atomicAdd(&A.out[6], (unsigned long long)K);
      if (BINNED && K > 1 && mark_prefilter_on(A)) {
        const int64_t pos = base + lane;
        bool need = false;
        if (lane < K && pos < n) {
          need = block_may_hit<D>(A, A.leaves[pos]);
          if (!need) M.hit[pos] = 0u;
        }
        unsigned m = __ballot_sync(0xffffffffu, need);
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1;
          mark_block<D, BINNED, CGN>(A, M, S, base + j, lane, wid, cn, t_acc, marked);
        }
      } else {
        for (int64_t j = 0; j < K && base + j < n; ++j) mark_block<D, BINNED, CGN>(A, M, S, base + j, lane, wid, cn, t_acc, marked);
      }
      nxt = __shfl_sync(0xffffffffu, nn, 0);
    }
  } else if (BINNED && mark_prefilter_on(A) && n - lo > G) {
    // several blocks per warp: the warp's blocks (the same strided set as
    // below) are prefiltered 32 at a time, one per lane, and only blocks with
    // a non-empty bin take the warp-wide path (C5 level 0: most of the 64^3
    // root blocks lie in empty bins, and each was one dependent-load chain)
    for (int64_t k0 = 0; lo + gw + k0 * G < n; k0 += 32) {
      const int64_t pos = lo + gw + (k0 + lane) * G;
      bool need = false;
      if (pos < n) {
        need = block_may_hit<D>(A, A.leaves[pos]);
        if (!need) M.hit[pos] = 0u;
      }
      unsigned m = __ballot_sync(0xffffffffu, need);
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        mark_block<D, BINNED, CGN>(A, M, S, lo + gw + (k0 + j) * G, lane, wid, cn, t_acc, marked);
      }
    }
  } else {
    for (int64_t pos = lo + gw; pos < n; pos += G) mark_block<D, BINNED, CGN>(A, M, S, pos, lane, wid, cn, t_acc, marked);
  }
  flush_counts(A, cn, lane);
  if (lane == 0) {
    if (t_acc) atomicAdd(&A.out[1], t_acc);
    if (marked) atomicAdd(&A.out[0], marked);
  }
}

template <int D, bool BINNED, int CGN>
__device__ __forceinline__ void mark_block(const MarkArgs& A, const MarkItems& M, MarkSmem<D, CGN>& S, int64_t pos,
                                           int lane, int wid, MarkCounts& cn, unsigned long long& t_acc,
                                           unsigned long long& marked) {
  constexpr int CPL = D == 3 ? 2 : 1;
  const int id = A.leaves[pos];
  if (lane == 0) M.hit[pos] = 0u;  // (this warp owns the block's hit word in this kernel; k_mark_items reads it after)
  double blo[3], bhi[3];
  float p[CPL][3];
  int bin[CPL];
  block_cells<D, BINNED>(A, id, lane, blo, bhi, p, bin);
  share_cells<D, CGN>(S, wid, lane, p);
  unsigned long long t = 0;
#pragma unroll
  for (int k = 0; k < CPL; ++k)
    if (bin[k] >= 0) t += BINNED ? (unsigned long long)A.bin_counts[bin[k]] : (unsigned long long)A.n_faces;
  // algorithmic test count T, one atomic per warp
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  t_acc += t;  // (every lane holds the sum; lane 0's is flushed)
  if (A.F.marks[id] == OW_MARKED) return;
  const double reach2 = DMUL(A.reach, A.reach);
  const float r2 = FMUL(A.d, A.d);
  bool pend[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) pend[k] = bin[k] >= 0;
  bool hit = false, inline_left = true;
  while (!hit) {
    int b = 0;  // next distinct bin: the bin of the lowest pending cell
    bool found = false;
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const unsigned m = __ballot_sync(0xffffffffu, pend[k]);
      if (m && !found) {
        b = __shfl_sync(0xffffffffu, bin[k], __ffs(m) - 1);
        found = true;
      }
    }
    if (!found) break;
#pragma unroll
    for (int k = 0; k < CPL; ++k) pend[k] = pend[k] && !(!BINNED || bin[k] == b);
    const int64_t off = BINNED ? A.bin_offsets[b] : 0;
    const int64_t cnt = BINNED ? A.bin_counts[b] : A.n_faces;
    if (cnt == 0) continue;
    bool act[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) act[k] = bin[k] >= 0 && (!BINNED || bin[k] == b);
    const int64_t g0 = off >> 5, g1 = (off + cnt - 1) >> 5;
    for (int64_t gb = g0; gb <= g1 && !hit; gb += 32) {
      const int64_t g = gb + lane;
      bool cok = false;
      if (g <= g1) {
        ++cn.culls;
        cok = box_ok<D>(blo, bhi, A.cbox[2 * g], A.cbox[2 * g + 1], reach2);
      }
      unsigned cm = __ballot_sync(0xffffffffu, cok);
      if (cm && inline_left) {
        inline_left = false;
        int64_t gc[CGN];
#pragma unroll
        for (int j = 0; j < CGN; ++j) {
          gc[j] = -1;
          if (cm) {
            gc[j] = gb + __ffs(cm) - 1;
            cm &= cm - 1;
          }
        }
        hit = sweep_chunks<D, BINNED, CGN>(A, S, wid, lane, gc, off, cnt, blo, bhi, reach2, r2, p, act, cn);
        if (hit) break;
      }
      if (cm) {  // the rest: (block, chunk, bin) items for the flat pass
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(M.n_items, (unsigned long long)__popc(cm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((int64_t)(base + __popc(cm)) <= M.cap) {
          if ((cm >> lane) & 1u) M.items[base + __popc(cm & lanemask_lt())] = make_int4((int)pos, (int)(gb + lane), b, 0);
        } else {
          // item list full: this warp sweeps its remaining chunks itself
          while (cm && !hit) {
            int64_t gc[CGN];
#pragma unroll
            for (int j = 0; j < CGN; ++j) {
              gc[j] = -1;
              if (cm) {
                gc[j] = gb + __ffs(cm) - 1;
                cm &= cm - 1;
              }
            }
            hit = sweep_chunks<D, BINNED, CGN>(A, S, wid, lane, gc, off, cnt, blo, bhi, reach2, r2, p, act, cn);
          }
        }
      }
    }
  }
  if (lane == 0) {
    if (hit && atomicOr(&M.hit[pos], 1u) == 0u) {
      A.F.marks[id] = OW_MARKED;
      ++marked;
    }
  }
}

template <int D, bool BINNED>
__global__ void __launch_bounds__(MARK_THREADS, 6) k_mark_items(MarkArgs A, MarkItems M) {
  ow_pdl_wait();
  constexpr int CPL = D == 3 ? 2 : 1;
  __shared__ MarkSmem<D> S;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t n = min((int64_t)*M.n_items, M.cap);  // items past cap were swept by their block warp
  const double reach2 = DMUL(A.reach, A.reach);
  const float r2 = FMUL(A.d, A.d);
  MarkCounts cn;
  unsigned long long marked = 0;
  for (int64_t it = (int64_t)blockIdx.x * MARK_WARPS + wid; it < n; it += (int64_t)gridDim.x * MARK_WARPS) {
    const int4 item = M.items[it];
    const int pos = item.x;
    // block already marked: lane 0 reads the flag (other warps atomicOr it at
    // any time) and broadcasts it, so the skip is warp-uniform before the
    // full-mask collectives below
    unsigned done = 0u;
    if (lane == 0) done = *(volatile unsigned*)&M.hit[pos];
    if (__shfl_sync(0xffffffffu, done, 0)) continue;
    const int id = A.leaves[pos];
    const int b = item.z;
    double blo[3], bhi[3];
    float p[CPL][3];
    int bin[CPL];
    block_cells<D, BINNED>(A, id, lane, blo, bhi, p, bin);
    share_cells<D, CG>(S, wid, lane, p);
    bool act[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) act[k] = bin[k] >= 0 && (!BINNED || bin[k] == b);
    const int64_t off = BINNED ? A.bin_offsets[b] : 0;
    const int64_t cnt = BINNED ? A.bin_counts[b] : A.n_faces;
    int64_t gc[CG];
#pragma unroll
    for (int j = 0; j < CG; ++j) gc[j] = j == 0 ? (int64_t)item.y : -1;
    const bool hit =
        sweep_chunks<D, BINNED, CG>(A, S, wid, lane, gc, off, cnt, blo, bhi, reach2, r2, p, act, cn);
    if (hit && lane == 0 && atomicOr(&M.hit[pos], 1u) == 0u) {
      A.F.marks[id] = OW_MARKED;
      ++marked;
    }
  }
  flush_counts(A, cn, lane);
  if (lane == 0 && marked) atomicAdd(&A.out[0], marked);
}

// ---------------------------------------------------------------------------
// cell-face links (build_cell_face_links, nearwall.py:522-594)
// Pass 1 counts the links of every leaf cell and finds the first overflowing
// (block position, bin, cell) key; pass 2 writes each cell's faces in
// ascending order (bins hold ascending ids; a warp walks them in order with
// a ballot prefix).  One CTA per leaf block, one warp per cell at a time.
// ---------------------------------------------------------------------------
struct LinkArgs {
  ForestC F;
  GridC g;
  const int32_t* leaves;
  const float4* box;
  const float4* pay;
  const int32_t* bin_ids;
  const int32_t* bin_counts;
  const int32_t* bin_offsets;
  float d;
  double reach;
  int64_t capacity;
  int32_t* cell_cnt;          // pass 1 out: per cell count
  unsigned long long* over;   // pass 1 out: min overflow key
  const int64_t* cell_off;    // pass 2 in: per cell link offset
  int32_t* face_ids;          // pass 2 out
};

template <int D, bool EMIT>
__global__ void __launch_bounds__(MARK_THREADS) k_links(LinkArgs A) {
  ow_pdl_wait();
  constexpr int C = D == 3 ? 64 : 16;
  constexpr int PW = D == 3 ? PAY3 : PAY2;
  __shared__ float s_cen[C][D];
  __shared__ int s_bin[C];
  __shared__ int s_cnt[C];
  const ForestC& F = A.F;
  const int64_t pos = blockIdx.x;
  const int id = A.leaves[pos];
  const int L = F.level[id];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double blo[3], bhi[3];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double q = block_len(F, a, L);
    blo[a] = DADD(F.dmin[a], DMUL((double)F.coord[a][id], q));
    bhi[a] = DADD(blo[a], q);
  }
  if (tid < C) {
    float p[3];
    int lin = 0, mul = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double q = block_len(F, a, L);
      double u = ((double)((tid >> (2 * a)) & 3) + 0.5) / 4.0;
      p[a] = __double2float_rn(DADD(blo[a], DMUL(u, q)));
      s_cen[tid][a] = p[a];
      lin += bin_axis(p[a], A.g.min32[a], A.g.len32[a], A.g.B) * mul;
      mul *= A.g.B;
    }
    s_bin[tid] = lin;
    s_cnt[tid] = 0;
  }
  __syncthreads();
  const double reach2 = DMUL(A.reach, A.reach);
  const float r2 = FMUL(A.d, A.d);
  for (int ci = warp; ci < C; ci += MARK_THREADS / 32) {
    const int b = s_bin[ci];
    const int32_t* src = A.bin_ids + A.bin_offsets[b];
    const int n = A.bin_counts[b];
    float p[3];
#pragma unroll
    for (int a = 0; a < D; ++a) p[a] = s_cen[ci][a];
    int64_t out = EMIT ? A.cell_off[pos * C + ci] : 0;
    int cnt = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      int j = j0 + lane;
      bool hit = false;
      int f = 0;
      if (j < n) {
        f = src[j];
        if (box_ok<D>(blo, bhi, A.box[2 * (int64_t)f], A.box[2 * (int64_t)f + 1], reach2))
          hit = near_face<D>(A.pay + (int64_t)f * PW, p, r2);
      }
      unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (EMIT && hit) A.face_ids[out + cnt + __popc(bal & lanemask_lt())] = f;
      cnt += __popc(bal);
    }
    if (lane == 0) s_cnt[ci] = cnt;
  }
  __syncthreads();
  if (!EMIT && tid < C) {
    int cnt = s_cnt[tid];
    A.cell_cnt[pos * C + tid] = cnt;
    if (cnt > A.capacity) {
      // first overflow in the reference's order: block asc, bin asc, cell asc
      unsigned long long key = ((unsigned long long)pos << 40) | ((unsigned long long)s_bin[tid] << 8) | tid;
      atomicMin(A.over, key);
    }
  }
}

struct CellCntLoad {
  const int32_t* c;
  __device__ int64_t operator()(int64_t i) const { return c[i]; }
};
struct CellOffStore {
  int64_t* off;
  __device__ void operator()(int64_t i, int64_t e, int64_t) const { off[i] = e; }
};
struct LinkedLoad {
  const int32_t* c;
  __device__ int64_t operator()(int64_t i) const { return c[i] > 0; }
};
struct NullStoreL {
  __device__ void operator()(int64_t, int64_t, int64_t) const {}
};
struct LinkedStore {
  const int32_t* leaves;
  const int32_t* cnt;
  const int64_t* cell_off;
  int C;
  int64_t* block_ids;
  int64_t* cell_idx;
  int64_t* offsets;
  __device__ void operator()(int64_t i, int64_t e, int64_t v) const {
    if (!v) return;
    block_ids[e] = leaves[i / C];
    cell_idx[e] = i % C;
    offsets[e] = cell_off[i];
  }
};

__global__ void k_near_pairs(int dim, const float* __restrict__ pts, const float* __restrict__ faces,
                             const float* __restrict__ dd, int64_t n, uint8_t* out) {
  ow_pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 pay[PAY3];
  float d = dd[i];
  float r2 = FMUL(d, d);
  float p[3];
  if (dim == 3) {
    face_prep_one<3>(faces, n, i, d, pay);
    for (int a = 0; a < 3; ++a) p[a] = pts[i * 3 + a];
    out[i] = near_face<3>(pay, p, r2);
  } else {
    face_prep_one<2>(faces, n, i, d, pay);
    for (int a = 0; a < 2; ++a) p[a] = pts[i * 2 + a];
    out[i] = near_face<2>(pay, p, r2);
  }
}

}  // namespace

// Launch one marking pass; statistics accumulate into d_out[0..2] (marked,
// tests, evaluated) on the device (no host round trip: the native driver reads
// them once at the end).
// (OW_MARK_MINB: resident CTAs per SM the 3D binned block pass is compiled
// for — 6: 80 registers (measured best of 4..8 at C2 / C4 / C5; 4 and 5 remove the
// spills but lose occupancy)
static int mark_minb() {
  static const int v = [] {
    const char* e = getenv("OW_MARK_MINB");
    return e ? atoi(e) : 6;
  }();
  return v;
}
// first level whose 3D binned block pass sweeps 8 chunks inline
// (OW_MARK_CG8_FROM: A/B, 99 = never; tools/ab_markcg8.sh on one B200: from
// level 2, C3 1.521 -> 1.439 ms, C4 2.100 -> 2.026; C2 / C5 mark levels 0-1
// only, where 8 inline chunks were slower: C2 0.319 -> 0.328 and C5 3.54 ->
// 3.73 ms with 8 on every level)
static int mark_cg8_from() {
  static const int v = [] {
    const char* e = getenv("OW_MARK_CG8_FROM");
    return e ? atoi(e) : 2;
  }();
  return v;
}
int ow_mark_launch(ow_ctx* ctx, ow_forest* f, const int32_t* d_leaves, int64_t n_leaves, const float* d_coords,
                   int64_t n_faces, int64_t geom_key, const ow_grid* grid, const int32_t* d_bin_ids,
                   const int32_t* d_bin_counts, const int32_t* d_bin_offsets, int64_t n_bin_entries, float d_spec,
                   double reach, unsigned long long* out, cudaStream_t s, const int64_t* d_n_leaves,
                   bool chunk_boxes_ready, const int64_t* d_slice, const int64_t* d_bin_entries, int level) {
  if (!(d_spec > 0.0f)) {
    ow_set_error("near-wall distance must be positive, got %g", (double)d_spec);
    return OW_ERR_INVALID;
  }
  if (n_faces <= 0) {
    ow_set_error("cannot mark near-wall blocks with empty geometry");
    return OW_ERR_INVALID;
  }
  const bool binned = d_bin_ids != nullptr;
  if (binned && (!grid || grid->dim != f->dim)) {
    ow_set_error("bin grid does not match the forest");
    return OW_ERR_INVALID;
  }
  OW_PROF_BEGIN(ctx, PROF_PREP, s);
  OW_TRY(prepare_faces(ctx, f->dim, d_coords, n_faces, geom_key, d_spec, reach, s));
  OW_PROF_END(ctx, PROF_PREP, s);
  if (n_leaves <= 0) return OW_OK;
  MarkArgs A;
  A.F = make_forestc(f);
  if (binned) A.g = make_gridc(grid);
  A.leaves = d_leaves;
  A.box = (const float4*)ctx->slot_ptr[SLOT_FACE_BOX];
  A.sph = (const float4*)ctx->slot_ptr[SLOT_FACE_SPHERE];
  A.pay = (const float4*)ctx->slot_ptr[SLOT_FACE_PREP];
  A.bin_ids = d_bin_ids;
  A.bin_counts = d_bin_counts;
  A.bin_offsets = d_bin_offsets;
  A.n_faces = n_faces;
  A.d = d_spec;
  A.reach = reach;
  A.out = out;
  {
    static const int pf = [] {
      const char* e = getenv("OW_MARK_PREFILTER");
      return e ? atoi(e) : 1;
    }();
    A.prefilter = pf;
    // dynamic block schedule (A/B on one B200, tools/ab_markdyn.sh, with 12
    // CTAs per SM: C2 0.321 -> 0.319 ms, C3 1.570 -> 1.523, C4 2.180 -> 2.105,
    // C5 3.577 -> 3.554; the static stride's best grid was 24 per SM)
    static const int dy = [] {
      const char* e = getenv("OW_MARK_DYN");
      return e ? atoi(e) : 1;
    }();
    A.dyn = dy;
  }
  const int64_t n_entries = binned ? n_bin_entries : n_faces;
  void *pc, *pi, *ph;
  OW_TRY(ow_slot(ctx, SLOT_MARK_CBOX, 32 * (size_t)((n_entries + 31) / 32 + 1), s, &pc));
  // (block, chunk) items: 16 per leaf; a block warp that finds the list full
  // sweeps its remaining chunks itself
  const int64_t cap = 16 * n_leaves + 256;
  OW_TRY(ow_slot(ctx, SLOT_MARK_ITEMS, 16 * (size_t)cap, s, &pi));
  OW_TRY(ow_slot(ctx, SLOT_MARK_HIT, 4 * (size_t)n_leaves + 8, s, &ph));
  A.cbox = (const float4*)pc;
  A.n_leaves = n_leaves;
  A.d_n = d_n_leaves;
  A.d_slice = d_slice;
  MarkItems M;
  M.items = (int4*)pi;
  M.n_items = out + 5;  // (zeroed with the statistics; the hit words are cleared by k_mark_blocks per block)
  M.cap = cap;
  M.hit = (unsigned*)ph;

  if (!chunk_boxes_ready) {  // the driver reuses them while the bins and face boxes are unchanged
    const int cg = ow_blocks((n_entries + 31) / 32, 4, 16 * OW_SMS);
    const int64_t* dn = binned ? d_bin_entries : nullptr;
    if (f->dim == 3) ow_launch(k_chunk_boxes<3>, cg, 128, 0, s, d_bin_ids, n_entries, A.box, (float4*)pc, dn);
    else ow_launch(k_chunk_boxes<2>, cg, 128, 0, s, d_bin_ids, n_entries, A.box, (float4*)pc, dn);
  }
  OW_PROF_BEGIN(ctx, PROF_MARK, s);
  // two waves of CTAs (k_mark_blocks takes its blocks from a per-pass counter)
  const int64_t nblk = (n_leaves + MARK_WARPS - 1) / MARK_WARPS;
  static const int64_t per_sm = [] {  // CTAs per SM of the block pass grid (OW_MARK_CTAS_PER_SM: A/B)
    const char* e = getenv("OW_MARK_CTAS_PER_SM");
    return e && atoi(e) > 0 ? (int64_t)atoi(e) : (int64_t)12;
  }();
  static const int64_t max_ctas = [] {  // OW_MARK_MAX_CTAS: total cap (tests: many blocks per warp)
    const char* e = getenv("OW_MARK_MAX_CTAS");
    return e && atoi(e) > 0 ? (int64_t)atoi(e) : (int64_t)0;
  }();
  int64_t ng = nblk < per_sm * OW_SMS ? nblk : per_sm * OW_SMS;
  if (max_ctas > 0 && ng > max_ctas) ng = max_ctas;
  dim3 grd((unsigned)ng);
  const int gi = 8 * OW_SMS;
  if (f->dim == 3) {
    if (binned) {
      // inline chunks per block: 8 from level mark_cg8_from() on (deeper
      // levels: small blocks inside large bins), 4 above
      if (level >= mark_cg8_from()) ow_launch(k_mark_blocks<3, true, 6, 8>, grd, MARK_THREADS, 0, s, A, M);
      else if (mark_minb() == 8) ow_launch(k_mark_blocks<3, true, 8>, grd, MARK_THREADS, 0, s, A, M);
      else if (mark_minb() == 7) ow_launch(k_mark_blocks<3, true, 7>, grd, MARK_THREADS, 0, s, A, M);
      else ow_launch(k_mark_blocks<3, true>, grd, MARK_THREADS, 0, s, A, M);
      ow_launch(k_mark_items<3, true>, gi, MARK_THREADS, 0, s, A, M);
    } else {
      ow_launch(k_mark_blocks<3, false>, grd, MARK_THREADS, 0, s, A, M);
      ow_launch(k_mark_items<3, false>, gi, MARK_THREADS, 0, s, A, M);
    }
  } else {
    if (binned) {
      ow_launch(k_mark_blocks<2, true>, grd, MARK_THREADS, 0, s, A, M);
      ow_launch(k_mark_items<2, true>, gi, MARK_THREADS, 0, s, A, M);
    } else {
      ow_launch(k_mark_blocks<2, false>, grd, MARK_THREADS, 0, s, A, M);
      ow_launch(k_mark_items<2, false>, gi, MARK_THREADS, 0, s, A, M);
    }
  }
  ctx->launches += 3;
  OW_PROF_END(ctx, PROF_MARK, s);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

extern "C" int ow_mark_near_wall(ow_ctx* ctx, ow_forest* f, const int32_t* d_leaves, int64_t n_leaves,
                                 const float* d_coords, int64_t n_faces, int64_t geom_key, const ow_grid* grid,
                                 const int32_t* d_bin_ids, const int32_t* d_bin_counts, const int32_t* d_bin_offsets,
                                 int64_t n_bin_entries, float d_spec, double reach, int64_t* out_marked,
                                 int64_t* out_tests, int64_t* out_evaluated, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* out = (unsigned long long*)(ctx->d_small + 16);
  OW_CUDA(cudaMemsetAsync(out, 0, MARK_STATS * 8, s));
  OW_TRY(ow_mark_launch(ctx, f, d_leaves, n_leaves, d_coords, n_faces, geom_key, grid, d_bin_ids, d_bin_counts,
                        d_bin_offsets, n_bin_entries, d_spec, reach, out, s));
  int64_t h[3];
  OW_TRY(ow_readback(ctx, ctx->d_small + 16, 3, h, s));
  *out_marked = h[0];
  *out_tests = h[1];
  *out_evaluated = h[2];
  return OW_OK;
}

extern "C" int ow_cell_face_links_count(ow_ctx* ctx, const ow_forest* f, const int32_t* d_leaves, int64_t n_leaves,
                                        const float* d_coords, int64_t n_faces, int64_t geom_key, const ow_grid* grid,
                                        const int32_t* d_bin_ids, const int32_t* d_bin_counts,
                                        const int32_t* d_bin_offsets, float d_link, double reach, int64_t capacity,
                                        int64_t* out_cells, int64_t* out_links, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!(d_link > 0.0f)) {
    ow_set_error("near-wall distance must be positive, got %g", (double)d_link);
    return OW_ERR_INVALID;
  }
  const int C = f->dim == 3 ? 64 : 16;
  OW_TRY(prepare_faces(ctx, f->dim, d_coords, n_faces, geom_key, d_link, reach, s));
  int64_t ncells = n_leaves * C;
  void *pc, *po;
  OW_TRY(ow_slot(ctx, SLOT_LINK_CNT, 4 * (size_t)ncells, s, &pc));
  OW_TRY(ow_slot(ctx, SLOT_LINK_OFF, 8 * (size_t)(ncells + 1), s, &po));
  unsigned long long* over = (unsigned long long*)(ctx->d_small + 24);
  OW_CUDA(cudaMemsetAsync(over, 0xff, 8, s));
  LinkArgs A;
  memset(&A, 0, sizeof(A));
  A.F = make_forestc(f);
  A.g = make_gridc(grid);
  A.leaves = d_leaves;
  A.box = (const float4*)ctx->slot_ptr[SLOT_FACE_BOX];
  A.pay = (const float4*)ctx->slot_ptr[SLOT_FACE_PREP];
  A.bin_ids = d_bin_ids;
  A.bin_counts = d_bin_counts;
  A.bin_offsets = d_bin_offsets;
  A.d = d_link;
  A.reach = reach;
  A.capacity = capacity;
  A.cell_cnt = (int32_t*)pc;
  A.over = over;
  if (n_leaves > 0) {
    if (f->dim == 3) ow_launch(k_links<3, false>, (unsigned)n_leaves, MARK_THREADS, 0, s, A);
    else ow_launch(k_links<2, false>, (unsigned)n_leaves, MARK_THREADS, 0, s, A);
    OW_LAUNCHED(ctx);
    OW_CHECK_LAUNCH();
  }
  OW_TRY(scan(ctx, CellCntLoad{(const int32_t*)pc}, CellOffStore{(int64_t*)po}, ncells, ctx->d_small + 25, s));
  OW_TRY(scan(ctx, LinkedLoad{(const int32_t*)pc}, NullStoreL{}, ncells, ctx->d_small + 26, s));
  int64_t h[3];
  OW_TRY(ow_readback(ctx, ctx->d_small + 24, 3, h, s));
  if (h[0] != -1) {
    unsigned long long key = (unsigned long long)h[0];
    int64_t pos = (int64_t)(key >> 40);
    int cell = (int)(key & 0xff);
    int32_t bid, cnt;
    OW_CUDA(cudaMemcpyAsync(&bid, d_leaves + pos, 4, cudaMemcpyDeviceToHost, s));
    OW_CUDA(cudaMemcpyAsync(&cnt, (int32_t*)pc + pos * C + cell, 4, cudaMemcpyDeviceToHost, s));
    OW_CUDA(cudaStreamSynchronize(s));
    ow_set_error("cell-face link overflow: block %d cell %d links %d faces, capacity %lld", bid, cell, cnt,
                 (long long)capacity);
    return OW_ERR_CAPACITY;
  }
  ctx->link_total = h[1];
  ctx->link_cells = h[2];
  ctx->link_leaves = n_leaves;
  ctx->link_dim = f->dim;
  ctx->link_forest = *f;
  ctx->link_grid = *grid;
  ctx->link_coords = d_coords;
  ctx->link_bin_ids = d_bin_ids;
  ctx->link_bin_counts = d_bin_counts;
  ctx->link_bin_offsets = d_bin_offsets;
  ctx->link_d = d_link;
  ctx->link_reach = reach;
  ctx->link_leaves_ptr = d_leaves;
  ctx->link_key = geom_key;
  ctx->link_faces = n_faces;
  *out_cells = h[2];
  *out_links = h[1];
  return OW_OK;
}

extern "C" int ow_cell_face_links_emit(ow_ctx* ctx, int64_t* d_block_ids, int64_t* d_cell_indices, int64_t* d_offsets,
                                       int32_t* d_face_ids, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (ctx->link_dim != 2 && ctx->link_dim != 3) {
    ow_set_error("ow_cell_face_links_emit without ow_cell_face_links_count");
    return OW_ERR_INVALID;
  }
  const int C = ctx->link_dim == 3 ? 64 : 16;
  int64_t ncells = ctx->link_leaves * C;
  OW_TRY(prepare_faces(ctx, ctx->link_dim, ctx->link_coords, ctx->link_faces, ctx->link_key, ctx->link_d,
                       ctx->link_reach, s));
  const int32_t* cnt = (const int32_t*)ctx->slot_ptr[SLOT_LINK_CNT];
  const int64_t* off = (const int64_t*)ctx->slot_ptr[SLOT_LINK_OFF];
  OW_TRY(scan(ctx, LinkedLoad{cnt},
              LinkedStore{ctx->link_leaves_ptr, cnt, off, C, d_block_ids, d_cell_indices, d_offsets}, ncells,
              nullptr, s));
  OW_CUDA(cudaMemcpyAsync(d_offsets + ctx->link_cells, &ctx->link_total, 8, cudaMemcpyHostToDevice, s));
  LinkArgs A;
  memset(&A, 0, sizeof(A));
  A.F = make_forestc(&ctx->link_forest);
  A.g = make_gridc(&ctx->link_grid);
  A.leaves = ctx->link_leaves_ptr;
  A.box = (const float4*)ctx->slot_ptr[SLOT_FACE_BOX];
  A.pay = (const float4*)ctx->slot_ptr[SLOT_FACE_PREP];
  A.bin_ids = ctx->link_bin_ids;
  A.bin_counts = ctx->link_bin_counts;
  A.bin_offsets = ctx->link_bin_offsets;
  A.d = ctx->link_d;
  A.reach = ctx->link_reach;
  A.cell_off = off;
  A.face_ids = d_face_ids;
  if (ctx->link_leaves > 0) {
    if (ctx->link_dim == 3) ow_launch(k_links<3, true>, (unsigned)ctx->link_leaves, MARK_THREADS, 0, s, A);
    else ow_launch(k_links<2, true>, (unsigned)ctx->link_leaves, MARK_THREADS, 0, s, A);
    OW_LAUNCHED(ctx);
    OW_CHECK_LAUNCH();
  }
  OW_CUDA(cudaStreamSynchronize(s));  // the host offset copy reads ctx memory
  return OW_OK;
}

extern "C" int ow_near_pairs(ow_ctx* ctx, int32_t dim, const float* d_points, const float* d_faces, const float* d_d,
                             int64_t n, uint8_t* d_out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (dim != 2 && dim != 3) {
    ow_set_error("dim must be 2 or 3, got %d", dim);
    return OW_ERR_INVALID;
  }
  if (n <= 0) return OW_OK;
  ow_launch(k_near_pairs, ow_blocks(n, 128), 128, 0, s, dim, d_points, d_faces, d_d, n, d_out);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}
