// Lattice boundary links + wall-distance fractions q on the finest level
// (north-star extension; no reference counterpart, oracle/lattice.py is the
// checker and DESIGN.md §Lattice links the definition).
//
// Candidates come from an AABB-overlap bin CSR (a face is stored in every bin
// its float32 AABB touches) plus a packed 64-byte record per face (v0, edge
// vectors, float32 box, first bin), built once per (geometry, grid).
// The work is flattened into three independent item lists so every stage
// runs at full occupancy without per-block serial latency:
//   k_lat_count : warp per finest leaf block, counts the faces whose box meets
//                 the block box grown by two cells (each face once: in the
//                 first bin of its range ∩ the block's range).
//   scan        : pair offsets + candidate-block ranks (one packed scan).
//   k_lat_pairs : (block, face) candidate pairs.
//   k_lat_star  : (pair, cell) items whose cell star box — the union of its
//                 link boxes — meets the face box.
//   k_lat_links : per item, every direction: exact float32 link-AABB test,
//                 then Moller-Trumbore (3D) / segment-segment (2D) with a fixed
//                 op order; atomicOr flag bits, atomicMin q bits.
//   k_lat_bcount + scan + k_lat_emit : boundary rows in (block, cell) order.
#include "ow_scan.cuh"
#include <string.h>

namespace {

using ow::scan;

constexpr int LAT_THREADS = 256;
constexpr int QMAX = 27;
constexpr int CNT_WARPS = 8;

struct Dirs {
  int8_t c[QMAX][3];
};

template <int D>
__device__ __forceinline__ void face_verts(const float* __restrict__ c, int64_t n, int64_t f, float v[3][3]) {
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int a = 0; a < D; ++a) v[j][a] = c[((int64_t)j * D + a) * n + f];
}

template <int D>
__device__ __forceinline__ void vert_box(const float v[3][3], float* lo, float* hi) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lo[a] = v[0][a];
    hi[a] = v[0][a];
#pragma unroll
    for (int j = 1; j < D; ++j) {
      lo[a] = fminf(lo[a], v[j][a]);
      hi[a] = fmaxf(hi[a], v[j][a]);
    }
  }
}

// ---- AABB-overlap bin CSR + packed face records ------------------------------
template <int D>
__device__ __forceinline__ int64_t abin_range(const GridC& g, const float* lo, const float* hi, int* blo, int* ext) {
  int64_t v = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    blo[a] = bin_axis(lo[a], g.min32[a], g.len32[a], g.B);
    ext[a] = bin_axis(hi[a], g.min32[a], g.len32[a], g.B) - blo[a] + 1;
    v *= ext[a];
  }
  return v;
}

template <int D>
struct AbinCountLoad {
  GridC g;
  const float* c;
  int64_t n;
  __device__ int64_t operator()(int64_t f) const {
    float v[3][3], lo[3], hi[3];
    int bl[3], ex[3];
    face_verts<D>(c, n, f, v);
    vert_box<D>(v, lo, hi);
    return abin_range<D>(g, lo, hi, bl, ex);
  }
};

// record layout (float4 x 4):
//  3D: [v0.xyz lo.x] [e1.xyz lo.y] [e2.xyz lo.z] [hi.xyz binlo]
//  2D: [a.xy s.xy]   [lo.xy hi.xy] [binlo 0 0 0] [0 0 0 0]
// binlo packs the face's first bin per axis, 10 bits each (B <= 1024).
template <int D>
__global__ void k_abin_emit(GridC g, const float* __restrict__ c, int64_t n, const int64_t* foff, uint32_t* keys,
                            int32_t* vals, int32_t* counts, float4* rec) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  float v[3][3], lo[3], hi[3];
  int bl[3] = {0, 0, 0}, ex[3];
  face_verts<D>(c, n, f, v);
  vert_box<D>(v, lo, hi);
  int64_t cnt = abin_range<D>(g, lo, hi, bl, ex);
  unsigned packed = (unsigned)bl[0] | ((unsigned)bl[1] << 10) | ((unsigned)(D == 3 ? bl[2] : 0) << 20);
  float pk = __uint_as_float(packed);
  if (D == 3) {
    rec[4 * f + 0] = make_float4(v[0][0], v[0][1], v[0][2], lo[0]);
    rec[4 * f + 1] = make_float4(FSUB(v[1][0], v[0][0]), FSUB(v[1][1], v[0][1]), FSUB(v[1][2], v[0][2]), lo[1]);
    rec[4 * f + 2] = make_float4(FSUB(v[2][0], v[0][0]), FSUB(v[2][1], v[0][1]), FSUB(v[2][2], v[0][2]), lo[2]);
    rec[4 * f + 3] = make_float4(hi[0], hi[1], hi[2], pk);
  } else {
    rec[4 * f + 0] = make_float4(v[0][0], v[0][1], FSUB(v[1][0], v[0][0]), FSUB(v[1][1], v[0][1]));
    rec[4 * f + 1] = make_float4(lo[0], lo[1], hi[0], hi[1]);
    rec[4 * f + 2] = make_float4(pk, 0.0f, 0.0f, 0.0f);
    rec[4 * f + 3] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
  int64_t pos = foff[f];
  for (int64_t k = 0; k < cnt; ++k) {
    int64_t rem = k, lin = 0, mul = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      lin += (int64_t)(bl[a] + rem % ex[a]) * mul;
      rem /= ex[a];
      mul *= g.B;
    }
    keys[pos + k] = (uint32_t)lin;
    vals[pos + k] = (int32_t)f;
    atomicAdd(&counts[lin], 1);
  }
}

template <int D>
int build_abins(ow_ctx* ctx, const GridC& g, const float* c, int64_t n, int64_t key, cudaStream_t s) {
  int64_t nb = 1;
  for (int a = 0; a < D; ++a) nb *= g.B;
  if (g.B > 1024) {
    ow_set_error("lattice candidate grid limited to 1024 bins per axis");
    return OW_ERR_INVALID;
  }
  if (key >= 0 && ctx->abin_key == key && ctx->abin_B == g.B && ctx->abin_dim == D) return OW_OK;
  void *pfo, *pcnt, *poff, *prec;
  OW_TRY(ow_slot(ctx, SLOT_LAT_BOFF, 8 * (size_t)(n + 1), s, &pfo));
  OW_TRY(scan(ctx, AbinCountLoad<D>{g, c, n}, ow::StoreExcl<int64_t>{(int64_t*)pfo}, n, ctx->d_small + 32, s));
  int64_t E;
  OW_TRY(ow_readback(ctx, ctx->d_small + 32, 1, &E, s));
  if (E >= (int64_t(1) << 31)) {
    ow_set_error("lattice candidate bins overflow (%lld entries)", (long long)E);
    return OW_ERR_CAPACITY;
  }
  void *pk0, *pv0, *pk1, *pv1;
  OW_TRY(ow_slot(ctx, SLOT_PAIR_KEY0, 4 * (size_t)E, s, &pk0));
  OW_TRY(ow_slot(ctx, SLOT_PAIR_VAL0, 4 * (size_t)E, s, &pv0));
  OW_TRY(ow_slot(ctx, SLOT_PAIR_KEY1, 4 * (size_t)E, s, &pk1));
  OW_TRY(ow_slot(ctx, SLOT_PAIR_VAL1, 4 * (size_t)E, s, &pv1));
  OW_TRY(ow_slot(ctx, SLOT_ABIN_CNT, 4 * (size_t)nb, s, &pcnt));
  OW_TRY(ow_slot(ctx, SLOT_ABIN_OFF, 4 * (size_t)nb, s, &poff));
  OW_TRY(ow_slot(ctx, SLOT_LAT_REC, 64 * (size_t)n, s, &prec));
  OW_CUDA(cudaMemsetAsync(pcnt, 0, 4 * (size_t)nb, s));
  k_abin_emit<D><<<ow_blocks(n, 256), 256, 0, s>>>(g, c, n, (const int64_t*)pfo, (uint32_t*)pk0, (int32_t*)pv0,
                                                  (int32_t*)pcnt, (float4*)prec);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  int bits = 0;
  while ((int64_t(1) << bits) < nb) ++bits;
  uint32_t* rk;
  int32_t* rv;
  OW_TRY(ow::radix_sort_pairs(ctx, (uint32_t*)pk0, (int32_t*)pv0, (uint32_t*)pk1, (int32_t*)pv1, E, bits, &rk, &rv, s));
  void* pids;
  OW_TRY(ow_slot(ctx, SLOT_ABIN_IDS, 4 * (size_t)E, s, &pids));
  if (E > 0) OW_CUDA(cudaMemcpyAsync(pids, rv, 4 * (size_t)E, cudaMemcpyDeviceToDevice, s));
  OW_TRY(scan(ctx, ow::LoadArr<int32_t>{(const int32_t*)pcnt}, ow::StoreExcl<int32_t>{(int32_t*)poff}, nb, nullptr, s));
  ctx->abin_key = key;
  ctx->abin_B = g.B;
  ctx->abin_dim = D;
  return OW_OK;
}

// ---- shared geometry of one finest block ---------------------------------------
struct BlockFrame {
  double blo[3];
  float h32[3], glo[3], ghi[3];  // cell size, outward-rounded box grown by two cells
  int rlo[3], rhi[3];            // bin range of the grown box
};

template <int D>
__device__ __forceinline__ BlockFrame block_frame(const ForestC& F, const GridC& g, int id) {
  BlockFrame b;
  const int L = F.level[id];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b.h32[a] = b.glo[a] = b.ghi[a] = 0.0f;
    b.rlo[a] = b.rhi[a] = 0;
    b.blo[a] = 0.0;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double q = block_len(F, a, L);
    b.blo[a] = DADD(F.dmin[a], DMUL((double)F.coord[a][id], q));
    double bhi = DADD(b.blo[a], q);
    double h64 = q / 4.0;  // exact (power-of-two scale)
    b.h32[a] = __double2float_rn(h64);
    b.glo[a] = __double2float_rd(b.blo[a] - 2.0 * h64);
    b.ghi[a] = __double2float_ru(bhi + 2.0 * h64);
    b.rlo[a] = bin_axis(b.glo[a], g.min32[a], g.len32[a], g.B);
    b.rhi[a] = bin_axis(b.ghi[a], g.min32[a], g.len32[a], g.B);
  }
  return b;
}

// candidate test on a packed record: face box meets the grown box, and this
// is the face's first bin inside the block's range
template <int D>
__device__ __forceinline__ bool is_candidate(const float4* __restrict__ rec, int f, const BlockFrame& b,
                                             const int* bx) {
  float lo[3], hi[3];
  unsigned pk;
  if (D == 3) {
    float4 r0 = rec[4 * f], r1 = rec[4 * f + 1], r2 = rec[4 * f + 2], r3 = rec[4 * f + 3];
    lo[0] = r0.w, lo[1] = r1.w, lo[2] = r2.w;
    hi[0] = r3.x, hi[1] = r3.y, hi[2] = r3.z;
    pk = __float_as_uint(r3.w);
  } else {
    float4 r1 = rec[4 * f + 1], r2 = rec[4 * f + 2];
    lo[0] = r1.x, lo[1] = r1.y, hi[0] = r1.z, hi[1] = r1.w;
    pk = __float_as_uint(r2.x);
  }
  bool ok = true;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    int fl = (int)((pk >> (10 * a)) & 1023u);
    ok &= lo[a] <= b.ghi[a] && hi[a] >= b.glo[a] && max(fl, b.rlo[a]) == bx[a];
  }
  return ok;
}

struct LatArgs {
  ForestC F;
  GridC g;
  Dirs dirs;
  int nq;
  const int32_t* leaves;
  int64_t n_leaves;
  const float4* rec;
  const int32_t* ab_ids;
  const int32_t* ab_cnt;
  const int32_t* ab_off;
  int32_t* cand_cnt;        // [n_leaves] candidate faces per finest block
  int64_t* cand_off;        // [n_leaves] packed: pair offset << 32 | candidate-block rank
  int32_t* cand_blocks;     // [n_cb] position of each candidate block
  int32_t* pair_face;       // [P] candidate face of each (block, face) pair
  int32_t* pair_blk;        // [P] leaf position of each pair
  int64_t n_pairs;
  uint32_t* star;           // [<= P*C] (pair << shift | cell) passing the star-box test
  unsigned long long* n_star;
  uint32_t* flags;          // [n_leaves * C]
  unsigned* qbits;          // [n_cb * C * nq] min-t float bits (+inf init)
  int32_t* bcount;          // [n_cb]
  const int64_t* boff;      // [n_cb]
  int64_t n_cb;
  int64_t* cells_out;
  float* q_out;
  unsigned long long* stats;  // [0] star-box, [1] link-box, [2] intersection tests
};

template <int D>
__global__ void __launch_bounds__(CNT_WARPS * 32) k_lat_count(LatArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t pos = (int64_t)blockIdx.x * CNT_WARPS + (threadIdx.x >> 5);
  if (pos >= A.n_leaves) return;
  const BlockFrame b = block_frame<D>(A.F, A.g, A.leaves[pos]);
  int count = 0;
  for (int bz = b.rlo[2]; bz <= b.rhi[2]; ++bz)
    for (int by = b.rlo[1]; by <= b.rhi[1]; ++by)
      for (int bx0 = b.rlo[0]; bx0 <= b.rhi[0]; ++bx0) {
        int bx[3] = {bx0, by, bz};
        int64_t lin = bx0 + (int64_t)A.g.B * (by + (int64_t)A.g.B * bz);
        const int32_t* src = A.ab_ids + A.ab_off[lin];
        const int cnt = A.ab_cnt[lin];
        for (int j0 = 0; j0 < cnt; j0 += 32) {
          bool ok = j0 + lane < cnt && is_candidate<D>(A.rec, src[j0 + lane], b, bx);
          count += __popc(__ballot_sync(0xffffffffu, ok));
        }
      }
  if (lane == 0) A.cand_cnt[pos] = count;
}

// one scan gives both the pair offset (high word) and the candidate-block rank (low word)
struct CandLoad {
  const int32_t* c;
  __device__ int64_t operator()(int64_t i) const {
    int64_t n = c[i];
    return (n << 32) | (n > 0 ? 1 : 0);
  }
};
struct CandStore {
  int64_t* off;
  int32_t* blocks;
  __device__ void operator()(int64_t i, int64_t e, int64_t v) const {
    off[i] = e;
    if (v) blocks[e & 0xffffffffll] = (int32_t)i;
  }
};

// warp per candidate block: write its (block, face) pairs
template <int D>
__global__ void __launch_bounds__(CNT_WARPS * 32) k_lat_pairs(LatArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * CNT_WARPS + (threadIdx.x >> 5);
  if (r >= A.n_cb) return;
  const int pos = A.cand_blocks[r];
  const BlockFrame b = block_frame<D>(A.F, A.g, A.leaves[pos]);
  int64_t out = A.cand_off[pos] >> 32;
  for (int bz = b.rlo[2]; bz <= b.rhi[2]; ++bz)
    for (int by = b.rlo[1]; by <= b.rhi[1]; ++by)
      for (int bx0 = b.rlo[0]; bx0 <= b.rhi[0]; ++bx0) {
        int bx[3] = {bx0, by, bz};
        int64_t lin = bx0 + (int64_t)A.g.B * (by + (int64_t)A.g.B * bz);
        const int32_t* src = A.ab_ids + A.ab_off[lin];
        const int cnt = A.ab_cnt[lin];
        for (int j0 = 0; j0 < cnt; j0 += 32) {
          const int f = j0 + lane < cnt ? src[j0 + lane] : 0;
          const bool ok = j0 + lane < cnt && is_candidate<D>(A.rec, f, b, bx);
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          if (ok) {
            const int64_t k = out + __popc(m & lanemask_lt());
            A.pair_face[k] = f;
            A.pair_blk[k] = pos;
          }
          out += __popc(m);
        }
      }
}

// cell centre (FP64 -> one FP32 rounding) and cell size of cell c of block id
template <int D>
__device__ __forceinline__ void cell_center(const ForestC& F, int id, int c, float* x, float* h) {
  const int L = F.level[id];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double q = block_len(F, a, L);
    double o = DADD(F.dmin[a], DMUL((double)F.coord[a][id], q));
    double u = ((double)((c >> (2 * a)) & 3) + 0.5) / 4.0;
    x[a] = __double2float_rn(DADD(o, DMUL(u, q)));
    h[a] = __double2float_rn(q / 4.0);
  }
}

__device__ __forceinline__ void face_lohi(const float4* __restrict__ rec, int f, int D, float* lo, float* hi) {
  if (D == 3) {
    float4 r0 = rec[4 * f], r1 = rec[4 * f + 1], r2 = rec[4 * f + 2], r3 = rec[4 * f + 3];
    lo[0] = r0.w, lo[1] = r1.w, lo[2] = r2.w, hi[0] = r3.x, hi[1] = r3.y, hi[2] = r3.z;
  } else {
    float4 r1 = rec[4 * f + 1];
    lo[0] = r1.x, lo[1] = r1.y, hi[0] = r1.z, hi[1] = r1.w;
  }
}

// (pair, cell) items whose cell "star" box [fl(x-h), fl(x+h)] — the union of
// all its link boxes — meets the face box; appended with warp-aggregated atomics
template <int D>
__global__ void __launch_bounds__(256) k_lat_star(LatArgs A) {
  constexpr int SH = D == 3 ? 6 : 4;  // log2 cells per block
  const int64_t total = A.n_pairs << SH;
  const int lane = threadIdx.x & 31;
  unsigned long long tests = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < total; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = base + threadIdx.x;
    bool ok = false;
    if (t < total) {
      const int64_t p = t >> SH;
      const int c = (int)(t & ((1 << SH) - 1));
      float x[3], h[3], lo[3], hi[3];
      cell_center<D>(A.F, A.leaves[A.pair_blk[p]], c, x, h);
      face_lohi(A.rec, A.pair_face[p], D, lo, hi);
      ok = true;
#pragma unroll
      for (int a = 0; a < D; ++a) ok = ok && lo[a] <= FADD(x[a], h[a]) && hi[a] >= FADD(x[a], -h[a]);
      ++tests;
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (m) {
      unsigned long long w = 0;
      if (lane == 0) w = atomicAdd(A.n_star, (unsigned long long)__popc(m));
      w = __shfl_sync(0xffffffffu, w, 0);
      if (ok) A.star[w + __popc(m & lanemask_lt())] = (uint32_t)t;
    }
  }
  for (int o = 16; o > 0; o >>= 1) tests += __shfl_xor_sync(0xffffffffu, tests, o);
  if (lane == 0 && tests) atomicAdd(&A.stats[0], tests);
}

// Moller-Trumbore, fixed op order (oracle/lattice.py:mt_hits); e1 = v1 - v0,
// e2 = v2 - v0 were formed by the same float32 subtractions at packing time.
__device__ __forceinline__ bool mt_hit_e(const float* x, const float* dv, const float* v0, const float* e1,
                                         const float* e2, float* tout) {
  float px = FSUB(FMUL(dv[1], e2[2]), FMUL(dv[2], e2[1]));
  float py = FSUB(FMUL(dv[2], e2[0]), FMUL(dv[0], e2[2]));
  float pz = FSUB(FMUL(dv[0], e2[1]), FMUL(dv[1], e2[0]));
  float det = dot3f(e1[0], e1[1], e1[2], px, py, pz);
  if (det == 0.0f) return false;
  float tx = FSUB(x[0], v0[0]), ty = FSUB(x[1], v0[1]), tz = FSUB(x[2], v0[2]);
  float u = FDIV(dot3f(tx, ty, tz, px, py, pz), det);
  if (!(u >= 0.0f)) return false;
  float qx = FSUB(FMUL(ty, e1[2]), FMUL(tz, e1[1]));
  float qy = FSUB(FMUL(tz, e1[0]), FMUL(tx, e1[2]));
  float qz = FSUB(FMUL(tx, e1[1]), FMUL(ty, e1[0]));
  float v = FDIV(dot3f(dv[0], dv[1], dv[2], qx, qy, qz), det);
  if (!(v >= 0.0f) || !(FADD(u, v) <= 1.0f)) return false;
  float t = FDIV(dot3f(e2[0], e2[1], e2[2], qx, qy, qz), det);
  if (!(t >= 0.0f) || !(t <= 1.0f)) return false;
  *tout = t;
  return true;
}

// segment-segment (oracle/lattice.py:seg_hits) with s = b - a pre-formed
__device__ __forceinline__ bool seg_hit_s(const float* x, const float* dv, const float* a, const float* sv,
                                          float* tout) {
  float den = FSUB(FMUL(dv[0], sv[1]), FMUL(dv[1], sv[0]));
  if (den == 0.0f) return false;
  float qx = FSUB(a[0], x[0]), qy = FSUB(a[1], x[1]);
  float t = FDIV(FSUB(FMUL(qx, sv[1]), FMUL(qy, sv[0])), den);
  float s = FDIV(FSUB(FMUL(qx, dv[1]), FMUL(qy, dv[0])), den);
  if (!(t >= 0.0f) || !(t <= 1.0f) || !(s >= 0.0f) || !(s <= 1.0f)) return false;
  *tout = t;
  return true;
}

// every link of a (cell, face) item: exact link-AABB test, then the
// intersection test; hits update the cell's flag word and min-t
template <int D>
__global__ void __launch_bounds__(256) k_lat_links(LatArgs A) {
  constexpr int SH = D == 3 ? 6 : 4;
  constexpr int C = 1 << SH;
  const int64_t total = (int64_t)*A.n_star;
  unsigned long long nbox = 0, nmt = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = A.star[e];
    const int64_t p = t >> SH;
    const int c = (int)(t & (C - 1));
    const int pos = A.pair_blk[p], f = A.pair_face[p];
    float x[3], h[3], lo[3], hi[3], v0[3], e1[3], e2[3];
    cell_center<D>(A.F, A.leaves[pos], c, x, h);
    const float4* R = A.rec + 4 * (int64_t)f;
    if (D == 3) {
      float4 r0 = R[0], r1 = R[1], r2 = R[2], r3 = R[3];
      v0[0] = r0.x, v0[1] = r0.y, v0[2] = r0.z, e1[0] = r1.x, e1[1] = r1.y, e1[2] = r1.z;
      e2[0] = r2.x, e2[1] = r2.y, e2[2] = r2.z;
      lo[0] = r0.w, lo[1] = r1.w, lo[2] = r2.w, hi[0] = r3.x, hi[1] = r3.y, hi[2] = r3.z;
    } else {
      float4 r0 = R[0], r1 = R[1];
      v0[0] = r0.x, v0[1] = r0.y, e1[0] = r0.z, e1[1] = r0.w;
      lo[0] = r1.x, lo[1] = r1.y, hi[0] = r1.z, hi[1] = r1.w;
    }
    const int64_t cell = (int64_t)pos * C + c;
    const int64_t qrow = ((int64_t)(A.cand_off[pos] & 0xffffffffll) * C + c) * A.nq;
    unsigned fl = 0;
    for (int d = 1; d < A.nq; ++d) {
      float dv[3];
      bool ov = true;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        dv[a] = FMUL((float)A.dirs.c[d][a], h[a]);  // exact: c in {-1,0,1}
        const float en = FADD(x[a], dv[a]);
        ov = ov && lo[a] <= fmaxf(x[a], en) && hi[a] >= fminf(x[a], en);
      }
      ++nbox;
      if (!ov) continue;
      ++nmt;
      float tt;
      const bool hit = D == 3 ? mt_hit_e(x, dv, v0, e1, e2, &tt) : seg_hit_s(x, dv, v0, e1, &tt);
      if (hit) {
        fl |= 1u << d;
        atomicMin(&A.qbits[qrow + d], __float_as_uint(FADD(tt, 0.0f)));  // -0 -> +0; t >= 0
      }
    }
    if (fl) atomicOr(&A.flags[cell], fl);
  }
  for (int o = 16; o > 0; o >>= 1) {
    nbox += __shfl_xor_sync(0xffffffffu, nbox, o);
    nmt += __shfl_xor_sync(0xffffffffu, nmt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (nbox) atomicAdd(&A.stats[1], nbox);
    if (nmt) atomicAdd(&A.stats[2], nmt);
  }
}

// boundary cells per candidate block (warp per block)
template <int D>
__global__ void k_lat_bcount(LatArgs A) {
  constexpr int C = D == 3 ? 64 : 16;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= A.n_cb) return;
  const int64_t pos = A.cand_blocks[r];
  int nb = 0;
  for (int c = lane; c < C; c += 32) nb += A.flags[pos * C + c] != 0;
  for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
  if (lane == 0) A.bcount[r] = nb;
}

// boundary rows in (block, cell) order: CTA of C threads per candidate block
template <int D>
__global__ void k_lat_emit(LatArgs A) {
  constexpr int C = D == 3 ? 64 : 16;
  const int64_t r = blockIdx.x;
  if (r >= A.n_cb || A.bcount[r] == 0) return;
  const int64_t pos = A.cand_blocks[r];
  const int c = threadIdx.x;
  const unsigned fl = A.flags[pos * C + c];
  __shared__ int s_b[C];
  s_b[c] = fl != 0;
  __syncthreads();
  if (!fl) return;
  int rank = 0;
  for (int c0 = 0; c0 < c; ++c0) rank += s_b[c0];
  const int64_t row = A.boff[r] + rank;
  A.cells_out[row] = pos * C + c;
  const unsigned* q = A.qbits + (r * C + c) * A.nq;
  for (int i = 0; i < A.nq; ++i) A.q_out[row * A.nq + i] = ((fl >> i) & 1) ? __uint_as_float(q[i]) : -1.0f;
}

LatArgs make_args(ow_ctx* ctx, const ow_forest* f, const ow_grid* grid, const int8_t* dirs, int nq,
                  const int32_t* leaves, int64_t n_leaves) {
  LatArgs A;
  memset(&A, 0, sizeof(A));
  A.F = make_forestc(f);
  A.g = make_gridc(grid);
  for (int i = 0; i < nq; ++i)
    for (int a = 0; a < 3; ++a) A.dirs.c[i][a] = a < f->dim ? dirs[i * 3 + a] : 0;
  A.nq = nq;
  A.leaves = leaves;
  A.n_leaves = n_leaves;
  A.rec = (const float4*)ctx->slot_ptr[SLOT_LAT_REC];
  A.ab_ids = (const int32_t*)ctx->slot_ptr[SLOT_ABIN_IDS];
  A.ab_cnt = (const int32_t*)ctx->slot_ptr[SLOT_ABIN_CNT];
  A.ab_off = (const int32_t*)ctx->slot_ptr[SLOT_ABIN_OFF];
  A.cand_cnt = (int32_t*)ctx->slot_ptr[SLOT_LAT_CCNT];
  A.cand_off = (int64_t*)ctx->slot_ptr[SLOT_LAT_COFF];
  A.cand_blocks = (int32_t*)ctx->slot_ptr[SLOT_LAT_LEAVES];
  A.pair_face = (int32_t*)ctx->slot_ptr[SLOT_LAT_PFACE];
  A.pair_blk = (int32_t*)ctx->slot_ptr[SLOT_LAT_PBLK];
  A.star = (uint32_t*)ctx->slot_ptr[SLOT_LAT_STAR];
  A.n_star = (unsigned long long*)(ctx->d_small + 37);
  A.bcount = (int32_t*)ctx->slot_ptr[SLOT_LAT_BCOUNT];
  A.boff = (const int64_t*)ctx->slot_ptr[SLOT_LAT_BOFFS];
  A.qbits = (unsigned*)ctx->slot_ptr[SLOT_LAT_TEMP];
  A.stats = (unsigned long long*)(ctx->d_small + 40);
  A.n_cb = ctx->lat_ncb;
  A.n_pairs = ctx->lat_pairs;
  return A;
}

}  // namespace

extern "C" int ow_lattice_links_count(ow_ctx* ctx, const ow_forest* f, const int32_t* d_leaves, int64_t n_leaves,
                                      const float* d_coords, int64_t n_faces, int64_t geom_key, const ow_grid* grid,
                                      const int8_t* h_dirs, int32_t n_dirs, uint32_t* d_flags, int64_t* out_boundary,
                                      void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n_dirs < 2 || n_dirs > QMAX || !grid || grid->dim != f->dim) {
    ow_set_error("lattice: bad direction set or grid");
    return OW_ERR_INVALID;
  }
  if (n_faces <= 0) {
    ow_set_error("lattice: empty geometry");
    return OW_ERR_INVALID;
  }
  const int D = f->dim, C = D == 3 ? 64 : 16;
  GridC g = make_gridc(grid);
  OW_PROF_BEGIN(ctx, PROF_PREP, s);
  OW_TRY(D == 3 ? build_abins<3>(ctx, g, d_coords, n_faces, geom_key, s)
                : build_abins<2>(ctx, g, d_coords, n_faces, geom_key, s));
  OW_PROF_END(ctx, PROF_PREP, s);
  void* p;
  const int64_t nl = n_leaves > 0 ? n_leaves : 1;
  OW_TRY(ow_slot(ctx, SLOT_LAT_CCNT, 4 * (size_t)nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_COFF, 8 * (size_t)nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_LEAVES, 4 * (size_t)nl, s, &p));
  int8_t dirs3[QMAX * 3];
  memset(dirs3, 0, sizeof(dirs3));
  for (int i = 0; i < n_dirs; ++i)
    for (int a = 0; a < D; ++a) dirs3[i * 3 + a] = h_dirs[i * D + a];
  ctx->lat_leaves = n_leaves;
  ctx->lat_boundary = 0;
  ctx->lat_ncb = 0;
  ctx->lat_pairs = 0;
  ctx->lat_dirs = n_dirs;
  memcpy(ctx->lat_dir, dirs3, sizeof(dirs3));
  ctx->lat_coords = d_coords;
  ctx->lat_faces = n_faces;
  ctx->lat_leaves_ptr = d_leaves;
  ctx->lat_forest = *f;
  ctx->lat_grid = *grid;
  ctx->lat_flags = d_flags;
  *out_boundary = 0;
  OW_CUDA(cudaMemsetAsync(ctx->d_small + 37, 0, 8, s));
  OW_CUDA(cudaMemsetAsync(ctx->d_small + 40, 0, 3 * 8, s));
  if (n_leaves <= 0) return OW_OK;
  OW_PROF_BEGIN(ctx, PROF_LATTICE, s);
  LatArgs A = make_args(ctx, f, grid, dirs3, n_dirs, d_leaves, n_leaves);
  if (D == 3) k_lat_count<3><<<ow_blocks(n_leaves, CNT_WARPS), CNT_WARPS * 32, 0, s>>>(A);
  else k_lat_count<2><<<ow_blocks(n_leaves, CNT_WARPS), CNT_WARPS * 32, 0, s>>>(A);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  OW_TRY(scan(ctx, CandLoad{A.cand_cnt}, CandStore{A.cand_off, A.cand_blocks}, n_leaves, ctx->d_small + 34, s));
  OW_CUDA(cudaMemsetAsync(d_flags, 0, 4 * (size_t)n_leaves * C, s));
  int64_t tot;
  OW_TRY(ow_readback(ctx, ctx->d_small + 34, 1, &tot, s));
  const int64_t n_pairs = tot >> 32, n_cb = tot & 0xffffffffll;
  ctx->lat_ncb = n_cb;
  ctx->lat_pairs = n_pairs;
  if (n_pairs * C >= (int64_t(1) << 32)) {
    ow_set_error("lattice: %lld candidate pairs exceed the 32-bit item encoding", (long long)n_pairs);
    return OW_ERR_CAPACITY;
  }
  if (n_cb > 0) {
    OW_TRY(ow_slot(ctx, SLOT_LAT_PFACE, 4 * (size_t)n_pairs, s, &p));
    OW_TRY(ow_slot(ctx, SLOT_LAT_PBLK, 4 * (size_t)n_pairs, s, &p));
    OW_TRY(ow_slot(ctx, SLOT_LAT_STAR, 4 * (size_t)n_pairs * C, s, &p));
    OW_TRY(ow_slot(ctx, SLOT_LAT_TEMP, 4 * (size_t)n_cb * C * n_dirs, s, &p));
    OW_TRY(ow_slot(ctx, SLOT_LAT_BCOUNT, 4 * (size_t)n_cb, s, &p));
    OW_TRY(ow_slot(ctx, SLOT_LAT_BOFFS, 8 * (size_t)n_cb, s, &p));
    A = make_args(ctx, f, grid, dirs3, n_dirs, d_leaves, n_leaves);
    A.flags = d_flags;
    OW_CUDA(cudaMemsetAsync(A.qbits, 0x7f, 4 * (size_t)n_cb * C * n_dirs, s));  // 3.39e38 > any t <= 1
    OW_PROF_BEGIN(ctx, PROF_LAT_SWEEP, s);
    const int grid_items = 8 * OW_SMS;
    if (D == 3) {
      k_lat_pairs<3><<<ow_blocks(n_cb, CNT_WARPS), CNT_WARPS * 32, 0, s>>>(A);
      k_lat_star<3><<<ow_blocks(n_pairs * C, 256, grid_items), 256, 0, s>>>(A);
      k_lat_links<3><<<grid_items, 256, 0, s>>>(A);
      k_lat_bcount<3><<<ow_blocks(n_cb, 8), 256, 0, s>>>(A);
    } else {
      k_lat_pairs<2><<<ow_blocks(n_cb, CNT_WARPS), CNT_WARPS * 32, 0, s>>>(A);
      k_lat_star<2><<<ow_blocks(n_pairs * C, 256, grid_items), 256, 0, s>>>(A);
      k_lat_links<2><<<grid_items, 256, 0, s>>>(A);
      k_lat_bcount<2><<<ow_blocks(n_cb, 8), 256, 0, s>>>(A);
    }
    OW_PROF_END(ctx, PROF_LAT_SWEEP, s);
    ctx->launches += 4;
    OW_CHECK_LAUNCH();
    OW_TRY(scan(ctx, ow::LoadArr<int32_t>{A.bcount}, ow::StoreExcl<int64_t>{(int64_t*)A.boff}, n_cb,
                ctx->d_small + 35, s));
  } else {
    OW_CUDA(cudaMemsetAsync(ctx->d_small + 35, 0, 8, s));
  }
  OW_PROF_END(ctx, PROF_LATTICE, s);
  int64_t nb;
  OW_TRY(ow_readback(ctx, ctx->d_small + 35, 1, &nb, s));
  ctx->lat_boundary = nb;
  *out_boundary = nb;
  return OW_OK;
}

extern "C" int ow_lattice_links_emit(ow_ctx* ctx, int64_t* d_cells, float* d_q, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (ctx->lat_dirs < 2) {
    ow_set_error("ow_lattice_links_emit without ow_lattice_links_count");
    return OW_ERR_INVALID;
  }
  if (ctx->lat_boundary == 0 || ctx->lat_ncb == 0) return OW_OK;
  LatArgs A = make_args(ctx, &ctx->lat_forest, &ctx->lat_grid, ctx->lat_dir, ctx->lat_dirs, ctx->lat_leaves_ptr,
                        ctx->lat_leaves);
  A.flags = ctx->lat_flags;
  A.cells_out = d_cells;
  A.q_out = d_q;
  const int C = ctx->lat_forest.dim == 3 ? 64 : 16;
  OW_PROF_BEGIN(ctx, PROF_LATTICE, s);
  if (ctx->lat_forest.dim == 3) k_lat_emit<3><<<(unsigned)ctx->lat_ncb, C, 0, s>>>(A);
  else k_lat_emit<2><<<(unsigned)ctx->lat_ncb, C, 0, s>>>(A);
  OW_PROF_END(ctx, PROF_LATTICE, s);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

extern "C" int ow_lattice_stats(ow_ctx* ctx, int64_t* out3, void* stream) {
  return ow_readback(ctx, ctx->d_small + 40, 3, out3, (cudaStream_t)stream);
}
