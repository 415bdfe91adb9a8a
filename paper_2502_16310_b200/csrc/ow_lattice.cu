// Lattice boundary links + wall-distance fractions q on the finest level
// (north-star extension; no reference counterpart, oracle/lattice.py is the
// checker and DESIGN.md §Lattice links the definition).
//
// Candidates come from an AABB-overlap bin CSR (a face is stored in every bin
// its float32 AABB touches), built once per (geometry, grid).  A CTA per
// finest leaf block gathers the faces of the bins under its box grown by two
// cells, visiting each face once (in the first bin of the overlap range), and
// tests every (cell, direction, face) triple: exact float32 link-AABB overlap,
// then Moller-Trumbore (3D) / segment-segment (2D) with a fixed op order.
// Pass 1 writes the per-cell flag words and per-block boundary counts; pass 2
// re-runs the blocks holding boundary cells and writes q rows in cell order.
#include "ow_scan.cuh"
#include <string.h>

namespace {

using ow::scan;

constexpr int LAT_THREADS = 256;
constexpr int LAT_STAGE = 256;
constexpr int QMAX = 27;

struct Dirs {
  int8_t c[QMAX][3];
};

template <int D>
__device__ __forceinline__ void face_box(const float* __restrict__ c, int64_t n, int64_t f, float* lo, float* hi) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float mn = c[(int64_t)a * n + f], mx = mn;
#pragma unroll
    for (int j = 1; j < D; ++j) {
      float x = c[((int64_t)j * D + a) * n + f];
      mn = fminf(mn, x);
      mx = fmaxf(mx, x);
    }
    lo[a] = mn;
    hi[a] = mx;
  }
}

// ---- AABB-overlap bin CSR -------------------------------------------------
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
    float lo[3], hi[3];
    int bl[3], ex[3];
    face_box<D>(c, n, f, lo, hi);
    return abin_range<D>(g, lo, hi, bl, ex);
  }
};

template <int D>
__global__ void k_abin_emit(GridC g, const float* __restrict__ c, int64_t n, const int64_t* foff, uint32_t* keys,
                            int32_t* vals, int32_t* counts) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  float lo[3], hi[3];
  int bl[3], ex[3];
  face_box<D>(c, n, f, lo, hi);
  int64_t v = abin_range<D>(g, lo, hi, bl, ex);
  int64_t pos = foff[f];
  for (int64_t k = 0; k < v; ++k) {
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
  if (key >= 0 && ctx->abin_key == key && ctx->abin_B == g.B && ctx->abin_dim == D) return OW_OK;
  void *pfo, *pcnt, *poff;
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
  OW_CUDA(cudaMemsetAsync(pcnt, 0, 4 * (size_t)nb, s));
  k_abin_emit<D><<<ow_blocks(n, 256), 256, 0, s>>>(g, c, n, (const int64_t*)pfo, (uint32_t*)pk0, (int32_t*)pv0,
                                                  (int32_t*)pcnt);
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

// ---- link kernel -------------------------------------------------------------
struct LatArgs {
  ForestC F;
  GridC g;
  Dirs dirs;
  int nq;
  const int32_t* leaves;
  const float* c;
  int64_t n;
  const int32_t* ab_ids;
  const int32_t* ab_cnt;
  const int32_t* ab_off;
  uint32_t* flags;    // pass 1 out [n_leaves * C]
  int32_t* bcount;    // pass 1 out [n_leaves]
  const int64_t* boff;  // pass 2 in
  int64_t* cells_out;   // pass 2 out
  float* q_out;         // pass 2 out
};

// Moller-Trumbore, fixed op order (oracle/lattice.py:mt_hits)
__device__ __forceinline__ bool mt_hit(const float* x, const float* dv, const float* v0, const float* v1,
                                       const float* v2, float* tout) {
  float e1[3] = {FSUB(v1[0], v0[0]), FSUB(v1[1], v0[1]), FSUB(v1[2], v0[2])};
  float e2[3] = {FSUB(v2[0], v0[0]), FSUB(v2[1], v0[1]), FSUB(v2[2], v0[2])};
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

// segment-segment (oracle/lattice.py:seg_hits)
__device__ __forceinline__ bool seg_hit(const float* x, const float* dv, const float* a, const float* b, float* tout) {
  float sx = FSUB(b[0], a[0]), sy = FSUB(b[1], a[1]);
  float den = FSUB(FMUL(dv[0], sy), FMUL(dv[1], sx));
  if (den == 0.0f) return false;
  float qx = FSUB(a[0], x[0]), qy = FSUB(a[1], x[1]);
  float t = FDIV(FSUB(FMUL(qx, sy), FMUL(qy, sx)), den);
  float s = FDIV(FSUB(FMUL(qx, dv[1]), FMUL(qy, dv[0])), den);
  if (!(t >= 0.0f) || !(t <= 1.0f) || !(s >= 0.0f) || !(s <= 1.0f)) return false;
  *tout = t;
  return true;
}

template <int D, bool EMIT>
__global__ void __launch_bounds__(LAT_THREADS) k_lattice(LatArgs A) {
  constexpr int C = D == 3 ? 64 : 16;
  __shared__ float s_cen[C][D];
  __shared__ float s_h[3];
  __shared__ int s_cand[LAT_STAGE];
  __shared__ int s_ncand;
  __shared__ unsigned s_flag[C];
  __shared__ unsigned s_q[C][QMAX];  // float bits of min t (t >= 0 => int order)
  const ForestC& F = A.F;
  const int64_t pos = blockIdx.x;
  if (EMIT && A.bcount[pos] == 0) return;
  const int id = A.leaves[pos];
  const int L = F.level[id];
  const int tid = threadIdx.x;
  double blo[3], bhi[3], h64[3];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double q = block_len(F, a, L);
    blo[a] = DADD(F.dmin[a], DMUL((double)F.coord[a][id], q));
    bhi[a] = DADD(blo[a], q);
    h64[a] = q / 4.0;  // exact (power-of-two scale)
  }
  if (tid < C) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double q = block_len(F, a, L);
      double u = ((double)((tid >> (2 * a)) & 3) + 0.5) / 4.0;
      s_cen[tid][a] = __double2float_rn(DADD(blo[a], DMUL(u, q)));
    }
    s_flag[tid] = 0u;
    for (int i = 0; i < QMAX; ++i) s_q[tid][i] = 0x7f800000u;  // +inf
  }
  if (tid < D) s_h[tid] = __double2float_rn(h64[tid]);
  // grown block box (two cells) and its bin range, padded by one bin
  double glo[3], ghi[3];
  int rlo[3], rhi[3];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    glo[a] = blo[a] - 2.0 * h64[a];
    ghi[a] = bhi[a] + 2.0 * h64[a];
    rlo[a] = max(bin_axis(__double2float_rd(glo[a]), A.g.min32[a], A.g.len32[a], A.g.B) - 1, 0);
    rhi[a] = min(bin_axis(__double2float_ru(ghi[a]), A.g.min32[a], A.g.len32[a], A.g.B) + 1, A.g.B - 1);
  }
  __syncthreads();
  const int nq = A.nq;
  const int work_cd = C * (nq - 1);
  int bx[3];
  const int nx = rhi[0] - rlo[0] + 1, ny = rhi[1] - rlo[1] + 1, nz = D == 3 ? rhi[2] - rlo[2] + 1 : 1;
  for (int bk = 0; bk < nx * ny * nz; ++bk) {
    bx[0] = rlo[0] + bk % nx;
    bx[1] = rlo[1] + (bk / nx) % ny;
    bx[2] = D == 3 ? rlo[2] + bk / (nx * ny) : 0;
    int64_t lin = bx[0] + (int64_t)A.g.B * (bx[1] + (int64_t)A.g.B * bx[2]);
    const int32_t* src = A.ab_ids + A.ab_off[lin];
    const int cnt = A.ab_cnt[lin];
    for (int base = 0; base < cnt; base += LAT_STAGE) {
      if (tid == 0) s_ncand = 0;
      __syncthreads();
      for (int j = base + tid; j < min(cnt, base + LAT_STAGE); j += LAT_THREADS) {
        int f = src[j];
        float lo[3], hi[3];
        face_box<D>(A.c, A.n, f, lo, hi);
        bool ok = true, first = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          ok &= (double)lo[a] <= ghi[a] && (double)hi[a] >= glo[a];
          // visit the face only in the first bin of (its bin range ∩ ours)
          int fl = max(bin_axis(lo[a], A.g.min32[a], A.g.len32[a], A.g.B), rlo[a]);
          first &= fl == bx[a];
        }
        if (ok && first) s_cand[atomicAdd(&s_ncand, 1)] = f;
      }
      __syncthreads();
      const int ncand = s_ncand;
      for (int k = tid; k < work_cd * ncand; k += LAT_THREADS) {
        int cd = k / ncand, j = k - cd * ncand;
        int ci = cd / (nq - 1), di = 1 + cd % (nq - 1);
        int f = s_cand[j];
        float x[3], dv[3], lo[3], hi[3];
        bool ov = true;
        face_box<D>(A.c, A.n, f, lo, hi);
#pragma unroll
        for (int a = 0; a < D; ++a) {
          x[a] = s_cen[ci][a];
          dv[a] = FMUL((float)A.dirs.c[di][a], s_h[a]);
          float e = FADD(x[a], dv[a]);
          float l = fminf(x[a], e), u = fmaxf(x[a], e);
          ov &= lo[a] <= u && hi[a] >= l;
        }
        if (!ov) continue;
        float v[3][3];
#pragma unroll
        for (int jj = 0; jj < D; ++jj)
#pragma unroll
          for (int a = 0; a < D; ++a) v[jj][a] = A.c[((int64_t)jj * D + a) * A.n + f];
        float t;
        bool hit = D == 3 ? mt_hit(x, dv, v[0], v[1], v[2], &t) : seg_hit(x, dv, v[0], v[1], &t);
        if (hit) {
          t = FADD(t, 0.0f);  // -0 -> +0
          atomicOr(&s_flag[ci], 1u << di);
          if (EMIT) atomicMin(&s_q[ci][di], __float_as_uint(t));
        }
      }
      __syncthreads();
    }
  }
  if (!EMIT) {
    if (tid < C) A.flags[pos * C + tid] = s_flag[tid];
    if (tid < 32) {
      int nb = 0;
      for (int c0 = tid; c0 < C; c0 += 32) nb += s_flag[c0] != 0;
      for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
      if (tid == 0) A.bcount[pos] = nb;
    }
    return;
  }
  // emit rows in cell order
  if (tid < C) {
    unsigned fl = s_flag[tid];
    int rank = 0;
    for (int c0 = 0; c0 < tid; ++c0) rank += s_flag[c0] != 0;
    if (fl) {
      int64_t row = A.boff[pos] + rank;
      A.cells_out[row] = pos * C + tid;
      for (int i = 0; i < nq; ++i)
        A.q_out[row * nq + i] = ((fl >> i) & 1) ? __uint_as_float(s_q[tid][i]) : -1.0f;
    }
  }
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
  GridC g = make_gridc(grid);
  OW_PROF_BEGIN(ctx, PROF_PREP, s);
  OW_TRY(f->dim == 3 ? build_abins<3>(ctx, g, d_coords, n_faces, geom_key, s)
                     : build_abins<2>(ctx, g, d_coords, n_faces, geom_key, s));
  void* pbc;
  OW_TRY(ow_slot(ctx, SLOT_LAT_BCOUNT, 4 * (size_t)(n_leaves + 1), s, &pbc));
  LatArgs A;
  memset(&A, 0, sizeof(A));
  A.F = make_forestc(f);
  A.g = g;
  for (int i = 0; i < n_dirs; ++i)
    for (int a = 0; a < 3; ++a) A.dirs.c[i][a] = a < f->dim ? h_dirs[i * f->dim + a] : 0;
  A.nq = n_dirs;
  A.leaves = d_leaves;
  A.c = d_coords;
  A.n = n_faces;
  A.ab_ids = (const int32_t*)ctx->slot_ptr[SLOT_ABIN_IDS];
  A.ab_cnt = (const int32_t*)ctx->slot_ptr[SLOT_ABIN_CNT];
  A.ab_off = (const int32_t*)ctx->slot_ptr[SLOT_ABIN_OFF];
  A.flags = d_flags;
  A.bcount = (int32_t*)pbc;
  if (n_leaves > 0) {
    OW_PROF_END(ctx, PROF_PREP, s);
    OW_PROF_BEGIN(ctx, PROF_LATTICE, s);
    if (f->dim == 3) k_lattice<3, false><<<(unsigned)n_leaves, LAT_THREADS, 0, s>>>(A);
    else k_lattice<2, false><<<(unsigned)n_leaves, LAT_THREADS, 0, s>>>(A);
    OW_PROF_END(ctx, PROF_LATTICE, s);
    OW_LAUNCHED(ctx);
    OW_CHECK_LAUNCH();
  }
  void* pofs;
  OW_TRY(ow_slot(ctx, SLOT_LAT_LEAVES, 8 * (size_t)(n_leaves + 1), s, &pofs));
  OW_TRY(scan(ctx, ow::LoadArr<int32_t>{(const int32_t*)pbc}, ow::StoreExcl<int64_t>{(int64_t*)pofs}, n_leaves,
              ctx->d_small + 33, s));
  int64_t nb;
  OW_TRY(ow_readback(ctx, ctx->d_small + 33, 1, &nb, s));
  ctx->lat_leaves = n_leaves;
  ctx->lat_boundary = nb;
  ctx->lat_dirs = n_dirs;
  memcpy(ctx->lat_dir, &A.dirs, sizeof(A.dirs) < sizeof(ctx->lat_dir) ? sizeof(A.dirs) : sizeof(ctx->lat_dir));
  ctx->lat_coords = d_coords;
  ctx->lat_faces = n_faces;
  ctx->lat_leaves_ptr = d_leaves;
  ctx->lat_forest = *f;
  ctx->lat_grid = *grid;
  *out_boundary = nb;
  return OW_OK;
}

extern "C" int ow_lattice_links_emit(ow_ctx* ctx, int64_t* d_cells, float* d_q, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (ctx->lat_dirs < 2) {
    ow_set_error("ow_lattice_links_emit without ow_lattice_links_count");
    return OW_ERR_INVALID;
  }
  if (ctx->lat_boundary == 0 || ctx->lat_leaves == 0) return OW_OK;
  LatArgs A;
  memset(&A, 0, sizeof(A));
  A.F = make_forestc(&ctx->lat_forest);
  A.g = make_gridc(&ctx->lat_grid);
  memcpy(&A.dirs, ctx->lat_dir, sizeof(A.dirs) < sizeof(ctx->lat_dir) ? sizeof(A.dirs) : sizeof(ctx->lat_dir));
  A.nq = ctx->lat_dirs;
  A.leaves = ctx->lat_leaves_ptr;
  A.c = ctx->lat_coords;
  A.n = ctx->lat_faces;
  A.ab_ids = (const int32_t*)ctx->slot_ptr[SLOT_ABIN_IDS];
  A.ab_cnt = (const int32_t*)ctx->slot_ptr[SLOT_ABIN_CNT];
  A.ab_off = (const int32_t*)ctx->slot_ptr[SLOT_ABIN_OFF];
  A.bcount = (int32_t*)ctx->slot_ptr[SLOT_LAT_BCOUNT];
  A.boff = (const int64_t*)ctx->slot_ptr[SLOT_LAT_LEAVES];
  A.cells_out = d_cells;
  A.q_out = d_q;
  OW_PROF_BEGIN(ctx, PROF_LATTICE, s);
  if (ctx->lat_forest.dim == 3) k_lattice<3, true><<<(unsigned)ctx->lat_leaves, LAT_THREADS, 0, s>>>(A);
  else k_lattice<2, true><<<(unsigned)ctx->lat_leaves, LAT_THREADS, 0, s>>>(A);
  OW_PROF_END(ctx, PROF_LATTICE, s);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}
