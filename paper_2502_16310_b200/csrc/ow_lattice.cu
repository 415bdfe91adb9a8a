// Lattice boundary links + wall-distance fractions q on the finest level
// (north-star extension; no reference counterpart, oracle/lattice.py is the
// checker and DESIGN.md §5 the definition).
//
// A link (cell, direction d) is tested against face f iff the face's float32
// AABB meets the link's float32 AABB [min(x, x+c_d h), max(x, x+c_d h)].  That
// test is separable per axis and monotone in the cell index along the axis
// (cell centres and fl(x + c h) are non-decreasing in the index), so for one
// (finest block, face) pair the cells whose d-link box meets the face box form
// an axis-aligned sub-box of the 4^D cells: [i0, i0+ext) per axis, one range per
// (axis, c in {-1,0,+1}).  The sweep therefore never tests boxes cell by cell:
//
//   k_lat_pos    : pos_of[leaf id] = leaf position, per-leaf cell-centre table.
//   k_lat_faces  : warp per face; walks the finest-level lattice blocks its box
//                  can reach (root-lattice descent, no bins), computes the
//                  per-axis cell ranges of each existing finest leaf and emits
//                  one row per (leaf, face, direction) with a non-empty cell
//                  box and a non-zero determinant (count pass, then EMIT).
//   scans        : row/unit offsets per face, candidate-block ranks, unit
//                  offsets per row (+ the first row of every MT tile).
//                  Rows are tested inline (warp-flattened (row, cell) units):
//                  the watertight segment-face test (Woop et al. 2013,
//                  oracle/lattice.py:wt_hits) with the oracle's float32 op
//                  order, one division per candidate crossing, deferred to a
//                  per-warp buffer; atomicOr flag bits and a compact hit list.
//   k_lat_mt     : (rows above a tunable size only; not launched by default)
//                  one thread per (row, cell) unit, load-balanced over rows
//                  staged in shared memory, the same test.
//   k_lat_bscan  : boundary cells per candidate block and their row offsets
//                  in (block, cell) order (one look-back scan).
//   k_lat_emit + k_lat_hits : cells, q rows (-1 / min t via atomicMin).
#include "ow_scan.cuh"
#include <stdlib.h>
#include <string.h>

namespace {

using ow::scan;

constexpr int QMAX = 27;
constexpr int MT_THREADS = 256;
constexpr int MT_ITEMS = 2;
constexpr int MT_TILE = MT_THREADS * MT_ITEMS;
constexpr int RU_ROW_BITS = 28;  // rows per pass < 2^28, units < 2^36
constexpr unsigned long long RU_ROW_MASK = (1ull << RU_ROW_BITS) - 1;

// row record: x = leaf position, y = face,
// z = dir | (i0_a | (ext_a-1) << 2) << (5 + 4a), w = units of the row
struct LatArgs {
  ForestC F;
  int nq, level;
  float h[3];               // finest cell size per axis (float32 of the FP64 value)
  float dv[QMAX][3];        // link vectors c_d * h (exact)
  unsigned frame[QMAX];     // watertight frame of direction d: kx | ky << 2 | kz << 4
  float4 shear[QMAX];       // (Sx, Sy, Sz, -) of direction d (float32 divisions, oracle/lattice.py:ray_frame)
  int8_t dc[QMAX][3];       // lattice directions c_d
  uint8_t dir_combo[32];    // combination index sum_a (c_a + 1) 3^a of direction d
  uint8_t combo_dir[27];    // direction of each combination (lattice subset)
  unsigned combo_info[27];  // direction | (4 (c_a + 1)) << (8 + 8a): range-field shifts of a combination
  unsigned dirmask;         // combinations of the lattice's moving directions
  unsigned spread[3][8];    // per-axis non-empty-c mask -> mask over combinations
  const float* coords;
  int64_t n_faces;
  const int32_t* leaves;
  int64_t n_leaves;
  int32_t* pos_of;          // [n_blocks]
  int32_t* grid;            // dense finest-level lattice -> leaf position (-1: no finest leaf), or null
  int gdim[3];              // its extent per axis (root << level)
  int64_t pos_lo, pos_hi;   // leaf positions this call owns (multi-GPU slice)
  float* cen;               // [n_leaves][D][4] cell-centre coordinates
  uint8_t* has_pair;        // [n_leaves]
  float4* rec;              // [n_faces * 3] (v0, e1, e2) / (a, s)
  double q[3];              // finest block size per axis
  double inv_q[3];          // 1 / q
  int4* rows;               // [R]
  int64_t* rowoff;          // [R] units per row -> exclusive unit offsets
  int32_t* tile_row;        // [n_tiles] row of the first unit of each MT tile
  int64_t row_cap, unit_cap;
  unsigned long long* ru_d;       // device (units << RU_ROW_BITS | rows) counter (may exceed the caps)
  int32_t* cand_rank;       // [n_leaves]
  int32_t* cand_blocks;     // [n_cb]
  int64_t n_cb;
  const int64_t* n_cb_d;    // device candidate-block count
  uint32_t* flags;          // [n_leaves * C]
  uint2* hits;              // [<= n_units] (flat cell, t bits)
  uint8_t* hit_dir;         // [<= n_units] direction of each hit
  int32_t* tile_hits;       // [n_tiles] hits of each MT tile
  uint2* ihits;             // [ihit_cap] hits of the rows swept inline by k_lat_faces
  uint8_t* ihit_dir;
  int64_t ihit_cap;
  unsigned long long* ihit_d;  // device inline-hit counter (may exceed the capacity)
  unsigned long long* iru_d;   // inline (units << RU_ROW_BITS | rows), statistics
  int inline_units;            // rows of more cells go to k_lat_mt (OW_INLINE_UNITS overrides; tuning)
  int lane_rows;               // batches whose rows have at most this many cells: a row per lane (0: off)
  int32_t* bcount;          // [n_cb] boundary cells per candidate block
  int32_t* hcount;          // [n_cb] boundary links (set flag bits) per candidate block
  int64_t* hoff;            // [n_cb] packed-q offsets
  unsigned long long* links_d;  // device boundary-link counter (set flag bits)
  unsigned long long* face_next;  // k_lat_faces: next face group (dynamic schedule)
  uint2* rows_out;          // [n_boundary] (cell id, flag word) per boundary row (packed output), or null
  float* qp_out;            // [n_links] q of the set bits, row-major (packed output)
  unsigned long long* bmask;  // [n_cb] boundary-cell mask
  const int64_t* boff;      // [n_cb]
  int64_t* cells_out;
  float* q_out;
  // device-sized pass (ow_lattice_dev_*): the candidate-block count is only on
  // the device, so the emit kernels stride over it and every output write is
  // bounded by the caller's buffers (rows: cells / q / packed rows; links:
  // packed q); a pass that would overflow one is re-run by the host
  int64_t out_row_cap, out_link_cap;
};

// d_small[48..53) = 0 (row / hit / statistics / link counters, face queue)
// and the dense lattice table (int32, slot 16-byte aligned, 4 words per uint4)
// filled with -1
__global__ void k_lat_init(int64_t* counters, uint4* grid, int64_t n4) {
  ow_pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x < 5) counters[threadIdx.x] = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    grid[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
}

template <int D>
__global__ void k_lat_pos(ForestC F, int level, const int32_t* __restrict__ leaves, int64_t n, int32_t* pos_of,
                          uint8_t* has_pair, float* cen, int32_t* grid, int g0, int g1, const int64_t* d_n,
                          uint4* zero_flags, int64_t* widen) {
  ow_pdl_wait();
  if (d_n && *d_n < n) n = *d_n;  // device-sized pass: the leaf count lives on the device
  if (zero_flags)  // ... and the flag words of those leaves are cleared here (no separate fill)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * (D == 3 ? 16 : 4);
         i += (int64_t)gridDim.x * blockDim.x)
      zero_flags[i] = make_uint4(0u, 0u, 0u, 0u);
  double q[3];
#pragma unroll
  for (int a = 0; a < D; ++a) q[a] = block_len(F, a, level);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int id = leaves[i];
    pos_of[id] = (int32_t)i;
    has_pair[i] = 0;
    if (widen) widen[i] = id;  // (device-sized pass: the int64 leaf output)
    if (grid) {  // finest leaves are the blocks of `level` with no children: one lattice cell each
      int64_t lin = F.coord[D - 1][id];
      if (D == 3) lin = lin * g1 + F.coord[1][id];
      grid[lin * g0 + F.coord[0][id]] = (int32_t)i;
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {  // forest.py:187-205: f32(o + u q), u = (i + 1/2) / 4
      const double o = DADD(F.dmin[a], DMUL((double)F.coord[a][id], q[a]));
      float4 v;
      v.x = __double2float_rn(DADD(o, DMUL(0.125, q[a])));
      v.y = __double2float_rn(DADD(o, DMUL(0.375, q[a])));
      v.z = __double2float_rn(DADD(o, DMUL(0.625, q[a])));
      v.w = __double2float_rn(DADD(o, DMUL(0.875, q[a])));
      reinterpret_cast<float4*>(cen)[i * D + a] = v;
    }
  }
}

// Per-axis cell ranges of one (block, face) pair: for c in {-1,0,+1} the
// contiguous set of cell indices i whose link box [min(x_i, e_i), max(x_i, e_i)],
// e_i = fl(x_i + c h), meets [lo, hi] — the per-cell test of oracle/lattice.py
// on the same float32 centres.  Packed in one register: bits [4 ci, 4 ci + 4)
// hold i0 | (ext-1) << 2 of c = ci - 1, bit 12 + ci marks an empty range.
__device__ __forceinline__ unsigned axis_ranges(const float4 x4, float h, float lo, float hi) {
  // e_i = fl(x_i + c h) is >= x_i for c = +1 and <= x_i for c = -1 (h > 0), so
  // the box is [x_i, e_i] / [e_i, x_i] / {x_i} and the two comparisons with x_i
  // are shared by the three directions
  const float x[4] = {x4.x, x4.y, x4.z, x4.w};
  unsigned mm = 0, m0 = 0, mp = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool a = lo <= x[i], b = hi >= x[i];
    mm |= (unsigned)(a && hi >= FADD(x[i], -h)) << i;
    m0 |= (unsigned)(a && b) << i;
    mp |= (unsigned)(lo <= FADD(x[i], h) && b) << i;
  }
  const unsigned m[3] = {mm, m0, mp};
  unsigned r = 0;
#pragma unroll
  for (int ci = 0; ci < 3; ++ci)
    r |= m[ci] == 0 ? (1u << (12 + ci))
                    : (((unsigned)(__ffs(m[ci]) - 1) | ((unsigned)(__popc(m[ci]) - 1) << 2)) << (4 * ci));
  return r;  // contiguous by monotonicity
}

// position of the (n+1)-th set bit of v (n < popc(v)): popc bisection
__device__ __forceinline__ int nth_set_bit(unsigned v, int n) {
  int pos = 0, c;
  c = __popc(v & 0xFFFFu);
  if (n >= c) n -= c, v >>= 16, pos += 16;
  c = __popc(v & 0xFFu);
  if (n >= c) n -= c, v >>= 8, pos += 8;
  c = __popc(v & 0xFu);
  if (n >= c) n -= c, v >>= 4, pos += 4;
  c = __popc(v & 0x3u);
  if (n >= c) n -= c, v >>= 2, pos += 2;
  return pos + (n >= (int)(v & 1u));
}

// row word of direction d from the packed axis ranges (0 when some axis is empty)
template <int D>
__device__ __forceinline__ unsigned row_word(const unsigned* R, const int8_t* c, int d, int* units) {
  unsigned w = (unsigned)d;
  int u = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int ci = c[a] + 1;
    if ((R[a] >> (12 + ci)) & 1u) return 0u;
    const unsigned ra = (R[a] >> (4 * ci)) & 0xFu;
    w |= ra << (5 + 4 * a);
    u *= (int)(ra >> 2) + 1;
  }
  *units = u;
  return w;
}

// Row r of a warp's flattened row list (see k_lat_faces): the owning lane j
// (excl_j <= r < excl_j + popc(valid_j)) is found by a 5-step shuffle search,
// the row is its (r - excl_j)-th set combination.  All lanes must call it
// (shuffles).  Returns (leaf position, face, row word, units); units = 0 past
// the end.
template <int D>
__device__ __forceinline__ int4 row_of(int r, int excl, unsigned valid, const unsigned* R, int pos, int face,
                                       const LatArgs& A) {
  int j = 0;  // last lane with excl <= r
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const int e = __shfl_sync(0xffffffffu, excl, j + step);
    if (e <= r) j += step;
  }
  const unsigned vj = __shfl_sync(0xffffffffu, valid, j);
  const unsigned Rj0 = __shfl_sync(0xffffffffu, R[0], j);
  const unsigned Rj1 = __shfl_sync(0xffffffffu, R[1], j);
  const unsigned Rj2 = __shfl_sync(0xffffffffu, D == 3 ? R[2] : 0u, j);
  const int pj = __shfl_sync(0xffffffffu, pos, j);
  const int fj = __shfl_sync(0xffffffffu, face, j);
  const int ej = __shfl_sync(0xffffffffu, excl, j);
  const int nth = r - ej;
  if (nth < 0 || nth >= __popc(vj)) return make_int4(0, 0, 0, 0);
  const unsigned info = A.combo_info[nth_set_bit(vj, nth)];
  const unsigned Rj[3] = {Rj0, Rj1, Rj2};
  unsigned w = info & 0xFFu;
  int units = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const unsigned ra = (Rj[a] >> ((info >> (8 + 8 * a)) & 0xFFu)) & 0xFu;
    w |= ra << (5 + 4 * a);
    units *= (int)(ra >> 2) + 1;
  }
  return make_int4(pj, fj, (int)w, units);
}

// q = fl(a / det) >= 0 is decided before dividing: it holds iff a is zero, a
// and det agree in sign, or the negative quotient underflows to -0
// (|a / det| <= 2^-150; |a| 2^150 is formed by two exact power-of-two scalings,
// overflow to +inf meaning "not tiny").  A miss never pays for a division and a
// hit gets the quotient bits the oracle computes.
__device__ __forceinline__ bool quot_nonneg(float a, float det) {
  // branch-free: evaluated for every unit of the sweep
  return (a == 0.0f) | ((a > 0.0f) == (det > 0.0f)) | (FMUL(FMUL(fabsf(a), 0x1p75f), 0x1p75f) <= fabsf(det));
}

// x / ext for 0 <= x < 64, ext in 1..4 (multiply-shift, exact in that range)
// (multipliers 256, 128, 86, 64 as packed bytes minus one: one shift and mask
// instead of a compare / select chain)
__device__ __forceinline__ int div_small(int x, int ext) {
  const int m = (int)((0x3F557FFFu >> (8 * (ext - 1))) & 0xFFu) + 1;
  return (x * m) >> 8;
}

// One link-face test, oracle/lattice.py:wt_hits (3D) / wt_hits2 (2D): the
// watertight segment test of Woop, Benthin & Wald (JCGT 2013) with the
// definition's fixed float32 op order.  Per direction a frame (LatArgs.frame:
// kx | ky << 2 | kz << 4, shear Sx, Sy, Sz), the face's vertices translated to
// the link origin (exact: nearby float32 values, Sterbenz) and sheared; the
// three edge functions decide the crossing (recomputed in float64 from the
// same sheared values when one is zero) and only candidate crossings form
// t = T / det.  Face vertices come from shared memory, indexed by the frame's
// axes (no register permutation); the centre by two selects per axis.
struct WtNum {
  float T, det;
};
__device__ __forceinline__ float sel3(float a0, float a1, float a2, unsigned k) {
  return k == 0 ? a0 : (k == 1 ? a1 : a2);
}
// v: 3 vertices x 4 floats (x, y, z, -) in shared memory
__device__ __forceinline__ bool wt_cand3(const float* x, const float* v, unsigned fr, float4 S, WtNum& num) {
  const unsigned kx = fr & 3u, ky = (fr >> 2) & 3u, kz = (fr >> 4) & 3u;
  const float xx = sel3(x[0], x[1], x[2], kx), xy = sel3(x[0], x[1], x[2], ky), xz = sel3(x[0], x[1], x[2], kz);
  float X[3], Y[3], Z[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float az = FSUB(v[4 * j + kz], xz);
    X[j] = FSUB(FSUB(v[4 * j + kx], xx), FMUL(S.x, az));
    Y[j] = FSUB(FSUB(v[4 * j + ky], xy), FMUL(S.y, az));
    Z[j] = az;
  }
  float U = FSUB(FMUL(X[2], Y[1]), FMUL(Y[2], X[1]));
  float V = FSUB(FMUL(X[0], Y[2]), FMUL(Y[0], X[2]));
  float W = FSUB(FMUL(X[1], Y[0]), FMUL(Y[1], X[0]));
  if ((U == 0.0f) | (V == 0.0f) | (W == 0.0f)) {  // exact signs: float products are exact in float64
    U = __double2float_rn(DSUB(DMUL((double)X[2], (double)Y[1]), DMUL((double)Y[2], (double)X[1])));
    V = __double2float_rn(DSUB(DMUL((double)X[0], (double)Y[2]), DMUL((double)Y[0], (double)X[2])));
    W = __double2float_rn(DSUB(DMUL((double)X[1], (double)Y[0]), DMUL((double)Y[1], (double)X[0])));
  }
  const bool mixed = ((U < 0.0f) | (V < 0.0f) | (W < 0.0f)) & ((U > 0.0f) | (V > 0.0f) | (W > 0.0f));
  const float det = FADD(FADD(U, V), W);
  const float T = FADD(FADD(FMUL(U, FMUL(S.z, Z[0])), FMUL(V, FMUL(S.z, Z[1]))), FMUL(W, FMUL(S.z, Z[2])));
  bool c = !mixed & (det != 0.0f) & quot_nonneg(T, det);
  // conservative t <= 1 bound (normal |det|): fl(|T|) > fl(1.00001 |det|)
  // implies |T| / |det| > 1 + 2^-21, hence fl(T / det) > 1
  const float ad = fabsf(det);
  if (ad >= 0x1p-100f) c = c & (fabsf(T) <= FMUL(ad, 1.00001f));
  num.T = T;
  num.det = det;
  return c;
}
__device__ __forceinline__ bool wt_finish(WtNum n, float& t) {
  t = FDIV(n.T, n.det);
  return t <= 1.0f;
}
__device__ __forceinline__ bool wt_test3(const float* x, const float* v, unsigned fr, float4 S, float& t) {
  WtNum n;
  return wt_cand3(x, v, fr, S, n) && wt_finish(n, t);
}
// 2D: v = (a.x, a.y, b.x, b.y); frame kx | kz << 4, S = (Sx, -, Sz)
__device__ __forceinline__ bool wt_test2(const float* x, const float* v, unsigned fr, float4 S, float& t) {
  const unsigned kx = fr & 3u, kz = (fr >> 4) & 3u;
  const float xx = kx ? x[1] : x[0], xz = kz ? x[1] : x[0];
  const float aaz = FSUB(v[kz], xz), baz = FSUB(v[2 + kz], xz);
  const float ax = FSUB(FSUB(v[kx], xx), FMUL(S.x, aaz));
  const float bx = FSUB(FSUB(v[2 + kx], xx), FMUL(S.x, baz));
  const float U = bx, V = -ax;
  const bool mixed = ((U < 0.0f) | (V < 0.0f)) & ((U > 0.0f) | (V > 0.0f));
  const float det = FADD(U, V);
  bool hit = false;
  if (!mixed && det != 0.0f) {
    const float T = FADD(FMUL(U, FMUL(S.z, aaz)), FMUL(V, FMUL(S.z, baz)));
    if (quot_nonneg(T, det)) {
      t = FDIV(T, det);
      hit = t <= 1.0f;
    }
  }
  return hit;
}

// The same tests on operands already permuted to the direction's frame:
// V[j] = (v_j[kx], v_j[ky], v_j[kz], S_j) with (S_0, S_1, S_2) = (Sx, Sy, Sz)
// and the centre (x[kx], x[ky], x[kz]): the oracle's op order, no selects.
__device__ __forceinline__ bool wt_cand_perm(float xx, float xy, float xz, const float4* V, WtNum& num) {
  const float sx = V[0].w, sy = V[1].w, sz = V[2].w;
  float X[3], Y[3], Z[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float az = FSUB(V[j].z, xz);
    X[j] = FSUB(FSUB(V[j].x, xx), FMUL(sx, az));
    Y[j] = FSUB(FSUB(V[j].y, xy), FMUL(sy, az));
    Z[j] = az;
  }
  float U = FSUB(FMUL(X[2], Y[1]), FMUL(Y[2], X[1]));
  float Vv = FSUB(FMUL(X[0], Y[2]), FMUL(Y[0], X[2]));
  float W = FSUB(FMUL(X[1], Y[0]), FMUL(Y[1], X[0]));
  if ((U == 0.0f) | (Vv == 0.0f) | (W == 0.0f)) {  // exact signs: float products are exact in float64
    U = __double2float_rn(DSUB(DMUL((double)X[2], (double)Y[1]), DMUL((double)Y[2], (double)X[1])));
    Vv = __double2float_rn(DSUB(DMUL((double)X[0], (double)Y[2]), DMUL((double)Y[0], (double)X[2])));
    W = __double2float_rn(DSUB(DMUL((double)X[1], (double)Y[0]), DMUL((double)Y[1], (double)X[0])));
  }
  const bool mixed = ((U < 0.0f) | (Vv < 0.0f) | (W < 0.0f)) & ((U > 0.0f) | (Vv > 0.0f) | (W > 0.0f));
  const float det = FADD(FADD(U, Vv), W);
  const float T = FADD(FADD(FMUL(U, FMUL(sz, Z[0])), FMUL(Vv, FMUL(sz, Z[1]))), FMUL(W, FMUL(sz, Z[2])));
  bool c = !mixed & (det != 0.0f) & quot_nonneg(T, det);
  const float ad = fabsf(det);
  if (ad >= 0x1p-100f) c = c & (fabsf(T) <= FMUL(ad, 1.00001f));
  num.T = T;
  num.det = det;
  return c;
}
// 2D: V[j] = (v_j[kx], v_j[kz], -, S) with S = Sx for j = 0 and Sz for j = 1
__device__ __forceinline__ bool wt_test_perm2(float xx, float xz, const float4* V, float& t) {
  const float sx = V[0].w, sz = V[1].w;
  const float aaz = FSUB(V[0].y, xz), baz = FSUB(V[1].y, xz);
  const float ax = FSUB(FSUB(V[0].x, xx), FMUL(sx, aaz));
  const float bx = FSUB(FSUB(V[1].x, xx), FMUL(sx, baz));
  const float U = bx, Vv = -ax;
  const bool mixed = ((U < 0.0f) | (Vv < 0.0f)) & ((U > 0.0f) | (Vv > 0.0f));
  const float det = FADD(U, Vv);
  bool hit = false;
  if (!mixed && det != 0.0f) {
    const float T = FADD(FMUL(U, FMUL(sz, aaz)), FMUL(Vv, FMUL(sz, baz)));
    if (quot_nonneg(T, det)) {
      t = FDIV(T, det);
      hit = t <= 1.0f;
    }
  }
  return hit;
}

// cell index (flat, within the block) and centre of unit `rem` of a row
// word w (cells in x-fastest order over the per-axis ranges)
template <int D>
__device__ __forceinline__ int row_cell(unsigned w, int rem, const float* cen_pos, float* x) {
  int cell = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const unsigned ra = (w >> (5 + 4 * a)) & 0xFu;
    int i;
    if (a + 1 < D) {
      const int ext = (int)(ra >> 2) + 1;
      const int qd = div_small(rem, ext);
      i = (int)(ra & 3u) + (rem - qd * ext);
      rem = qd;
    } else {
      i = (int)(ra & 3u) + rem;  // the last axis takes the quotient as is (rem < ext)
    }
    cell |= i << (2 * a);
    x[a] = __ldg(cen_pos + a * 4 + i);
  }
  return cell;
}

// FACES_PER_WARP faces per warp, SLOT_LANES lanes per face: each lane group
// walks the finest-level lattice blocks its face box can reach (root-lattice
// descent, no bins; link boxes of block k span [o_k - q/8, o_k + 9q/8] and a
// 0.01-block margin absorbs float rounding), computes the per-axis cell ranges
// of each existing finest leaf (the exact filter) and the directions whose
// cell box is non-empty on every axis.  The warp then walks its flattened row
// list 32 rows at a time, reserves rows and units with one packed atomic (row
// order and unit order agree, so unit offsets are monotone without a scan)
// and writes them; rows past the capacities are counted, not written (the
// host re-runs with room).  Links parallel to the face (det == 0) are rejected
// by k_lat_mt.
// (FPW faces per warp is a template parameter: 4 for faces spanning several
// finest blocks, 8 when most faces reach only one or two, see faces_per_warp)
// Rows of at most this many cells are tested inside k_lat_faces; larger ones
// by k_lat_mt.  Measured on C2/C3/C5 (OW_INLINE_UNITS sweep, profiles/): the
// inline sweep wins at every row size, so by default every row is inline
// (64 = 4^3 cells) and k_lat_mt only runs for a lower override.
constexpr int INLINE_UNITS = 64;
constexpr int HITBUF = 64;        // per-warp hit buffer (flushed with one atomic)
constexpr int CANDBUF = 64;       // per-warp candidate buffer (3D: divisions run on full warps)

// a warp's buffered hits -> the inline hit list (one reservation); returns 0
__device__ __forceinline__ int flush_hits(const LatArgs& A, const uint2* hb, const uint8_t* hd, int nh, int lane) {
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(A.ihit_d, (unsigned long long)nh);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int j = lane; j < nh; j += 32)
    if ((int64_t)base + j < A.ihit_cap) {  // past the capacity: counted only (the host re-runs)
      A.ihits[base + j] = hb[j];
      A.ihit_dir[base + j] = hd[j];
    }
  __syncwarp();
  return 0;
}


// record the hits of one warp-wide step (hit / cellg / d per lane)
__device__ __forceinline__ int record_hits(const LatArgs& A, uint2* hb, uint8_t* hd, int nh, bool hit,
                                           unsigned cellg, int d, float t, int lane) {
  const unsigned hm = __ballot_sync(0xffffffffu, hit);
  if (hm) {
    if (nh + __popc(hm) > HITBUF) nh = flush_hits(A, hb, hd, nh, lane);
    if (hit) {
      atomicOr(&A.flags[cellg], 1u << d);
      const int k = nh + __popc(hm & lanemask_lt());
      hb[k] = make_uint2(cellg, __float_as_uint(FADD(t, 0.0f)));  // -0 -> +0
      hd[k] = (uint8_t)d;
    }
    nh += __popc(hm);
    __syncwarp();
  }
  return nh;
}

// divide the top n (<= 32) buffered candidates of a warp, one per lane
__device__ __forceinline__ int drain_cands(const LatArgs& A, const WtNum* cnum, const uint2* cmeta, int nc, int n,
                                           uint2* hb, uint8_t* hd, int nh, int lane) {
  bool hit = false;
  float t = 0.0f;
  uint2 m = make_uint2(0u, 0u);
  if (lane < n) {
    m = cmeta[nc - n + lane];
    hit = wt_finish(cnum[nc - n + lane], t);
  }
  __syncwarp();  // the drained slots are reused by the next pushes
  return record_hits(A, hb, hd, nh, hit, m.x, (int)m.y, t, lane);
}

template <int D, int FPW>
__global__ void __launch_bounds__(128) k_lat_faces(LatArgs A) {
  ow_pdl_wait();
  constexpr int C = D == 3 ? 64 : 16;
  constexpr int FACES_PER_WARP = FPW, SLOT_LANES = 32 / FPW;
  __shared__ float4 s_face[4][FACES_PER_WARP][3];  // per warp: vertices (v0, v1, v2) / (a.xy, b.xy) of its faces
  __shared__ uint2 s_hit[4][HITBUF];
  __shared__ uint8_t s_hdir[4][HITBUF];
  __shared__ unsigned s_frame[QMAX];
  __shared__ float4 s_shear[QMAX];
  // 3D: candidate hits (T, det) + (flat cell, direction), divided 32 at a time
  __shared__ WtNum s_cnum[4][D == 3 ? CANDBUF : 1];
  // the current batch of (<= 32) inline rows, staged in their own frames
  __shared__ int4 s_rmeta[4][32];       // leaf position, first unit, packed box / axes / direction, kx*ky extent
  __shared__ float4 s_rv[4][32][D];     // vertex j along (kx, ky, kz), shear j in .w
  __shared__ float4 s_rc[4][32][D];     // cell centres of the leaf along kx, ky, kz
  __shared__ uint8_t s_rlane[4][32];    // rank of a row with units -> its lane
  __shared__ uint2 s_cmeta[4][D == 3 ? CANDBUF : 1];
  int nc = 0;  // candidates buffered by this warp
  for (int i = threadIdx.x; i < QMAX; i += blockDim.x) {
    s_frame[i] = A.frame[i];
    s_shear[i] = A.shear[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sl = lane % SLOT_LANES;
  int nh = 0;  // hits buffered by this warp
  unsigned long long iru = 0;  // inline units / rows of this warp (statistics)
  // persistent warps take face groups from a global counter: the cost of a
  // face (blocks in reach x rows x cells) varies by orders of magnitude, so
  // dynamic assignment replaces the static one-group-per-warp grid (whose
  // single wave ended in a long tail of a few heavy warps)
  for (;;) {
  unsigned long long grp = 0;
  if (lane == 0) grp = atomicAdd(A.face_next, 1ull);
  grp = __shfl_sync(0xffffffffu, grp, 0);
  const int64_t fbase = (int64_t)grp * FACES_PER_WARP;
  if (fbase >= A.n_faces) break;  // whole warp past the end
  const int64_t f = fbase + lane / SLOT_LANES;
  const bool live = f < A.n_faces;
  float v[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  if (live) {
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int a = 0; a < D; ++a) v[j][a] = A.coords[((int64_t)j * D + a) * A.n_faces + f];
  }
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
  if (live && sl == 0) {  // the face's vertices (the watertight test translates them per link)
    float4 r0, r1 = make_float4(0.0f, 0.0f, 0.0f, 0.0f), r2 = r1;
    if (D == 3) {
      r0 = make_float4(v[0][0], v[0][1], v[0][2], 0.0f);
      r1 = make_float4(v[1][0], v[1][1], v[1][2], 0.0f);
      r2 = make_float4(v[2][0], v[2][1], v[2][2], 0.0f);
    } else {
      r0 = make_float4(v[0][0], v[0][1], v[1][0], v[1][1]);
    }
    if (A.inline_units < C) {  // records for k_lat_mt (no large rows when every row is inline)
      A.rec[3 * f + 0] = r0;
      if (D == 3) {
        A.rec[3 * f + 1] = r1;
        A.rec[3 * f + 2] = r2;
      }
    }
    float4* sf = s_face[wid][lane / SLOT_LANES];
    sf[0] = r0;
    sf[1] = r1;
    sf[2] = r2;
  }
  __syncwarp();
  const int L = A.level;
  int k0[3] = {0, 0, 0}, ext[3] = {1, 1, 1};
  float rext[3] = {1.0f, 1.0f, 1.0f};
  int nslots = live ? 1 : 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int64_t nmax = ((int64_t)A.F.root[a] << L) - 1;
    int64_t a0 = (int64_t)ceil(((double)lo[a] - A.F.dmin[a]) * A.inv_q[a] - 1.135);
    int64_t a1 = (int64_t)floor(((double)hi[a] - A.F.dmin[a]) * A.inv_q[a] + 0.135);
    if (a0 < 0) a0 = 0;
    if (a1 > nmax) a1 = nmax;
    k0[a] = (int)a0;
    ext[a] = a1 >= a0 ? (int)(a1 - a0 + 1) : 0;
    if (a + 1 < D) rext[a] = ext[a] ? __frcp_rn((float)ext[a]) : 0.0f;  // (unused for the last axis)
    nslots *= ext[a];
  }
  const int max_slots = __reduce_max_sync(0xffffffffu, nslots);
  for (int s0 = 0; s0 < max_slots; s0 += SLOT_LANES) {
    const int slot = s0 + sl;
    int nrow = 0, pos = 0;
    unsigned R[3] = {0u, 0u, 0u}, valid = 0u;
    if (slot < nslots) {
      int32_t nc[3] = {0, 0, 0};
      int rem = slot;
#pragma unroll
      for (int a = 0; a < D; ++a) {  // rem / ext by a float reciprocal, corrected to exact
        if (a + 1 == D) {  // last axis: rem < ext
          nc[a] = k0[a] + rem;
          break;
        }
        int qd = (int)(__fmul_rz((float)rem, rext[a]));
        int rr = rem - qd * ext[a];
        while (rr < 0) rr += ext[a], --qd;
        while (rr >= ext[a]) rr -= ext[a], ++qd;
        nc[a] = k0[a] + rr;
        rem = qd;
      }
      // finest leaf at lattice cell nc: one load from the dense lattice table
      // (or the root-lattice descent when the level is too fine for one)
      int pn = -1;
      if (A.grid) {
        int64_t lin = nc[D - 1];
        if (D == 3) lin = lin * A.gdim[1] + nc[1];
        pn = __ldg(A.grid + lin * A.gdim[0] + nc[0]);
      } else {
        int depth;
        const int node = locate(A.F, L, nc, &depth);
        if (depth == L && A.F.first_child[node] < 0) pn = A.pos_of[node];
      }
      // (leaves outside this call's position slice belong to another rank; no
      // early `continue` here: the whole warp must reach the shuffles below)
      if (pn >= 0) {
        if (pn >= A.pos_lo && pn < A.pos_hi) {
          pos = pn;
#pragma unroll
          for (int a = 0; a < D; ++a)
            R[a] = axis_ranges(reinterpret_cast<const float4*>(A.cen)[(int64_t)pos * D + a], A.h[a], lo[a], hi[a]);
          // directions with a non-empty cell box on every axis, as a mask over
          // the 3^D combinations (outer product of the per-axis masks)
          valid = A.dirmask;
#pragma unroll
          for (int a = 0; a < D; ++a) valid &= A.spread[a][(~R[a] >> 12) & 7u];
          nrow = __popc(valid);
          if (nrow) A.has_pair[pos] = 1;
        }
      }
    }
    int incl = nrow;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (!total) continue;
    const int excl = incl - nrow;
    const int fi = (int)f;
    for (int r0 = 0; r0 < total; r0 += 32) {
      const int r = r0 + lane;
      const int4 row = row_of<D>(r, excl, valid, R, pos, fi, A);  // units 0 past the end
      const int units = row.w;
      // rows of more than INLINE_UNITS cells go to k_lat_mt (load-balanced over
      // units): one packed reservation of rows and units per chunk, so row
      // order and unit order agree and unit offsets stay monotone
      const bool big = units > A.inline_units;
      const unsigned bm = __ballot_sync(0xffffffffu, big);
      if (bm) {
        const int ub = big ? units : 0;
        int ui = ub;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, ui, o);
          if (lane >= o) ui += y;
        }
        const unsigned long long tu = (unsigned long long)__shfl_sync(0xffffffffu, ui, 31);
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(A.ru_d, (tu << RU_ROW_BITS) | (unsigned long long)__popc(bm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (big) {
          const int64_t k = (int64_t)(base & RU_ROW_MASK) + __popc(bm & lanemask_lt());
          const int64_t u = (int64_t)(base >> RU_ROW_BITS) + ui - ub;
          if (k < A.row_cap && u + ub <= A.unit_cap) {
            A.rows[k] = row;
            A.rowoff[k] = u;
            for (int64_t t = (u + MT_TILE - 1) / MT_TILE; t * MT_TILE < u + ub; ++t) A.tile_row[t] = (int32_t)k;
          }
        }
      }
      // the other rows: their units flattened over the warp and tested here
      const int us = big ? 0 : units;
      int si = us;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, si, o);
        if (lane >= o) si += y;
      }
      const int S = __shfl_sync(0xffffffffu, si, 31);
      const int se = si - us;
      iru += ((unsigned long long)S << RU_ROW_BITS) + (unsigned long long)__popc(__ballot_sync(0xffffffffu, us > 0));
      if (!S) continue;
      // Batches of short rows (every row at most lane_rows cells: the common
      // case for faces far smaller than the finest blocks) skip the staging
      // below: each lane tests its own row's cells, one per warp step, with
      // the row's frame-permuted vertices and cell box in registers.
      if (D == 3 && A.lane_rows > 0) {
        const int umax = __reduce_max_sync(0xffffffffu, us);
        if (umax <= A.lane_rows) {
          float4 V[3];
          int b0[3] = {0, 0, 0}, e0 = 1, e1 = 1, d = 0;
          unsigned kx = 0, ky = 0, kz = 0;
          const float* cp = A.cen;
          if (us > 0) {
            const unsigned w = (unsigned)row.z;
            d = (int)(w & 31u);
            const unsigned fr = s_frame[d];
            kx = fr & 3u;
            ky = (fr >> 2) & 3u;
            kz = (fr >> 4) & 3u;
            const float* F = reinterpret_cast<const float*>(s_face[wid][row.y - fbase]);
            const float4 sh = s_shear[d];
            V[0] = make_float4(F[kx], F[ky], F[kz], sh.x);
            V[1] = make_float4(F[4 + kx], F[4 + ky], F[4 + kz], sh.y);
            V[2] = make_float4(F[8 + kx], F[8 + ky], F[8 + kz], sh.z);
            const unsigned k3[3] = {kx, ky, kz};
            int ex[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const unsigned ra = (w >> (5 + 4 * k3[q])) & 0xFu;  // i0 | (ext-1) << 2 of axis k3[q]
              b0[q] = (int)(ra & 3u);
              ex[q] = (int)(ra >> 2) + 1;
            }
            e0 = ex[0];
            e1 = ex[1];
            cp = A.cen + (int64_t)row.x * 12;
          } else {
            V[0] = V[1] = V[2] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          }
          for (int k = 0; k < umax; ++k) {
            bool cand = false;
            WtNum num{0.0f, 0.0f};
            unsigned cellg = 0;
            if (k < us) {
              const int q0 = div_small(k, e0);
              const int c0 = b0[0] + (k - q0 * e0);
              const int j2 = div_small(q0, e1);
              const int c1 = b0[1] + (q0 - j2 * e1), c2 = b0[2] + j2;
              const float x0 = __ldg(cp + kx * 4 + c0), x1 = __ldg(cp + ky * 4 + c1), x2 = __ldg(cp + kz * 4 + c2);
              cellg = (unsigned)row.x * (unsigned)C + (unsigned)(c0 << (2 * kx) | c1 << (2 * ky) | c2 << (2 * kz));
              cand = wt_cand_perm(x0, x1, x2, V, num);
            }
            const unsigned cm = __ballot_sync(0xffffffffu, cand);
            if (cm) {
              if (cand) {
                const int kk = nc + __popc(cm & lanemask_lt());
                s_cnum[wid][kk] = num;
                s_cmeta[wid][kk] = make_uint2(cellg, (unsigned)d);
              }
              nc += __popc(cm);
              __syncwarp();
              if (nc >= 32) {
                nh = drain_cands(A, s_cnum[wid], s_cmeta[wid], nc, 32, s_hit[wid], s_hdir[wid], nh, lane);
                nc -= 32;
              }
            }
          }
          continue;
        }
      }
      // Stage the batch's rows in the row's own watertight frame: the face's
      // vertices permuted to (kx, ky, kz) with the shears in .w, the leaf's
      // cell centres per permuted axis, and the cell box along the permuted
      // axes (units run kx-fastest; the order of a row's units is free).  A
      // unit then costs one owner lookup, a few shared loads and the test —
      // no per-unit shuffles, frame selects or global loads.
      const unsigned nzm = __ballot_sync(0xffffffffu, us > 0);
      if (us > 0) {
        const unsigned w = (unsigned)row.z;
        const int d = (int)(w & 31u);
        const unsigned fr = s_frame[d];
        const unsigned kx = fr & 3u, ky = (fr >> 2) & 3u, kz = (fr >> 4) & 3u;
        const unsigned k3[3] = {kx, D == 3 ? ky : kz, kz};  // permuted axis order (2D: kx, kz)
        unsigned pk = (unsigned)d << 26;
        int ext[3] = {1, 1, 1};
#pragma unroll
        for (int q = 0; q < D; ++q) {
          const unsigned ra = (w >> (5 + 4 * k3[q])) & 0xFu;  // i0 | (ext-1) << 2 of axis k3[q]
          ext[q] = (int)(ra >> 2) + 1;
          pk |= (ra & 3u) << (2 * q) | (ra >> 2) << (6 + 2 * q) | k3[q] << (12 + 2 * q);
        }
        s_rmeta[wid][lane] = make_int4(row.x, se, (int)pk, ext[0] * (D == 3 ? ext[1] : 1));
        const float* F = reinterpret_cast<const float*>(s_face[wid][row.y - fbase]);
        const float4 sh = s_shear[d];
        const float shv[3] = {sh.x, sh.y, sh.z};
        const float4* cg = reinterpret_cast<const float4*>(A.cen) + (int64_t)row.x * D;
#pragma unroll
        for (int j = 0; j < D; ++j) {  // vertex j along the permuted axes, shear j in .w
          if (D == 3)
            s_rv[wid][lane][j] = make_float4(F[4 * j + kx], F[4 * j + ky], F[4 * j + kz], shv[j]);
          else
            s_rv[wid][lane][j] = make_float4(F[2 * j + kx], F[2 * j + kz], 0.0f, j ? sh.z : sh.x);
        }
#pragma unroll
        for (int q = 0; q < D; ++q) s_rc[wid][lane][q] = __ldg(cg + k3[q]);
      }
      // rank -> lane of the rows with units (rows are in lane order)
      if (us > 0) s_rlane[wid][__popc(nzm & lanemask_lt())] = (uint8_t)lane;
      __syncwarp();
      int base = 0, carry = 0;  // rows started before the window / the row owning its first unit
      for (int u0 = 0; u0 < S; u0 += 32) {
        const int u = u0 + lane;
        // owner of unit u: the last row starting at or before u (one bit per
        // row start in this 32-unit window)
        const unsigned sb = (us > 0 && se >= u0 && se < u0 + 32) ? 1u << (se - u0) : 0u;
        const unsigned M = __reduce_or_sync(0xffffffffu, sb);
        const int kr = __popc(M & (lanemask_lt() | (1u << lane)));
        const int jl = kr ? (int)s_rlane[wid][base + kr - 1] : carry;
        base += __popc(M);
        carry = M ? (int)s_rlane[wid][base - 1] : carry;
        bool hit = false;
        float t = 0.0f;
        unsigned cellg = 0;
        int d = 0;
        if (D == 3) {
          bool cand = false;
          WtNum num{0.0f, 0.0f};
          if (u < S) {
            const int4 m = s_rmeta[wid][jl];
            const unsigned pk = (unsigned)m.z;
            d = (int)(pk >> 26);
            int k = u - m.y;
            const int e0 = (int)((pk >> 6) & 3u) + 1, e1 = (int)((pk >> 8) & 3u) + 1;
            const int q0 = div_small(k, e0);
            const int j0 = k - q0 * e0;
            const int j2 = div_small(q0, e1);
            const int j1 = q0 - j2 * e1;
            const int c0 = (int)(pk & 3u) + j0, c1 = (int)((pk >> 2) & 3u) + j1, c2 = (int)((pk >> 4) & 3u) + j2;
            const float4* rc = s_rc[wid][jl];
            const float x0 = reinterpret_cast<const float*>(&rc[0])[c0];
            const float x1 = reinterpret_cast<const float*>(&rc[1])[c1];
            const float x2 = reinterpret_cast<const float*>(&rc[2])[c2];
            const int cell = c0 << (2 * ((pk >> 12) & 3u)) | c1 << (2 * ((pk >> 14) & 3u)) | c2 << (2 * ((pk >> 16) & 3u));
            cellg = (unsigned)m.x * (unsigned)C + (unsigned)cell;
            cand = wt_cand_perm(x0, x1, x2, s_rv[wid][jl], num);
          }
          const unsigned cm = __ballot_sync(0xffffffffu, cand);
          if (cm) {
            if (cand) {
              const int k = nc + __popc(cm & lanemask_lt());
              s_cnum[wid][k] = num;
              s_cmeta[wid][k] = make_uint2(cellg, (unsigned)d);
            }
            nc += __popc(cm);
            __syncwarp();
            if (nc >= 32) {  // a full warp of divisions
              nh = drain_cands(A, s_cnum[wid], s_cmeta[wid], nc, 32, s_hit[wid], s_hdir[wid], nh, lane);
              nc -= 32;
            }
          }
        } else {
          if (u < S) {
            const int4 m = s_rmeta[wid][jl];
            const unsigned pk = (unsigned)m.z;
            d = (int)(pk >> 26);
            const int k = u - m.y;
            const int e0 = (int)((pk >> 6) & 3u) + 1;
            const int j1 = div_small(k, e0);
            const int c0 = (int)(pk & 3u) + (k - j1 * e0), c1 = (int)((pk >> 2) & 3u) + j1;
            const float4* rc = s_rc[wid][jl];
            const float xx = reinterpret_cast<const float*>(&rc[0])[c0];
            const float xz = reinterpret_cast<const float*>(&rc[1])[c1];
            const int cell = c0 << (2 * ((pk >> 12) & 3u)) | c1 << (2 * ((pk >> 14) & 3u));
            cellg = (unsigned)m.x * (unsigned)C + (unsigned)cell;
            hit = wt_test_perm2(xx, xz, s_rv[wid][jl], t);
          }
          nh = record_hits(A, s_hit[wid], s_hdir[wid], nh, hit, cellg, d, t, lane);
        }
      }
      __syncwarp();  // the staged rows are rewritten by the next batch
    }
  }
  __syncwarp();  // s_face is rewritten by the next group
  }
  if (D == 3 && nc > 0) nh = drain_cands(A, s_cnum[wid], s_cmeta[wid], nc, nc, s_hit[wid], s_hdir[wid], nh, lane);
  if (nh) flush_hits(A, s_hit[wid], s_hdir[wid], nh, lane);
  if (iru && lane == 0) atomicAdd(A.iru_d, iru);
}

// multi-GPU: after the flag words of every rank's slice are exchanged, the
// candidate blocks are the leaves with a boundary cell (every rank ranks the
// same blocks, so boundary rows are numbered identically everywhere; blocks
// whose rows all missed have no boundary row either way)
template <int D>
__global__ void k_has_from_flags(const uint32_t* __restrict__ flags, int64_t n_leaves, uint8_t* has_pair) {
  ow_pdl_wait();
  constexpr int C = D == 3 ? 64 : 16;
  const int lane = threadIdx.x & 31;
  for (int64_t pos = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; pos < n_leaves;
       pos += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    bool any = false;
#pragma unroll
    for (int k = 0; k < (C + 31) / 32; ++k) any |= (lane + 32 * k < C) && flags[pos * C + lane + 32 * k] != 0u;
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) has_pair[pos] = any ? 1 : 0;
  }
}

// multi-GPU: the q words of this rank's boundary rows (candidate blocks at
// positions [pos_lo, pos_hi), contiguous in row order) -> range[0..1)
__global__ void k_own_q_words(const int32_t* cand_rank, const int64_t* boff, const int64_t* n_cb_d, int64_t n_leaves,
                              int64_t n_boundary, int64_t pos_lo, int64_t pos_hi, int nq, int64_t* range) {
  ow_pdl_wait();
  if (threadIdx.x != 0) return;
  const int64_t ncb = *n_cb_d;
  const int64_t r0 = pos_lo < n_leaves ? cand_rank[pos_lo] : ncb, r1 = pos_hi < n_leaves ? cand_rank[pos_hi] : ncb;
  range[0] = (r0 < ncb ? boff[r0] : n_boundary) * nq;
  range[1] = (r1 < ncb ? boff[r1] : n_boundary) * nq;
}

// ranks of candidate blocks (leaves with at least one row)
struct CandLoad {
  const uint8_t* h;
  __device__ int64_t operator()(int64_t i) const { return h[i]; }
};
struct CandStore {
  int32_t* rank;
  int32_t* blocks;
  __device__ void operator()(int64_t i, int64_t e, int64_t v) const {
    rank[i] = (int32_t)e;
    if (v) blocks[e] = (int32_t)i;
  }
};

// scans bounded by a device-side count (rows / candidate blocks are counted
// on the device; the launch covers the host-known capacity)
struct BcountLoad {
  const int32_t* c;
  const int64_t* n;
  __device__ int64_t operator()(int64_t i) const { return i < *n ? c[i] : 0; }
};
struct BoffStore {
  int64_t* off;
  const int64_t* n;
  __device__ void operator()(int64_t i, int64_t e, int64_t) const {
    if (i < *n) off[i] = e;
  }
};

// Persistent, load-balanced over units: a tile of MT_TILE consecutive units
// covers at most MT_TILE + 1 rows (the first one recorded by the unit scan).
// The tile's rows are staged in shared memory with their face vertices; each
// unit runs the watertight test (oracle/lattice.py:wt_hits / wt_hits2).  Each
// thread binary-searches the row of its first unit and walks forward.
template <int D>
__global__ void __launch_bounds__(MT_THREADS) k_lat_mt(LatArgs A) {
  ow_pdl_wait();
  constexpr int C = D == 3 ? 64 : 16;
  __shared__ int s_off[MT_TILE + 1];
  __shared__ int4 s_meta[MT_TILE + 1];    // pos, face, w, units
  __shared__ float4 s_tri[MT_TILE + 1][3];  // the row's face vertices (2D: (a.xy, b.xy))
  __shared__ unsigned s_frame[QMAX];
  __shared__ float4 s_shear[QMAX];
  __shared__ int s_nh;
  for (int i = threadIdx.x; i < QMAX; i += MT_THREADS) {
    s_frame[i] = A.frame[i];
    s_shear[i] = A.shear[i];
  }
  if (threadIdx.x == 0) s_nh = 0;
  const unsigned long long ru = *A.ru_d;
  const int64_t U = (int64_t)(ru >> RU_ROW_BITS);
  const int64_t R = (int64_t)(ru & RU_ROW_MASK);
  if (R > A.row_cap || U > A.unit_cap) return;  // overflow: the host re-runs with room
  const int64_t n_tiles = (U + MT_TILE - 1) / MT_TILE;
  const int lane = threadIdx.x & 31;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t u0 = tile * MT_TILE;
    const int64_t u1 = min(U, u0 + MT_TILE);
    const int64_t r0 = A.tile_row[tile];
    const int nr = (int)((tile + 1 < n_tiles ? (int64_t)A.tile_row[tile + 1] : R - 1) - r0 + 1);
    __syncthreads();  // previous tile done with the staging buffers (and the frames written)
    for (int i = threadIdx.x; i < nr; i += MT_THREADS) {
      const int4 m = A.rows[r0 + i];
      s_off[i] = (int)(A.rowoff[r0 + i] - u0);  // >= -63 for the first row
      s_meta[i] = m;
      const float4* Rf = A.rec + 3 * (int64_t)m.y;
      s_tri[i][0] = Rf[0];
      if (D == 3) {
        s_tri[i][1] = Rf[1];
        s_tri[i][2] = Rf[2];
      }
    }
    __syncthreads();
    const int ub = threadIdx.x * MT_ITEMS;  // tile-relative
    const int un_tile = (int)(u1 - u0);
    int row = 0;
    if (ub < un_tile) {
      int lo = 0, hi = nr;  // last row with s_off <= ub
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_off[mid] <= ub) lo = mid;
        else hi = mid;
      }
      row = lo;
    }
#pragma unroll
    for (int k = 0; k < MT_ITEMS; ++k) {
      const int u = ub + k;
      bool hit = false;
      int cellg = 0, d = 0;
      float t = 0.0f;
      if (u < un_tile) {
        while (row + 1 < nr && s_off[row + 1] <= u) ++row;
        const int4 m = s_meta[row];
        const unsigned w = (unsigned)m.z;
        d = (int)(w & 31u);
        float x[3];
        const int cell = row_cell<D>(w, u - s_off[row], A.cen + (int64_t)m.x * D * 4, x);
        cellg = m.x * C + cell;
        const float* tv = reinterpret_cast<const float*>(s_tri[row]);
        if (D == 3) hit = wt_test3(x, tv, s_frame[d], s_shear[d], t);
        else hit = wt_test2(x, tv, s_frame[d], s_shear[d], t);
      }
      // hits of this tile go to its own slots [u0, u0 + n) of the hit list
      // (a tile has at most MT_TILE hits): shared-memory append, no global counter
      const unsigned hm = __ballot_sync(0xffffffffu, hit);
      if (hm) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&s_nh, __popc(hm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (hit) {
          atomicOr(&A.flags[cellg], 1u << d);
          const int64_t k = u0 + base + __popc(hm & lanemask_lt());
          A.hits[k] = make_uint2((unsigned)cellg, __float_as_uint(FADD(t, 0.0f)));  // -0 -> +0
          A.hit_dir[k] = (uint8_t)d;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      A.tile_hits[tile] = s_nh;
      s_nh = 0;
    }
  }
}

// Boundary cells of each candidate block and their row offsets in one pass
// (a single-pass scan with decoupled look-back over tiles of 256 candidate
// blocks, ow_scan.cuh): a thread per candidate block reads its flag words
// (16-byte loads, all in flight), forms the boundary-cell mask, the cell
// count and the link count; the tile's counts are scanned and the rows of
// the blocks before it come from the look-back.  Writes bmask / bcount /
// hcount / boff per candidate, the row total into *nb_total and the links
// into A.links_d (one atomic per warp).
constexpr int BSCAN_THREADS = 256;
template <int D>
__global__ void __launch_bounds__(BSCAN_THREADS)
k_lat_bscan(LatArgs A, int64_t* boff, int64_t n_bound, int64_t* nb_total, unsigned long long* status,
            unsigned long long epoch, const unsigned long long* d_epoch_base) {
  ow_pdl_wait();
  if (d_epoch_base) epoch += *d_epoch_base * ow::GRAPH_SITES;  // inside a CUDA graph (ow_graph.cu)
  constexpr int C = D == 3 ? 64 : 16;
  constexpr int W = BSCAN_THREADS / 32;
  __shared__ int64_t s_w[W];
  __shared__ int64_t s_pre;
  const int64_t ncb = *A.n_cb_d < n_bound ? *A.n_cb_d : n_bound;
  const int64_t tile = blockIdx.x;
  if (tile > 0 && tile * BSCAN_THREADS >= ncb) return;  // (past the candidates: nobody looks back here)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = tile * BSCAN_THREADS + threadIdx.x;
  unsigned long long m = 0;
  int links = 0;
  if (r < ncb) {
    const uint4* fp = reinterpret_cast<const uint4*>(A.flags + (int64_t)A.cand_blocks[r] * C);
    uint4 w[C / 4];
#pragma unroll
    for (int k = 0; k < C / 4; ++k) w[k] = fp[k];
#pragma unroll
    for (int k = 0; k < C / 4; ++k) {
      m |= (unsigned long long)((unsigned)(w[k].x != 0u) | (unsigned)(w[k].y != 0u) << 1 |
                                (unsigned)(w[k].z != 0u) << 2 | (unsigned)(w[k].w != 0u) << 3)
           << (4 * k);
      links += __popc(w[k].x) + __popc(w[k].y) + __popc(w[k].z) + __popc(w[k].w);
    }
  }
  const int bc = __popcll(m);
  int x = bc;  // warp inclusive scan of the cell counts
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  const int lsum = __reduce_add_sync(0xffffffffu, links);
  if (lane == 0 && lsum) atomicAdd(A.links_d, (unsigned long long)lsum);
  __syncthreads();
  if (warp == 0) {
    int64_t y = lane < W ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < W; o <<= 1) {
      const int64_t z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    const int64_t agg = __shfl_sync(0xffffffffu, y, W - 1);
    const int64_t wex = y - (lane < W ? s_w[lane] : 0);
    const int64_t prefix = ow::lookback(status, tile, agg, epoch, lane);
    __syncwarp();
    if (lane < W) s_w[lane] = prefix + wex;
    if (lane == 0) s_pre = prefix;
  }
  __syncthreads();
  const int64_t e = s_w[warp] + (x - bc);
  if (r < ncb) {
    boff[r] = e;
    A.bmask[r] = m;
    A.bcount[r] = bc;
    A.hcount[r] = links;
    if (r == ncb - 1) *nb_total = e + bc;
  }
  if (ncb == 0 && threadIdx.x == 0) *nb_total = 0;
  (void)s_pre;
}

// tiles / launch of k_lat_bscan over at most n_bound candidate blocks
template <int D>
int lat_bscan(ow_ctx* ctx, const LatArgs& A, int64_t n_bound, int64_t* nb_total, cudaStream_t s) {
  const int64_t tiles = n_bound > 0 ? (n_bound + BSCAN_THREADS - 1) / BSCAN_THREADS : 1;
  unsigned long long* status;
  unsigned long long epoch;
  OW_TRY(ow::scan_status(ctx, tiles, s, &status, &epoch));
  ow_launch(k_lat_bscan<D>, (unsigned)tiles, BSCAN_THREADS, 0, s, A, (int64_t*)A.boff, n_bound, nb_total, status, epoch,
            (const unsigned long long*)(ctx->capturing ? ctx->d_graph_epoch : nullptr));
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

// boundary rows in (block, cell) order: cells and q rows (-1 where the link
// misses; flagged entries start at +big and receive min t from k_lat_hits).
// CTA per candidate block: the block's q rows are one contiguous run, written
// linearly (coalesced) from the flags staged in shared memory.
// The loop is software-pipelined: the header (mask, block, row offset) of the
// CTA's block two iterations ahead and the flag word of the next one are
// loaded before the current block is written, so the two dependent loads of
// a block overlap the stores of the ones before it.
template <int D>
__global__ void k_lat_emit(LatArgs A) {
  ow_pdl_wait();
  constexpr int C = D == 3 ? 64 : 16;
  __shared__ unsigned s_fl[C];
  const int64_t ncb = *A.n_cb_d;
  const int c = threadIdx.x;
  const int nq = A.nq;
  const int64_t G = gridDim.x;
  struct Hdr {
    unsigned long long m;
    int64_t pos, row0;
  };
  auto header = [&](int64_t r) {
    Hdr h{0ull, 0, 0};
    if (r < ncb) h = Hdr{A.bmask[r], (int64_t)A.cand_blocks[r], A.boff[r]};
    return h;
  };
  auto flag = [&](int64_t r, const Hdr& h) {
    return (r < ncb && ((h.m >> c) & 1ull)) ? A.flags[h.pos * C + c] : 0u;
  };
  int64_t r = blockIdx.x;
  Hdr h0 = header(r), h1 = header(r + G);
  unsigned f0 = flag(r, h0);
  for (; r < ncb; r += G) {
    const Hdr h2 = header(r + 2 * G);  // two blocks ahead
    const unsigned f1 = flag(r + G, h1);  // the next block's flag word
    const unsigned long long m = h0.m;
    const int64_t pos = h0.pos, row0 = h0.row0;
    const int nrow = __popcll(m);
    if (row0 + nrow <= A.out_row_cap) {  // (uniform per CTA; past the cap the host re-runs with room)
      if ((m >> c) & 1ull) {
        const int k = __popcll(m & ((1ull << c) - 1ull));
        s_fl[k] = f0;
        A.cells_out[row0 + k] = pos * C + c;
        if (A.rows_out) A.rows_out[row0 + k] = make_uint2((unsigned)(pos * C + c), f0);
      }
      __syncthreads();
      float* q = A.q_out + row0 * nq;
      for (int i = c; i < nrow * nq; i += C) {
        const int k = i / nq, d = i - k * nq;
        q[i] = ((s_fl[k] >> d) & 1u) ? __uint_as_float(0x7f7f7f7fu) : -1.0f;
      }
      __syncthreads();  // s_fl is rewritten by the next block
    }
    h0 = h1;
    h1 = h2;
    f0 = f1;
  }
}

// min t per (boundary row, direction): t >= 0, so float order = uint order.
// Warp per MT tile over that tile's hit slots.
template <int D>
__global__ void k_lat_hits(LatArgs A) {
  ow_pdl_wait();
  constexpr int C = D == 3 ? 64 : 16;
  const unsigned long long ru = *A.ru_d;
  const int64_t U = (int64_t)(ru >> RU_ROW_BITS);
  if ((int64_t)(ru & RU_ROW_MASK) > A.row_cap || U > A.unit_cap) return;
  const int64_t n_tiles = (U + MT_TILE - 1) / MT_TILE;
  const int lane = threadIdx.x & 31;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_tiles;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int n = A.tile_hits[t];
    for (int j = lane; j < n; j += 32) {
      const int64_t i = t * MT_TILE + j;
      const uint2 h = A.hits[i];
      const int64_t pos = h.x / C;
      const int c = (int)(h.x % C);
      const int r = A.cand_rank[pos];
      const int64_t row = A.boff[r] + __popcll(A.bmask[r] & ((1ull << c) - 1ull));
      if (row < A.out_row_cap) atomicMin(reinterpret_cast<unsigned*>(A.q_out) + row * A.nq + A.hit_dir[i], h.y);
    }
  }
  // hits of the rows swept inline (<= capacity here): HU independent chains
  // (hit -> rank -> row offset / mask -> atomic) in flight per thread
  constexpr int HU = 4;
  const int64_t ni = (int64_t)*A.ihit_d;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < ni; i0 += HU * stride) {
    uint2 h[HU];
    int dir[HU], r[HU];
#pragma unroll
    for (int k = 0; k < HU; ++k) {
      const int64_t i = i0 + k * stride;
      h[k] = i < ni ? A.ihits[i] : make_uint2(0u, 0u);
      dir[k] = i < ni ? A.ihit_dir[i] : 0;
    }
#pragma unroll
    for (int k = 0; k < HU; ++k) r[k] = i0 + k * stride < ni ? A.cand_rank[h[k].x / C] : 0;
#pragma unroll
    for (int k = 0; k < HU; ++k) {
      if (i0 + k * stride >= ni) continue;
      const int c = (int)(h[k].x % C);
      const int64_t row = A.boff[r[k]] + __popcll(A.bmask[r[k]] & ((1ull << c) - 1ull));
      if (row < A.out_row_cap) atomicMin(reinterpret_cast<unsigned*>(A.q_out) + row * A.nq + dir[k], h[k].y);
    }
  }
}

// Packed q (host output): per candidate block (CTA, thread per cell) the q of
// every set flag bit, rows in (block, cell) order and directions ascending
// within a row — q[row][d] for the bits of rows[row].y, concatenated.  With the
// flag words it is the whole result (q = -1 where the bit is clear).
template <int D>
__global__ void k_lat_pack(LatArgs A) {
  ow_pdl_wait();
  constexpr int C = D == 3 ? 64 : 16;
  __shared__ int s_n[2];
  const int64_t ncb = *A.n_cb_d;
  for (int64_t r = blockIdx.x; r < ncb; r += gridDim.x) {
  const unsigned long long m = A.bmask[r];
  const int c = threadIdx.x, lane = c & 31, w = c >> 5;
  if (A.boff[r] + __popcll(m) > A.out_row_cap || A.hoff[r] + A.hcount[r] > A.out_link_cap) continue;  // (uniform)
  const int k = __popcll(m & ((1ull << c) - 1ull));  // row of cell c within the block
  const int64_t row = A.boff[r] + k;
  const unsigned fl = ((m >> c) & 1ull) ? A.rows_out[row].y : 0u;
  constexpr unsigned FULL = C >= 32 ? 0xffffffffu : (1u << C) - 1u;  // 2D: a 16-thread CTA
  int incl = __popc(fl);
#pragma unroll
  for (int o = 1; o < (C < 32 ? C : 32); o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (C > 32) {
    if (lane == 31) s_n[w] = incl;
    __syncthreads();
    if (w == 1) incl += s_n[0];
  }
  int64_t o = A.hoff[r] + incl - __popc(fl);
  const float* q = A.q_out + row * A.nq;
  for (unsigned b = fl; b; b &= b - 1u) A.qp_out[o++] = q[__ffs(b) - 1];
  if (C > 32) __syncthreads();  // s_n is rewritten by the next block
  }
}

// Faces per warp of k_lat_faces: 16 lane pairs when faces are far smaller than
// the finest blocks, 8 lane groups of 4 when they are small (most reach one or
// two blocks per axis), else 4 of 8.
// OW_FACES_PER_WARP overrides (tuning).
int faces_per_warp(const ow_ctx* ctx, int D, int64_t n_faces, int64_t n_leaves) {
  static const int env = [] {
    const char* e = getenv("OW_FACES_PER_WARP");
    return e ? atoi(e) : 0;
  }();
  if (ctx->lat_fpw) return ctx->lat_fpw;
  if (env == 1 || env == 2 || env == 4 || env == 8 || env == 16 || env == 32) return env;
  if (ctx->lat_mean_extent > 0.0f) {  // measured (C2-C5 sweep): 8 wins at 0.17 and 0.28 blocks, 4 at 0.69 and 0.94
    const ow_forest* f = &ctx->lat_forest;
    double q = INFINITY;
    for (int a = 0; a < D; ++a) q = fmin(q, f->dext[a] / (double)((int64_t)f->root[a] << ctx->lat_level));
    // (C5 sweep: 16 faces per warp 1.75 ms vs 8 1.82 vs 32 1.84 at 0.15 blocks;
    // C2 at 0.6-1 blocks: 4 0.098 ms vs 16 0.164)
    const double r = (double)ctx->lat_mean_extent / q;
    // (round 2 sweep, 1/2/4/8/16: C2 0.093 ms at 2 vs 0.098 at 4, C3 0.514 vs 0.528;
    // C4 0.56 at 8; C5 1.75 at 16 vs 1.82 at 8)
    return r < 0.25 ? 16 : (r < 0.5 ? 8 : 2);
  }
  return n_faces > 4 * n_leaves ? 8 : 4;
}

// persistent face pass: resident CTAs only (occupancy of the instantiation,
// queried once: 10 per SM at 48 registers x 128 threads), fewer when the faces
// do not fill them; OW_LAT_CTAS_PER_SM overrides (tuning)
template <int D, int FPW>
unsigned lat_face_grid(int64_t n_faces) {
  static const int per_sm = [] {
    const char* e = getenv("OW_LAT_CTAS_PER_SM");
    if (e && atoi(e) > 0) return atoi(e);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_lat_faces<D, FPW>, 128, 0) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 8;
    }
    return n;
  }();
  const int64_t need = (n_faces + 4 * FPW - 1) / (4 * FPW);
  const int64_t cap = (int64_t)per_sm * OW_SMS;
  return (unsigned)(need < cap ? need : cap);
}

// k_lat_emit: resident CTAs only (32 per SM of 64 / 16 threads), so each CTA
// walks several candidate blocks and its software pipeline has work to
// overlap (OW_LAT_EMIT_CTAS_PER_SM: A/B, 0 = one CTA per candidate block)
unsigned emit_grid(unsigned g) {
  static const int per_sm = [] {
    const char* e = getenv("OW_LAT_EMIT_CTAS_PER_SM");
    return e ? atoi(e) : 32;
  }();
  if (per_sm <= 0) return g;
  const unsigned cap = (unsigned)per_sm * OW_SMS;
  return g < cap ? g : cap;
}

int inline_units_setting(const ow_ctx* ctx) {
  if (ctx->lat_inline_set) return ctx->lat_inline_units;
  static const int v = [] {
    const char* e = getenv("OW_INLINE_UNITS");
    return e ? atoi(e) : INLINE_UNITS;
  }();
  return v;
}

LatArgs make_args(ow_ctx* ctx) {
  LatArgs A;
  memset(&A, 0, sizeof(A));
  const ow_forest* f = &ctx->lat_forest;
  A.F = make_forestc(f);
  A.nq = ctx->lat_dirs;
  A.level = ctx->lat_level;
  for (int a = 0; a < 3; ++a) {
    // float32 of the FP64 cell size, as the device's block_len / 4 (IEEE division both sides)
    A.q[a] = a < f->dim ? f->dext[a] / (double)((int64_t)f->root[a] << A.level) : 1.0;
    A.inv_q[a] = 1.0 / A.q[a];
    A.h[a] = a < f->dim ? (float)(A.q[a] / 4.0) : 0.0f;
  }
  for (int i = 0; i < A.nq; ++i) {
    int ci = 0, mul = 1;
    for (int a = 0; a < 3; ++a) {
      A.dc[i][a] = ctx->lat_dir[i * 3 + a];
      A.dv[i][a] = (float)ctx->lat_dir[i * 3 + a] * A.h[a];  // exact
      if (a < f->dim) {
        ci += (ctx->lat_dir[i * 3 + a] + 1) * mul;
        mul *= 3;
      }
    }
    {  // watertight frame (oracle/lattice.py:ray_frame): kz = first axis of max |dv|
      const int D = f->dim;
      int kz = 0;
      for (int a = 1; a < D; ++a)
        if (fabsf(A.dv[i][a]) > fabsf(A.dv[i][kz])) kz = a;
      int kx, ky = 0;
      if (D == 2) {
        kx = 1 - kz;
      } else {
        kx = (kz + 1) % 3;
        ky = (kz + 2) % 3;
        if (A.dv[i][kz] < 0.0f) {
          const int t = kx;
          kx = ky;
          ky = t;
        }
      }
      A.frame[i] = (unsigned)kx | (unsigned)ky << 2 | (unsigned)kz << 4;
      volatile float dz = A.dv[i][kz];  // (IEEE float32 divisions, as the oracle's)
      if (i > 0) {
        A.shear[i].x = A.dv[i][kx] / dz;
        A.shear[i].y = D == 3 ? A.dv[i][ky] / dz : 0.0f;
        A.shear[i].z = 1.0f / dz;
      }
    }
    A.dir_combo[i] = (uint8_t)ci;
    A.combo_dir[ci] = (uint8_t)i;
    A.combo_info[ci] = (unsigned)i;
    for (int a = 0, cc = ci; a < f->dim; ++a, cc /= 3) A.combo_info[ci] |= (unsigned)(4 * (cc % 3)) << (8 + 8 * a);
    if (i > 0) A.dirmask |= 1u << ci;
  }
  for (int a = 0; a < 3; ++a)
    for (int m = 0; m < 8; ++m) {
      unsigned sp = 0;
      int ncomb = f->dim == 3 ? 27 : 9, div = a == 0 ? 1 : (a == 1 ? 3 : 9);
      for (int c = 0; c < ncomb; ++c)
        if ((m >> ((c / div) % 3)) & 1) sp |= 1u << c;
      A.spread[a][m] = a < f->dim ? sp : 0xffffffffu;
    }
  A.coords = ctx->lat_coords;
  A.n_faces = ctx->lat_faces;
  A.leaves = ctx->lat_leaves_ptr;
  A.n_leaves = ctx->lat_leaves;
  A.pos_lo = ctx->lat_pos_lo;
  A.pos_hi = ctx->lat_pos_hi;
  A.pos_of = (int32_t*)ctx->slot_ptr[SLOT_LAT_POS];
  A.grid = ctx->lat_grid_on ? (int32_t*)ctx->slot_ptr[SLOT_LAT_GRID] : nullptr;
  for (int a = 0; a < 3; ++a) A.gdim[a] = a < f->dim ? (int)((int64_t)f->root[a] << A.level) : 1;
  A.cen = (float*)ctx->slot_ptr[SLOT_LAT_CEN];
  A.has_pair = (uint8_t*)ctx->slot_ptr[SLOT_LAT_HAS];
  A.rec = (float4*)ctx->slot_ptr[SLOT_LAT_REC];
  A.rows = (int4*)ctx->slot_ptr[SLOT_LAT_ROWS];
  A.rowoff = (int64_t*)ctx->slot_ptr[SLOT_LAT_ROWOFF];
  A.tile_row = (int32_t*)ctx->slot_ptr[SLOT_LAT_TILEROW];
  A.row_cap = ctx->lat_row_cap;
  A.unit_cap = ctx->lat_unit_cap;
  A.ru_d = (unsigned long long*)(ctx->d_small + 48);
  A.cand_rank = (int32_t*)ctx->slot_ptr[SLOT_LAT_RANK];
  A.cand_blocks = (int32_t*)ctx->slot_ptr[SLOT_LAT_LEAVES];
  A.n_cb = ctx->lat_ncb;
  A.n_cb_d = ctx->d_small + 33;
  A.flags = ctx->lat_flags;
  A.hits = (uint2*)ctx->slot_ptr[SLOT_LAT_HITS];
  A.hit_dir = (uint8_t*)ctx->slot_ptr[SLOT_LAT_HITDIR];
  A.tile_hits = (int32_t*)ctx->slot_ptr[SLOT_LAT_TILEHITS];
  A.ihits = (uint2*)ctx->slot_ptr[SLOT_LAT_IHITS];
  A.ihit_dir = (uint8_t*)ctx->slot_ptr[SLOT_LAT_IHITDIR];
  A.ihit_cap = ctx->lat_ihit_cap;
  A.ihit_d = (unsigned long long*)(ctx->d_small + 49);
  A.iru_d = (unsigned long long*)(ctx->d_small + 50);
  A.inline_units = inline_units_setting(ctx);
  {
    // batches whose rows all have at most 2 cells skip the staging (A/B on one
    // B200, OW_LAT_LANE_ROWS 0-4, tools/ab_lat.sh: C5 sweep 1.909 -> 1.846 ms
    // at 2, C2 / C3 / C4 within noise; 4 is slower again at C5)
    static const int lr = [] {  // OW_LAT_LANE_ROWS overrides (A/B)
      const char* e = getenv("OW_LAT_LANE_ROWS");
      return e ? atoi(e) : 2;
    }();
    A.lane_rows = lr;
  }
  A.bcount = (int32_t*)ctx->slot_ptr[SLOT_LAT_BCOUNT];
  A.bmask = (unsigned long long*)ctx->slot_ptr[SLOT_LAT_BMASK];
  A.boff = (const int64_t*)ctx->slot_ptr[SLOT_LAT_BOFFS];
  A.hcount = (int32_t*)ctx->slot_ptr[SLOT_LAT_HCOUNT];
  A.hoff = (int64_t*)ctx->slot_ptr[SLOT_LAT_HOFFS];
  A.links_d = (unsigned long long*)(ctx->d_small + 51);
  A.face_next = (unsigned long long*)(ctx->d_small + 52);
  A.out_row_cap = A.out_link_cap = INT64_MAX;
  return A;
}

}  // namespace

extern "C" int ow_lattice_links_count(ow_ctx* ctx, const ow_forest* f, int32_t level, const int32_t* d_leaves,
                                      int64_t n_leaves, const float* d_coords, int64_t n_faces, int64_t geom_key,
                                      const ow_grid* grid, const int8_t* h_dirs, int32_t n_dirs, uint32_t* d_flags,
                                      int64_t* out_boundary, void* stream) {
  return ow_lattice_links_count_range(ctx, f, level, d_leaves, n_leaves, 0, n_leaves, d_coords, n_faces, geom_key,
                                      grid, h_dirs, n_dirs, d_flags, out_boundary, stream);
}

namespace {
// d_nl (device-sized pass, ow_lattice_dev_count): the leaf count is read on the
// device, n_leaves only bounds it (buffers and grids); the flag words are
// cleared by k_lat_pos and nothing is read back (the caller reads the counts
// after the pass and re-runs it on this synchronous path when a capacity was
// short)
int lat_count(ow_ctx* ctx, const ow_forest* f, int32_t level, const int32_t* d_leaves, int64_t n_leaves,
              int64_t pos_lo, int64_t pos_hi, const float* d_coords, int64_t n_faces, int64_t geom_key,
              const ow_grid* grid, const int8_t* h_dirs, int32_t n_dirs, uint32_t* d_flags, int64_t* out_boundary,
              cudaStream_t stream, const int64_t* d_nl, int64_t* widen_out = nullptr) {
  (void)geom_key;
  if (pos_lo < 0 || pos_hi > n_leaves || pos_lo > pos_hi) {
    ow_set_error("lattice: leaf range [%lld, %lld) outside [0, %lld)", (long long)pos_lo, (long long)pos_hi,
                 (long long)n_leaves);
    return OW_ERR_INVALID;
  }
  ctx->lat_pos_lo = pos_lo;
  ctx->lat_pos_hi = pos_hi;
  cudaStream_t s = (cudaStream_t)stream;
  if (n_dirs < 2 || n_dirs > QMAX || (grid && grid->dim != f->dim) || level < 0 || level >= 28) {
    ow_set_error("lattice: bad direction set, grid or level");
    return OW_ERR_INVALID;
  }
  if (n_faces <= 0) {
    ow_set_error("lattice: empty geometry");
    return OW_ERR_INVALID;
  }
  const int D = f->dim, C = D == 3 ? 64 : 16;
  if (n_leaves * C >= (int64_t(1) << 32)) {
    ow_set_error("lattice: %lld finest cells exceed the 32-bit cell index", (long long)(n_leaves * C));
    return OW_ERR_CAPACITY;
  }
  memset(ctx->lat_dir, 0, sizeof(ctx->lat_dir));
  for (int i = 0; i < n_dirs; ++i)
    for (int a = 0; a < D; ++a) ctx->lat_dir[i * 3 + a] = h_dirs[i * D + a];
  ctx->lat_level = level;
  ctx->lat_leaves = n_leaves;
  ctx->lat_boundary = 0;
  ctx->lat_links = 0;
  ctx->lat_ncb = 0;
  ctx->lat_rows = 0;
  ctx->lat_units = 0;
  ctx->lat_dirs = n_dirs;
  ctx->lat_coords = d_coords;
  ctx->lat_faces = n_faces;
  ctx->lat_leaves_ptr = d_leaves;
  ctx->lat_forest = *f;
  ctx->lat_flags = d_flags;
  *out_boundary = 0;
  if (n_leaves <= 0) return OW_OK;
  // row / unit capacities: last pass's sizes + 25 % (first pass: per-face guess);
  // an overflow is detected at the single readback and the pass re-runs
  const int inline_all = inline_units_setting(ctx) >= C;  // no rows for k_lat_mt
  const int64_t rows0 = inline_all ? 1024 : 64 * n_faces + 1024;
  if (ctx->lat_row_cap < rows0) ctx->lat_row_cap = rows0;
  if (ctx->lat_unit_cap < 8 * ctx->lat_row_cap) ctx->lat_unit_cap = 8 * ctx->lat_row_cap;
  if (ctx->lat_ihit_cap < 8 * n_faces + 65536) ctx->lat_ihit_cap = 8 * n_faces + 65536;
  const int64_t rcap = ctx->lat_row_cap, ucap = ctx->lat_unit_cap, icap = ctx->lat_ihit_cap;
  void* p;
  const int64_t nl = n_leaves;
  OW_TRY(ow_slot(ctx, SLOT_LAT_POS, 4 * (size_t)(d_nl ? f->capacity : f->n_blocks), s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_HAS, (size_t)nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_CEN, 16 * (size_t)D * nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_RANK, 4 * (size_t)nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_LEAVES, 4 * (size_t)nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_REC, 48 * (size_t)n_faces, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_ROWS, 16 * (size_t)rcap, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_ROWOFF, 8 * (size_t)rcap, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_TILEROW, 4 * (size_t)(ucap / MT_TILE + 2), s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_HITS, 8 * (size_t)ucap, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_HITDIR, (size_t)ucap, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_TILEHITS, 4 * (size_t)(ucap / MT_TILE + 2), s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_IHITS, 8 * (size_t)icap, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_IHITDIR, (size_t)icap, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_BCOUNT, 4 * (size_t)nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_BMASK, 8 * (size_t)nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_BOFFS, 8 * (size_t)nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_HCOUNT, 4 * (size_t)nl, s, &p));
  OW_TRY(ow_slot(ctx, SLOT_LAT_HOFFS, 8 * (size_t)nl, s, &p));
  {  // dense finest-lattice table when it is at most 2^26 cells (256 MB)
    int64_t cells = 1;
    for (int a = 0; a < D; ++a) cells *= (int64_t)f->root[a] << level;
    ctx->lat_grid_on = cells <= (int64_t(1) << 26) && !getenv("OW_LAT_NO_GRID");
    if (ctx->lat_grid_on) OW_TRY(ow_slot(ctx, SLOT_LAT_GRID, 4 * (size_t)cells, s, &p));
  }
  if (!d_nl) OW_TRY(ow_fill_async(ctx, d_flags, 0, 4 * (size_t)n_leaves * C, s));
  OW_PROF_BEGIN(ctx, PROF_LATTICE, s);
  LatArgs A = make_args(ctx);
  {  // the sweep's counters cleared and the dense lattice table set to -1, one launch
    const int64_t cells = A.grid ? (int64_t)A.gdim[0] * A.gdim[1] * A.gdim[2] : 0;
    ow_launch(k_lat_init, ow_blocks((cells + 3) / 4, 256, 8 * OW_SMS), 256, 0, s, ctx->d_small + 48,
              reinterpret_cast<uint4*>(A.grid), (cells + 3) / 4);
    OW_LAUNCHED(ctx);
  }
  uint4* zf = d_nl ? reinterpret_cast<uint4*>(d_flags) : nullptr;
  if (D == 3) ow_launch(k_lat_pos<3>, ow_blocks(nl, 256, 8 * OW_SMS), 256, 0, s, A.F, level, d_leaves, nl, A.pos_of, A.has_pair, A.cen, A.grid, A.gdim[0], A.gdim[1], d_nl, zf, widen_out);
  else ow_launch(k_lat_pos<2>, ow_blocks(nl, 256, 8 * OW_SMS), 256, 0, s, A.F, level, d_leaves, nl, A.pos_of, A.has_pair, A.cen, A.grid, A.gdim[0], A.gdim[1], d_nl, zf, widen_out);
  // the sweep: k_lat_faces (rows; small rows tested inline) + k_lat_mt (large rows)
  OW_PROF_BEGIN(ctx, PROF_LAT_SWEEP, s);
  const int fpw = faces_per_warp(ctx, D, n_faces, nl);
  if (D == 3) {
    if (fpw == 32) ow_launch(k_lat_faces<3, 32>, lat_face_grid<3, 32>(n_faces), 128, 0, s, A);
    else if (fpw == 16) ow_launch(k_lat_faces<3, 16>, lat_face_grid<3, 16>(n_faces), 128, 0, s, A);
    else if (fpw == 8) ow_launch(k_lat_faces<3, 8>, lat_face_grid<3, 8>(n_faces), 128, 0, s, A);
    else if (fpw == 2) ow_launch(k_lat_faces<3, 2>, lat_face_grid<3, 2>(n_faces), 128, 0, s, A);
    else if (fpw == 1) ow_launch(k_lat_faces<3, 1>, lat_face_grid<3, 1>(n_faces), 128, 0, s, A);
    else ow_launch(k_lat_faces<3, 4>, lat_face_grid<3, 4>(n_faces), 128, 0, s, A);
  } else {
    if (fpw == 8) ow_launch(k_lat_faces<2, 8>, lat_face_grid<2, 8>(n_faces), 128, 0, s, A);
    else ow_launch(k_lat_faces<2, 4>, lat_face_grid<2, 4>(n_faces), 128, 0, s, A);
  }
  ctx->launches += 2;  // (k_lat_pos, the face pass)
  OW_CHECK_LAUNCH();
  const int64_t tiles_max = ucap / MT_TILE + 1;
  if (!inline_all) {  // (every row inline: no k_lat_mt rows, and k_lat_hits sees zero units)
    if (D == 3) ow_launch(k_lat_mt<3>, ow_blocks(tiles_max, 1, 6 * OW_SMS), MT_THREADS, 0, s, A);
    else ow_launch(k_lat_mt<2>, ow_blocks(tiles_max, 1, 6 * OW_SMS), MT_THREADS, 0, s, A);
    OW_LAUNCHED(ctx);
  }
  if (!d_nl && ctx->lat_comm && ctx->lat_comm->world > 1) {
    // multi-GPU: every rank swept the faces against its own leaf slice; the
    // flag words of the slices are all-gathered over peer memory.  A rank
    // whose own sweep outgrew its row / hit buffers re-runs it first (a local
    // decision: it must precede the exchange every rank takes part in)
    int64_t hs[3];
    OW_TRY(ow_readback(ctx, ctx->d_small + 48, 3, hs, s));
    const int64_t r0 = (int64_t)((uint64_t)hs[0] & RU_ROW_MASK), u0 = (int64_t)((uint64_t)hs[0] >> RU_ROW_BITS);
    if (r0 > rcap || u0 > ucap || hs[1] > icap) {
      ctx->lat_row_cap = r0 + r0 / 4 + 1024;
      ctx->lat_unit_cap = u0 + u0 / 4 + 4096;
      if (hs[1] > icap) ctx->lat_ihit_cap = hs[1] + hs[1] / 4 + 65536;
      if (ctx->lat_unit_cap >= (int64_t(1) << 31)) {
        ow_set_error("lattice: %lld link-face tests exceed one pass (2^31)", (long long)u0);
        return OW_ERR_CAPACITY;
      }
      return lat_count(ctx, f, level, d_leaves, n_leaves, pos_lo, pos_hi, d_coords, n_faces, geom_key, grid, h_dirs,
                       n_dirs, d_flags, out_boundary, stream, nullptr);
    }
    OW_TRY(ow_comm_allgather_words(ctx, ctx->lat_comm, d_flags, nullptr, pos_lo * C, pos_hi * C, nullptr, nl * C, s));
    if (D == 3) ow_launch(k_has_from_flags<3>, ow_blocks(nl, 8, 8 * OW_SMS), 256, 0, s, (const uint32_t*)d_flags, nl, A.has_pair);
    else ow_launch(k_has_from_flags<2>, ow_blocks(nl, 8, 8 * OW_SMS), 256, 0, s, (const uint32_t*)d_flags, nl, A.has_pair);
    OW_LAUNCHED(ctx);
  }
  OW_TRY(ow::scan01(ctx, CandLoad{A.has_pair}, CandStore{A.cand_rank, A.cand_blocks}, nl, ctx->d_small + 33, s, d_nl));
  OW_PROF_END(ctx, PROF_LAT_SWEEP, s);
  if (D == 3) OW_TRY(lat_bscan<3>(ctx, A, nl, ctx->d_small + 35, s));
  else OW_TRY(lat_bscan<2>(ctx, A, nl, ctx->d_small + 35, s));
  OW_PROF_END(ctx, PROF_LATTICE, s);
  if (d_nl) return OW_OK;  // (counts checked by the caller after the pass)
  // single readback: candidate blocks, (scan scratch), boundary cells, rows, units, links
  int64_t h[19];
  OW_TRY(ow_readback(ctx, ctx->d_small + 33, 19, h, s));
  const int64_t n_cb = h[0], nb = h[2], n_links = h[18];
  const int64_t n_rows = (int64_t)((uint64_t)h[15] & RU_ROW_MASK), n_units = (int64_t)((uint64_t)h[15] >> RU_ROW_BITS);
  const int64_t n_ihits = h[16];
  if (n_rows >= (int64_t(1) << RU_ROW_BITS) - (int64_t(1) << 20)) {
    ow_set_error("lattice: %lld (block, face, direction) rows exceed one pass", (long long)n_rows);
    return OW_ERR_CAPACITY;
  }
  if (n_rows > rcap || n_units > ucap || n_ihits > icap) {
    ctx->lat_row_cap = n_rows + n_rows / 4 + 1024;
    ctx->lat_unit_cap = n_units + n_units / 4 + 4096;
    if (n_ihits > icap) ctx->lat_ihit_cap = n_ihits + n_ihits / 4 + 65536;
    if (ctx->lat_unit_cap >= (int64_t(1) << 31)) {
      ow_set_error("lattice: %lld link-face tests exceed one pass (2^31)", (long long)n_units);
      return OW_ERR_CAPACITY;
    }
    return lat_count(ctx, f, level, d_leaves, n_leaves, pos_lo, pos_hi, d_coords, n_faces, geom_key, grid, h_dirs,
                     n_dirs, d_flags, out_boundary, stream, nullptr);
  }
  ctx->lat_ncb = n_cb;
  // statistics over both sweeps (rows of k_lat_mt + rows tested inline)
  ctx->lat_rows = n_rows + (int64_t)((uint64_t)h[17] & RU_ROW_MASK);
  ctx->lat_units = n_units + (int64_t)((uint64_t)h[17] >> RU_ROW_BITS);
  ctx->lat_boundary = nb;
  ctx->lat_links = n_links;
  *out_boundary = nb;
  return OW_OK;
}
}  // namespace

extern "C" int ow_lattice_links_count_range(ow_ctx* ctx, const ow_forest* f, int32_t level, const int32_t* d_leaves,
                                            int64_t n_leaves, int64_t pos_lo, int64_t pos_hi, const float* d_coords,
                                            int64_t n_faces, int64_t geom_key, const ow_grid* grid,
                                            const int8_t* h_dirs, int32_t n_dirs, uint32_t* d_flags,
                                            int64_t* out_boundary, void* stream) {
  return lat_count(ctx, f, level, d_leaves, n_leaves, pos_lo, pos_hi, d_coords, n_faces, geom_key, grid, h_dirs,
                   n_dirs, d_flags, out_boundary, (cudaStream_t)stream, nullptr);
}

// Device-sized lattice stage of the fused pass: the finest leaves' count
// *d_nl (<= nl_cap) is on the device; count (no readback) ...
int ow_lattice_dev_count(ow_ctx* ctx, const ow_forest* f, int32_t level, const int32_t* d_leaves, const int64_t* d_nl,
                         int64_t nl_cap, const float* d_coords, int64_t n_faces, const int8_t* h_dirs, int32_t n_dirs,
                         uint32_t* d_flags, cudaStream_t s, int64_t* d_leaves64) {
  int64_t nb = 0;
  // (positions >= nl_cap are rejected by the face pass: a stale leaf position
  // of an earlier pass can then never index past this pass's buffers)
  return lat_count(ctx, f, level, d_leaves, nl_cap, 0, nl_cap, d_coords, n_faces, -1, nullptr, h_dirs, n_dirs, d_flags,
                   &nb, s, d_nl, d_leaves64);
}

// ... then emit with the candidate-block count on the device: persistent grids
// of ncb_grid CTAs, writes bounded by row_cap (cells, q, packed rows) and
// link_cap (packed q).  The caller reads the counts afterwards.
int ow_lattice_dev_emit(ow_ctx* ctx, int64_t* d_cells, float* d_q, int64_t row_cap, uint32_t* d_rows,
                        float* d_q_packed, int64_t link_cap, int64_t ncb_grid, cudaStream_t s) {
  LatArgs A = make_args(ctx);
  A.cells_out = d_cells;
  A.q_out = d_q;
  A.rows_out = reinterpret_cast<uint2*>(d_rows);
  A.qp_out = d_q_packed;
  A.out_row_cap = row_cap;
  A.out_link_cap = link_cap;
  const int C = ctx->lat_forest.dim == 3 ? 64 : 16;
  const int64_t nl = ctx->lat_leaves;  // (the bound)
  const unsigned g = (unsigned)(ncb_grid < 1 ? 1 : (ncb_grid > nl ? (nl > 0 ? nl : 1) : ncb_grid));
  OW_PROF_BEGIN(ctx, PROF_LATTICE, s);
  if (d_q_packed)
    OW_TRY(scan(ctx, BcountLoad{A.hcount, A.n_cb_d}, BoffStore{A.hoff, A.n_cb_d}, nl, ctx->d_small + 36, s));
  if (ctx->lat_forest.dim == 3) {
    ow_launch(k_lat_emit<3>, emit_grid(g), C, 0, s, A);
    ow_launch(k_lat_hits<3>, 8 * OW_SMS, 256, 0, s, A);
    if (d_q_packed) ow_launch(k_lat_pack<3>, g, C, 0, s, A);
  } else {
    ow_launch(k_lat_emit<2>, emit_grid(g), C, 0, s, A);
    ow_launch(k_lat_hits<2>, 8 * OW_SMS, 256, 0, s, A);
    if (d_q_packed) ow_launch(k_lat_pack<2>, g, C, 0, s, A);
  }
  OW_PROF_END(ctx, PROF_LATTICE, s);
  ctx->launches += d_q_packed ? 3 : 2;
  OW_CHECK_LAUNCH();
  return OW_OK;
}

extern "C" int ow_lattice_links_emit(ow_ctx* ctx, int64_t* d_cells, float* d_q, void* stream) {
  return ow_lattice_links_emit_packed(ctx, d_cells, d_q, nullptr, nullptr, stream);
}

extern "C" int ow_lattice_links_emit_packed(ow_ctx* ctx, int64_t* d_cells, float* d_q, uint32_t* d_rows,
                                            float* d_q_packed, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if ((d_rows == nullptr) != (d_q_packed == nullptr)) {
    ow_set_error("ow_lattice_links_emit_packed: packed rows and packed q go together");
    return OW_ERR_INVALID;
  }
  if (ctx->lat_dirs < 2) {
    ow_set_error("ow_lattice_links_emit without ow_lattice_links_count");
    return OW_ERR_INVALID;
  }
  if (ctx->lat_boundary == 0 || ctx->lat_ncb == 0) return OW_OK;
  LatArgs A = make_args(ctx);
  A.cells_out = d_cells;
  A.q_out = d_q;
  A.rows_out = reinterpret_cast<uint2*>(d_rows);
  A.qp_out = d_q_packed;
  const int C = ctx->lat_forest.dim == 3 ? 64 : 16;
  OW_PROF_BEGIN(ctx, PROF_LATTICE, s);
  if (d_q_packed)  // packed-q offsets per candidate block (host-known count: no device bound)
    OW_TRY(scan(ctx, ow::LoadArr<int32_t>{A.hcount}, ow::StoreExcl<int64_t>{A.hoff}, ctx->lat_ncb,
                ctx->d_small + 36, s));
  if (ctx->lat_forest.dim == 3) {
    ow_launch(k_lat_emit<3>, emit_grid((unsigned)ctx->lat_ncb), C, 0, s, A);
    ow_launch(k_lat_hits<3>, 8 * OW_SMS, 256, 0, s, A);
  } else {
    ow_launch(k_lat_emit<2>, emit_grid((unsigned)ctx->lat_ncb), C, 0, s, A);
    ow_launch(k_lat_hits<2>, 8 * OW_SMS, 256, 0, s, A);
  }
  if (ctx->lat_comm && ctx->lat_comm->world > 1) {
    // multi-GPU: a rank's hits fill the q rows of its own slice only; the
    // rows are all-gathered over peer memory (row order = leaf order)
    int64_t* range = ctx->d_small + 40;
    ow_launch(k_own_q_words, 1, 32, 0, s, (const int32_t*)A.cand_rank, A.boff, A.n_cb_d, ctx->lat_leaves,
              ctx->lat_boundary, ctx->lat_pos_lo, ctx->lat_pos_hi, A.nq, range);
    OW_LAUNCHED(ctx);
    OW_TRY(ow_comm_allgather_words(ctx, ctx->lat_comm, reinterpret_cast<uint32_t*>(d_q), range, 0, 0, nullptr,
                                   ctx->lat_boundary * A.nq, s));
  }
  if (d_q_packed) {
    if (ctx->lat_forest.dim == 3) ow_launch(k_lat_pack<3>, (unsigned)ctx->lat_ncb, C, 0, s, A);
    else ow_launch(k_lat_pack<2>, (unsigned)ctx->lat_ncb, C, 0, s, A);
  }
  OW_PROF_END(ctx, PROF_LATTICE, s);
  ctx->launches += d_q_packed ? 3 : 2;
  OW_CHECK_LAUNCH();
  return OW_OK;
}

// Tuning / testing knobs: rows of more than `inline_units` cells are tested by
// k_lat_mt, the others inside k_lat_faces; faces_per_warp 4 or 8 fixes the
// face-pass shape.  Negative values restore the defaults.
extern "C" int ow_lattice_tune(ow_ctx* ctx, int32_t inline_units, int32_t faces_per_warp) {
  if (faces_per_warp > 0 && faces_per_warp != 1 && faces_per_warp != 2 && faces_per_warp != 4 &&
      faces_per_warp != 8 && faces_per_warp != 16 && faces_per_warp != 32) {
    ow_set_error("lattice: faces_per_warp must be 1, 2, 4, 8, 16 or 32, got %d", faces_per_warp);
    return OW_ERR_INVALID;
  }
  ctx->lat_inline_set = inline_units >= 0;
  ctx->lat_inline_units = inline_units;
  ctx->lat_fpw = faces_per_warp > 0 ? faces_per_warp : 0;
  return OW_OK;
}

// boundary links (set flag bits) of the last count pass = packed-q length
extern "C" int ow_lattice_links_n_links(ow_ctx* ctx, int64_t* out) {
  *out = ctx->lat_links;
  return OW_OK;
}

// [0] candidate blocks, [1] (block, face, direction) rows, [2] intersection tests
extern "C" int ow_lattice_stats(ow_ctx* ctx, int64_t* out3, void* stream) {
  (void)stream;
  out3[0] = ctx->lat_ncb;
  out3[1] = ctx->lat_rows;
  out3[2] = ctx->lat_units;
  return OW_OK;
}
