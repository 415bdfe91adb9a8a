// FP32 near-face predicate (Algorithm 1 of arXiv 2502.16310) with the
// reference's exact operation order: octowall/distance.py:167-245.
//
// Per-face terms (unit normal, unit edges, slab anchors v0 -+ d*n) are
// precomputed once per (geometry, d) by k_face_prep with the same float32
// operations the reference evaluates per pair; the cheap ones (edge vectors,
// squared edge lengths, in-plane edge normals n x e_k) are re-formed per pair
// from the stored operands by the same operations.  Either way each term is a
// pure function of the face and d, so the predicate is bit-identical to the
// per-pair evaluation.  Per pair the predicate costs 130 FP32 operations (3
// IEEE divisions), SURVEY.md §8(d).
#pragma once

#include "ow_common.cuh"

// payload float4 layout (3D, 7 x float4 = 112 B per face):
//  [k]     k=0..2 : v_k.xyz, n_k            (v_k vertex; unit normal component k)
//  [3+k]          : eh_k.xyz, alo_k         (eh_k = e_k/|e_k|, e_k = v_{k+1}-v_k; alo = v0 - d*n)
//  [6]            : ahi.xyz, 0              (ahi = v0 + d*n)
// (e_k, |e_k|^2 and m_k = n x eh_k are re-formed by near_tri: 51 FP32
// operations per pair instead of 80 B more per face written by k_face_prep and
// read by every evaluated pair; C5 writes 5.2 M payloads per pass)
// 2D (3 x float4 = 48 B): [a.xy b.xy] [e.xy el2 0] [eh.xy 0 0]
constexpr int PAY3 = 7;
constexpr int PAY2 = 3;

// in-plane edge normal m = n x eh (distance.py:203-205), the op order of the
// reference's np.cross
__device__ __forceinline__ void edge_normal(const float* nn, float ex, float ey, float ez, float* m) {
  m[0] = FSUB(FMUL(nn[1], ez), FMUL(nn[2], ey));
  m[1] = FSUB(FMUL(nn[2], ex), FMUL(nn[0], ez));
  m[2] = FSUB(FMUL(nn[0], ey), FMUL(nn[1], ex));
}

template <int D>
__device__ __forceinline__ void face_prep_one(const float* __restrict__ c, int64_t n, int64_t f, float d,
                                              float4* pay) {
  if (D == 3) {
    float v[3][3];
    for (int j = 0; j < 3; ++j)
      for (int a = 0; a < 3; ++a) v[j][a] = c[((int64_t)j * 3 + a) * n + f];
    float e[3][3], el2[3], eh[3][3];
    for (int k = 0; k < 3; ++k) {
      const float* A = v[k];
      const float* B = v[(k + 1) % 3];
      for (int a = 0; a < 3; ++a) e[k][a] = FSUB(B[a], A[a]);
      el2[k] = dot3f(e[k][0], e[k][1], e[k][2], e[k][0], e[k][1], e[k][2]);
      float el = FSQRT(el2[k]);
      for (int a = 0; a < 3; ++a) eh[k][a] = FDIV(e[k][a], el);
    }
    // unit normal, distance.py:238-245 (u = v1 - v0, w = v2 - v0)
    float ux = FSUB(v[1][0], v[0][0]), uy = FSUB(v[1][1], v[0][1]), uz = FSUB(v[1][2], v[0][2]);
    float wx = FSUB(v[2][0], v[0][0]), wy = FSUB(v[2][1], v[0][1]), wz = FSUB(v[2][2], v[0][2]);
    float nx = FSUB(FMUL(uy, wz), FMUL(uz, wy));
    float ny = FSUB(FMUL(uz, wx), FMUL(ux, wz));
    float nz = FSUB(FMUL(ux, wy), FMUL(uy, wx));
    float nl = FSQRT(dot3f(nx, ny, nz, nx, ny, nz));
    float nn[3] = {FDIV(nx, nl), FDIV(ny, nl), FDIV(nz, nl)};
    float alo[3], ahi[3];
    for (int a = 0; a < 3; ++a) {  // distance.py:210-211: (a - d*n), (a + d*n)
      alo[a] = FSUB(v[0][a], FMUL(d, nn[a]));
      ahi[a] = FADD(v[0][a], FMUL(d, nn[a]));
    }
    for (int k = 0; k < 3; ++k) {
      pay[k] = make_float4(v[k][0], v[k][1], v[k][2], nn[k]);
      pay[3 + k] = make_float4(eh[k][0], eh[k][1], eh[k][2], alo[k]);
    }
    pay[6] = make_float4(ahi[0], ahi[1], ahi[2], 0.0f);
  } else {
    float ax = c[0 * n + f], ay = c[1 * n + f], bx = c[2 * n + f], by = c[3 * n + f];
    float ex = FSUB(bx, ax), ey = FSUB(by, ay);
    float el2 = FADD(FMUL(ex, ex), FMUL(ey, ey));
    float el = FSQRT(el2);
    pay[0] = make_float4(ax, ay, bx, by);
    pay[1] = make_float4(ex, ey, el2, 0.0f);
    pay[2] = make_float4(FDIV(ex, el), FDIV(ey, el), 0.0f, 0.0f);
  }
}

// 3D predicate on a prepared face; r2 = d*d (float32).
__device__ __forceinline__ bool near_tri(const float4* __restrict__ P, float px, float py, float pz, float r2) {
  float4 V[3], H[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    V[k] = P[k];
    H[k] = P[3 + k];
  }
  const float4 AH = P[6];
  const float nn[3] = {V[0].w, V[1].w, V[2].w};
  float w[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    w[k][0] = FSUB(V[k].x, px);
    w[k][1] = FSUB(V[k].y, py);
    w[k][2] = FSUB(V[k].z, pz);
  }
  bool hit = false;
  bool inside = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float* W = w[k];
    const float* Wn = w[(k + 1) % 3];  // b - p, identical to the reference's (bx - px)
    const float4 Vn = V[(k + 1) % 3];
    // edge vector and squared length, k_face_prep's operations (v_{k+1} - v_k)
    float ex = FSUB(Vn.x, V[k].x), ey = FSUB(Vn.y, V[k].y), ez = FSUB(Vn.z, V[k].z);
    float el2 = dot3f(ex, ey, ez, ex, ey, ez);
    float ball = dot3f(W[0], W[1], W[2], W[0], W[1], W[2]);
    float cx = FSUB(FMUL(ey, W[2]), FMUL(ez, W[1]));
    float cy = FSUB(FMUL(ez, W[0]), FMUL(ex, W[2]));
    float cz = FSUB(FMUL(ex, W[1]), FMUL(ey, W[0]));
    float d2 = FDIV(dot3f(cx, cy, cz, cx, cy, cz), el2);
    float de1 = -dot3f(W[0], W[1], W[2], H[k].x, H[k].y, H[k].z);
    float de2 = dot3f(Wn[0], Wn[1], Wn[2], H[k].x, H[k].y, H[k].z);
    hit |= (ball <= r2) | ((d2 <= r2) & (de1 >= 0.0f) & (de2 >= 0.0f));
    // prism interior: (p - a_k) . m_k >= 0, with p - a_k == -(a_k - p) exactly
    float m[3];
    edge_normal(nn, H[k].x, H[k].y, H[k].z, m);
    inside &= -dot3f(W[0], W[1], W[2], m[0], m[1], m[2]) >= 0.0f;
  }
  float lo = -dot3f(FSUB(H[0].w, px), FSUB(H[1].w, py), FSUB(H[2].w, pz), nn[0], nn[1], nn[2]);
  float hi = dot3f(FSUB(AH.x, px), FSUB(AH.y, py), FSUB(AH.z, pz), nn[0], nn[1], nn[2]);
  return hit | (inside & (lo >= 0.0f) & (hi >= 0.0f));
}

// 2D predicate on a prepared edge (distance.py:216-235)
__device__ __forceinline__ bool near_edge(const float4* __restrict__ P, float px, float py, float r2) {
  float4 ab = P[0], e = P[1], h = P[2];
  float wax = FSUB(ab.x, px), way = FSUB(ab.y, py);
  float wbx = FSUB(ab.z, px), wby = FSUB(ab.w, py);
  bool disks = (FADD(FMUL(wax, wax), FMUL(way, way)) <= r2) | (FADD(FMUL(wbx, wbx), FMUL(wby, wby)) <= r2);
  float cr = FSUB(FMUL(e.x, way), FMUL(e.y, wax));
  float d2 = FDIV(FMUL(cr, cr), e.z);
  float de1 = -FADD(FMUL(wax, h.x), FMUL(way, h.y));
  float de2 = FADD(FMUL(wbx, h.x), FMUL(wby, h.y));
  return disks | ((d2 <= r2) & (de1 >= 0.0f) & (de2 >= 0.0f));
}

template <int D>
__device__ __forceinline__ bool near_face(const float4* __restrict__ P, const float* p, float r2) {
  if (D == 3) return near_tri(P, p[0], p[1], p[2], r2);
  return near_edge(P, p[0], p[1], r2);
}
