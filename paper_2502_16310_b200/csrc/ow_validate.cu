// Predicate-vs-referee sampling on the GPU (validate.py:98-141): for n
// independent (point, face, d) cases, the FP32 near-face predicate (the
// marking kernels' device function) and the exact FP64 distance referee
// (exact_point_triangle_distance distance.py:275-345 / point_segment_distance_sq
// 260-272), with the reference's double-precision operation order (no FMA:
// compiled -fmad=false; IEEE division and sqrt).
#include "ow_predicate.cuh"

namespace {

__device__ double exact_tri(const double* p, const double* a, const double* b, const double* c) {
  const double abx = b[0] - a[0], aby = b[1] - a[1], abz = b[2] - a[2];
  const double acx = c[0] - a[0], acy = c[1] - a[1], acz = c[2] - a[2];
  const double apx = p[0] - a[0], apy = p[1] - a[1], apz = p[2] - a[2];
  const double d1 = abx * apx + aby * apy + abz * apz;
  const double d2 = acx * apx + acy * apy + acz * apz;
  if (d1 <= 0.0 && d2 <= 0.0) return sqrt(apx * apx + apy * apy + apz * apz);
  const double bpx = p[0] - b[0], bpy = p[1] - b[1], bpz = p[2] - b[2];
  const double d3 = abx * bpx + aby * bpy + abz * bpz;
  const double d4 = acx * bpx + acy * bpy + acz * bpz;
  if (d3 >= 0.0 && d4 <= d3) return sqrt(bpx * bpx + bpy * bpy + bpz * bpz);
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    const double t = d1 / (d1 - d3);
    const double qx = apx - t * abx, qy = apy - t * aby, qz = apz - t * abz;
    return sqrt(qx * qx + qy * qy + qz * qz);
  }
  const double cpx = p[0] - c[0], cpy = p[1] - c[1], cpz = p[2] - c[2];
  const double d5 = abx * cpx + aby * cpy + abz * cpz;
  const double d6 = acx * cpx + acy * cpy + acz * cpz;
  if (d6 >= 0.0 && d5 <= d6) return sqrt(cpx * cpx + cpy * cpy + cpz * cpz);
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    const double t = d2 / (d2 - d6);
    const double qx = apx - t * acx, qy = apy - t * acy, qz = apz - t * acz;
    return sqrt(qx * qx + qy * qy + qz * qz);
  }
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    const double bcx = c[0] - b[0], bcy = c[1] - b[1], bcz = c[2] - b[2];
    const double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    const double qx = bpx - t * bcx, qy = bpy - t * bcy, qz = bpz - t * bcz;
    return sqrt(qx * qx + qy * qy + qz * qz);
  }
  const double denom = 1.0 / (va + vb + vc);
  const double v = vb * denom, w = vc * denom;
  const double qx = apx - (v * abx + w * acx);
  const double qy = apy - (v * aby + w * acy);
  const double qz = apz - (v * abz + w * acz);
  return sqrt(qx * qx + qy * qy + qz * qz);
}

// squared distance to the closed segment [a, b] (distance.py:260-272)
__device__ double seg_dist_sq(const double* p, const double* a, const double* b) {
  const double ex = b[0] - a[0], ey = b[1] - a[1];
  const double el2 = ex * ex + ey * ey;
  double t = ((p[0] - a[0]) * ex + (p[1] - a[1]) * ey) / el2;
  t = fmin(1.0, fmax(0.0, t));
  const double qx = p[0] - (a[0] + t * ex), qy = p[1] - (a[1] + t * ey);
  return qx * qx + qy * qy;
}

__global__ void k_referee(int dim, const float* __restrict__ pts, const float* __restrict__ faces,
                          const double* __restrict__ dd, int64_t n, double* exact, uint8_t* mask) {
  ow_pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 pay[PAY3];
  const float d = (float)dd[i];
  const float r2 = FMUL(d, d);
  float p[3];
  double pd[3], v[3][3];
  for (int a = 0; a < dim; ++a) {
    p[a] = pts[i * dim + a];
    pd[a] = (double)p[a];
    for (int j = 0; j < dim; ++j) v[j][a] = (double)faces[((int64_t)j * dim + a) * n + i];
  }
  if (dim == 3) {
    face_prep_one<3>(faces, n, i, d, pay);
    mask[i] = near_face<3>(pay, p, r2);
    exact[i] = exact_tri(pd, v[0], v[1], v[2]);
  } else {
    face_prep_one<2>(faces, n, i, d, pay);
    mask[i] = near_face<2>(pay, p, r2);
    exact[i] = sqrt(seg_dist_sq(pd, v[0], v[1]));
  }
}

}  // namespace

extern "C" int ow_referee_pairs(ow_ctx* ctx, int32_t dim, const float* d_points, const float* d_faces,
                                const double* d_d, int64_t n, double* d_exact, uint8_t* d_mask, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (dim != 2 && dim != 3) {
    ow_set_error("dim must be 2 or 3, got %d", dim);
    return OW_ERR_INVALID;
  }
  if (n <= 0) return OW_OK;
  ow_launch(k_referee, ow_blocks(n, 128), 128, 0, s, dim, d_points, d_faces, d_d, n, d_exact, d_mask);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}
