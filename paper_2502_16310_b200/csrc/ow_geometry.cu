// Geometry import kernels: binary STL records -> SoA, index->coords gather,
// degenerate-face / bounding-box / non-finite reduction.
// Reference: octowall/geometry.py:262-308 (index_to_coords, validate_faces,
// bounding_box) and 415-436 (_parse_binary_stl, _tris_to_geometry).
#include "ow_common.cuh"

namespace {

constexpr int STL_TILE = 256;  // faces per CTA

// 50-byte records are only 2-byte aligned: stage the tile's bytes through
// shared memory with coalesced 16-bit loads, then emit 9 coalesced float planes.
__global__ void __launch_bounds__(STL_TILE)
k_stl_to_soa(const uint16_t* rec16, int64_t n, float* coords) {
  ow_pdl_wait();
  __shared__ __align__(16) uint16_t s[STL_TILE * 25];
  const int64_t f0 = (int64_t)blockIdx.x * STL_TILE;
  const int64_t nf = min((int64_t)STL_TILE, n - f0);
  const uint16_t* src = rec16 + f0 * 25;
  int i0 = 0;  // 16-byte loads when the tile is 16-byte aligned (the common case), 2-byte for the rest
  if ((((uintptr_t)src) & 15) == 0) {
    const int nv = (int)(nf * 50 / 16);
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(s);
    for (int i = threadIdx.x; i < nv; i += STL_TILE) d4[i] = s4[i];
    i0 = nv * 8;
  }
  for (int i = i0 + threadIdx.x; i < nf * 25; i += STL_TILE) s[i] = src[i];
  __syncthreads();
  if (threadIdx.x < nf) {
    const uint16_t* r = s + threadIdx.x * 25 + 6;  // skip the 12-byte normal
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      uint32_t bits = (uint32_t)r[2 * j] | ((uint32_t)r[2 * j + 1] << 16);
      coords[(int64_t)j * n + f0 + threadIdx.x] = __uint_as_float(bits);
    }
  }
}

__global__ void k_index_to_coords(int dim, const float* __restrict__ verts, const int32_t* __restrict__ faces,
                                  int64_t n, float* coords) {
  ow_pdl_wait();
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  for (int j = 0; j < dim; ++j) {
    int64_t v = faces[k * dim + j];
    for (int c = 0; c < dim; ++c) coords[((int64_t)j * dim + c) * n + k] = verts[v * dim + c];
  }
}

__device__ __forceinline__ void atomic_min_f(float* a, float v) {
  if (__float_as_uint(v) >> 31) atomicMax((unsigned*)a, __float_as_uint(v));
  else atomicMin((int*)a, __float_as_int(v));
}
__device__ __forceinline__ void atomic_max_f(float* a, float v) {
  if (__float_as_uint(v) >> 31) atomicMin((unsigned*)a, __float_as_uint(v));
  else atomicMax((int*)a, __float_as_int(v));
}

// small[0] first degenerate (u64 min), small[1] first non-finite (u64 min),
// then floats: min[3], max[3], absmax at ((float*)(small+2))[0..6]
// (the dimension is a template parameter: the per-face vertex array then
// lives in registers instead of local memory)
// per-face part of the check: the reference's degeneracy test (FP64), finite
// coordinates, bounding box, |max| and the largest box side (work shape)
struct FaceAcc {
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY}, am = 0.0f;
  float ext_sum = 0.0f;  // sum of per-face largest bounding-box sides (a work-shape estimate)
  unsigned long long bad_deg = ~0ull, bad_fin = ~0ull;
};

template <int dim>
__device__ __forceinline__ void face_check_one(const float (&v)[3][3], int64_t k, FaceAcc& acc) {
  bool finite = true;
#pragma unroll
  for (int j = 0; j < dim; ++j)
#pragma unroll
    for (int a = 0; a < dim; ++a) {
      const float x = v[j][a];
      finite &= isfinite(x);
      acc.mn[a] = fminf(acc.mn[a], x);
      acc.mx[a] = fmaxf(acc.mx[a], x);
      acc.am = fmaxf(acc.am, fabsf(x));
    }
  if (!finite) {
    acc.bad_fin = min(acc.bad_fin, (unsigned long long)k);
    return;
  }
  float side = 0.0f;
#pragma unroll
  for (int a = 0; a < dim; ++a) {
    float lo = v[0][a], hi = v[0][a];
#pragma unroll
    for (int j = 1; j < dim; ++j) lo = fminf(lo, v[j][a]), hi = fmaxf(hi, v[j][a]);
    side = fmaxf(side, hi - lo);
  }
  acc.ext_sum += side;
  bool deg;
  if (dim == 2) {  // geometry.py:281-285
    double dx = DSUB((double)v[1][0], (double)v[0][0]), dy = DSUB((double)v[1][1], (double)v[0][1]);
    deg = DADD(DMUL(dx, dx), DMUL(dy, dy)) == 0.0;
  } else {  // geometry.py:287-297, FP64
    double u[3], w[3], z[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      u[a] = DSUB((double)v[1][a], (double)v[0][a]);
      w[a] = DSUB((double)v[2][a], (double)v[0][a]);
      z[a] = DSUB((double)v[2][a], (double)v[1][a]);
    }
    double su = DADD(DADD(DMUL(u[0], u[0]), DMUL(u[1], u[1])), DMUL(u[2], u[2]));
    double sw = DADD(DADD(DMUL(w[0], w[0]), DMUL(w[1], w[1])), DMUL(w[2], w[2]));
    double sz = DADD(DADD(DMUL(z[0], z[0]), DMUL(z[1], z[1])), DMUL(z[2], z[2]));
    double scale = fmax(fmax(su, sw), sz);
    double cx = DSUB(DMUL(u[1], w[2]), DMUL(u[2], w[1]));
    double cy = DSUB(DMUL(u[2], w[0]), DMUL(u[0], w[2]));
    double cz = DSUB(DMUL(u[0], w[1]), DMUL(u[1], w[0]));
    double area = __dsqrt_rn(DADD(DADD(DMUL(cx, cx), DMUL(cy, cy)), DMUL(cz, cz)));
    deg = (scale == 0.0) || (area < DMUL(1e-12, scale));
  }
  if (deg) acc.bad_deg = min(acc.bad_deg, (unsigned long long)k);
}

// warp and CTA reduction of the accumulators, one atomic per quantity per CTA
// (all threads of the CTA call it)
template <int dim>
__device__ __forceinline__ void face_check_flush(FaceAcc& acc, int64_t* small) {
  for (int o = 16; o > 0; o >>= 1) {
    for (int a = 0; a < 3; ++a) {
      acc.mn[a] = fminf(acc.mn[a], __shfl_xor_sync(0xffffffffu, acc.mn[a], o));
      acc.mx[a] = fmaxf(acc.mx[a], __shfl_xor_sync(0xffffffffu, acc.mx[a], o));
    }
    acc.am = fmaxf(acc.am, __shfl_xor_sync(0xffffffffu, acc.am, o));
    acc.ext_sum += __shfl_xor_sync(0xffffffffu, acc.ext_sum, o);
    acc.bad_deg = min(acc.bad_deg, __shfl_xor_sync(0xffffffffu, acc.bad_deg, o));
    acc.bad_fin = min(acc.bad_fin, __shfl_xor_sync(0xffffffffu, acc.bad_fin, o));
  }
  __shared__ float s_f[8][8];
  __shared__ unsigned long long s_b[8][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    for (int a = 0; a < 3; ++a) s_f[w][a] = acc.mn[a], s_f[w][3 + a] = acc.mx[a];
    s_f[w][6] = acc.am;
    s_f[w][7] = acc.ext_sum;
    s_b[w][0] = acc.bad_deg;
    s_b[w][1] = acc.bad_fin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int k = 1; k < nw; ++k) {
      for (int a = 0; a < 3; ++a) acc.mn[a] = fminf(acc.mn[a], s_f[k][a]), acc.mx[a] = fmaxf(acc.mx[a], s_f[k][3 + a]);
      acc.am = fmaxf(acc.am, s_f[k][6]);
      acc.ext_sum += s_f[k][7];
      acc.bad_deg = min(acc.bad_deg, s_b[k][0]);
      acc.bad_fin = min(acc.bad_fin, s_b[k][1]);
    }
    float* fs = (float*)(small + 2);
    for (int a = 0; a < dim; ++a) {
      atomic_min_f(&fs[a], acc.mn[a]);
      atomic_max_f(&fs[3 + a], acc.mx[a]);
    }
    atomic_max_f(&fs[6], acc.am);
    atomicAdd(&fs[7], acc.ext_sum);
    if (acc.bad_deg != ~0ull) atomicMin((unsigned long long*)&small[0], acc.bad_deg);
    if (acc.bad_fin != ~0ull) atomicMin((unsigned long long*)&small[1], acc.bad_fin);
  }
}

// small[0] first degenerate (u64 min), small[1] first non-finite (u64 min),
// then floats: min[3], max[3], absmax at ((float*)(small+2))[0..6]
// (the dimension is a template parameter: the per-face vertex array then
// lives in registers instead of local memory)
template <int dim>
__global__ void __launch_bounds__(256) k_face_check(const float* __restrict__ c, int64_t n, int64_t* small) {
  ow_pdl_wait();
  FaceAcc acc;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    float v[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int j = 0; j < dim; ++j)
#pragma unroll
      for (int a = 0; a < dim; ++a) v[j][a] = c[((int64_t)j * dim + a) * n + k];
    face_check_one<dim>(v, k, acc);
  }
  face_check_flush<dim>(acc, small);
}

// Binary STL records -> SoA coordinates and the face check in one pass (the
// fused pass: the check reads the vertices from registers instead of the
// coordinates it just wrote).  Persistent over tiles of STL_TILE faces.
__global__ void __launch_bounds__(STL_TILE) k_stl_to_soa_check(const uint16_t* rec16, int64_t n, float* coords,
                                                              int64_t* small) {
  ow_pdl_wait();
  __shared__ __align__(16) uint16_t s[STL_TILE * 25];
  FaceAcc acc;
  for (int64_t f0 = (int64_t)blockIdx.x * STL_TILE; f0 < n; f0 += (int64_t)gridDim.x * STL_TILE) {
    const int64_t nf = min((int64_t)STL_TILE, n - f0);
    const uint16_t* src = rec16 + f0 * 25;
    __syncthreads();  // (the staging of the previous tile is consumed)
    int i0 = 0;
    if ((((uintptr_t)src) & 15) == 0) {
      const int nv = (int)(nf * 50 / 16);
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      uint4* d4 = reinterpret_cast<uint4*>(s);
      for (int i = threadIdx.x; i < nv; i += STL_TILE) d4[i] = s4[i];
      i0 = nv * 8;
    }
    for (int i = i0 + threadIdx.x; i < nf * 25; i += STL_TILE) s[i] = src[i];
    __syncthreads();
    if (threadIdx.x < nf) {
      const uint16_t* r = s + threadIdx.x * 25 + 6;  // skip the 12-byte normal
      float v[3][3];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        const uint32_t bits = (uint32_t)r[2 * j] | ((uint32_t)r[2 * j + 1] << 16);
        v[j / 3][j % 3] = __uint_as_float(bits);
        coords[(int64_t)j * n + f0 + threadIdx.x] = v[j / 3][j % 3];
      }
      face_check_one<3>(v, f0 + threadIdx.x, acc);
    }
  }
  face_check_flush<3>(acc, small);
}

__global__ void k_face_check_init(int64_t* small) {
  ow_pdl_wait();
  small[0] = -1;  // 0xfff.. as unsigned = "none"
  small[1] = -1;
  float* fs = (float*)(small + 2);
  for (int a = 0; a < 3; ++a) {
    fs[a] = INFINITY;
    fs[3 + a] = -INFINITY;
  }
  fs[6] = 0.0f;
  fs[7] = 0.0f;
}

}  // namespace

extern "C" int ow_stl_binary_to_soa(ow_ctx* ctx, const uint8_t* d_records, int64_t n, float* d_coords,
                                    void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0 || (n > 0 && (!d_records || !d_coords))) {
    ow_set_error("ow_stl_binary_to_soa: bad arguments");
    return OW_ERR_INVALID;
  }
  if (((uintptr_t)d_records & 1) != 0) {
    ow_set_error("ow_stl_binary_to_soa: records must be 2-byte aligned");
    return OW_ERR_INVALID;
  }
  if (n == 0) return OW_OK;
  OW_PROF_BEGIN(ctx, PROF_STL, s);
  ow_launch(k_stl_to_soa, ow_blocks(n, STL_TILE), STL_TILE, 0, s, (const uint16_t*)d_records, n, d_coords);
  OW_PROF_END(ctx, PROF_STL, s);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

extern "C" int ow_index_to_coords(ow_ctx* ctx, int32_t dim, const float* d_vertices, const int32_t* d_faces,
                                  int64_t n, float* d_coords, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (dim != 2 && dim != 3) {
    ow_set_error("dim must be 2 or 3, got %d", dim);
    return OW_ERR_INVALID;
  }
  if (n == 0) return OW_OK;
  ow_launch(k_index_to_coords, ow_blocks(n, 256), 256, 0, s, dim, d_vertices, d_faces, n, d_coords);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

// face summary words [0, 6) from a readback -> ow_face_summary
void ow_face_summary_from(const int64_t* h, int64_t n, ow_face_summary* out) {
  out->first_degenerate = h[0];
  out->first_nonfinite = h[1];
  const float* fs = (const float*)(h + 2);
  for (int a = 0; a < 3; ++a) {
    out->bbox_min[a] = fs[a];
    out->bbox_max[a] = fs[3 + a];
  }
  out->abs_max = fs[6];
  out->mean_extent = n > 0 ? fs[7] / (float)n : 0.0f;
}

// fused pass: STL records -> coordinates + the face check into d_small[dst, dst + 6)
int ow_stl_to_soa_checked(ow_ctx* ctx, const uint8_t* d_records, int64_t n, float* d_coords, int64_t* dst,
                          cudaStream_t s, bool init_summary) {
  if (n < 0 || (n > 0 && (!d_records || !d_coords)) || ((uintptr_t)d_records & 1) != 0) {
    ow_set_error("ow_stl_binary_to_soa: bad arguments (records must be 2-byte aligned)");
    return OW_ERR_INVALID;
  }
  if (init_summary) {  // (else the caller initialised the summary words: ow_face_summary_init_words)
    ow_launch(k_face_check_init, 1, 1, 0, s, dst);
    OW_LAUNCHED(ctx);
  }
  if (n > 0) {
    OW_PROF_BEGIN(ctx, PROF_STL, s);
    ow_launch(k_stl_to_soa_check, ow_blocks(n, STL_TILE, 8 * OW_SMS), STL_TILE, 0, s, (const uint16_t*)d_records, n,
              d_coords, dst);
    OW_PROF_END(ctx, PROF_STL, s);
    OW_LAUNCHED(ctx);
  }
  OW_CHECK_LAUNCH();
  return OW_OK;
}

// launch the face check into d_small[dst, dst + 6) without reading it back
int ow_face_check_launch(ow_ctx* ctx, int32_t dim, const float* d_coords, int64_t n, int64_t* dst, cudaStream_t s) {
  if (dim != 2 && dim != 3) {
    ow_set_error("dim must be 2 or 3, got %d", dim);
    return OW_ERR_INVALID;
  }
  ow_launch(k_face_check_init, 1, 1, 0, s, dst);
  OW_LAUNCHED(ctx);
  if (n > 0) {
    if (dim == 3) ow_launch(k_face_check<3>, ow_blocks(n, 256, 16 * OW_SMS), 256, 0, s, d_coords, n, dst);
    else ow_launch(k_face_check<2>, ow_blocks(n, 256, 16 * OW_SMS), 256, 0, s, d_coords, n, dst);
    OW_LAUNCHED(ctx);
  }
  OW_CHECK_LAUNCH();
  return OW_OK;
}

extern "C" int ow_face_check(ow_ctx* ctx, int32_t dim, const float* d_coords, int64_t n,
                             ow_face_summary* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  OW_TRY(ow_face_check_launch(ctx, dim, d_coords, n, ctx->d_small, s));
  int64_t h[6];
  OW_TRY(ow_readback(ctx, ctx->d_small, 6, h, s));
  ow_face_summary_from(h, n, out);
  return OW_OK;
}
