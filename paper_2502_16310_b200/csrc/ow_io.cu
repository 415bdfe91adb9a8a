// Legacy ASCII VTK export of the forest's leaf blocks (export_vtk,
// vtk_io.py:17-69), written natively: one device->host copy of the block
// arrays, leaf boxes in FP64 with the reference's formula (forest.py:156-161,
// 207-215), text formatted in parallel host threads.  The file is byte-for-
// byte the reference's: corners "%.9g %.9g %.9g", quads (2D) / hexahedra (3D)
// with unwelded corner points, `level` and `marked` cell scalars.
#include <stdio.h>
#include <string.h>

#include <string>
#include <thread>
#include <vector>

#include "ow_common.cuh"

namespace {

constexpr int VTK_QUAD = 9;
constexpr int VTK_HEXAHEDRON = 12;

// format lines [lo, hi) of one section with `fmt(i, buf)` into per-thread strings
template <class Fmt>
std::string format_parallel(int64_t n, Fmt fmt) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 4;
  if (nt > 32) nt = 32;
  if (n < 4096) nt = 1;
  std::vector<std::string> parts(nt);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) {
    th.emplace_back([&, t]() {
      const int64_t a = n * t / nt, b = n * (t + 1) / nt;
      std::string& out = parts[t];
      out.reserve((size_t)(b - a) * 32);
      char buf[256];
      for (int64_t i = a; i < b; ++i) {
        const int len = fmt(i, buf);
        out.append(buf, (size_t)len);
      }
    });
  }
  for (auto& x : th) x.join();
  std::string all;
  size_t tot = 0;
  for (auto& p : parts) tot += p.size();
  all.reserve(tot);
  for (auto& p : parts) all += p;
  return all;
}

}  // namespace

extern "C" int ow_export_vtk(ow_ctx* ctx, const ow_forest* f, const char* path, const char* title, void* stream) {
  (void)ctx;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = f->n_blocks;
  const int D = f->dim;
  std::vector<int16_t> level((size_t)n);
  std::vector<int32_t> coord[3], fc((size_t)n);
  std::vector<int8_t> marks((size_t)n);
  if (n > 0) {
    OW_CUDA(cudaMemcpyAsync(level.data(), f->d_level, 2 * (size_t)n, cudaMemcpyDeviceToHost, s));
    for (int a = 0; a < D; ++a) {
      coord[a].resize((size_t)n);
      OW_CUDA(cudaMemcpyAsync(coord[a].data(), f->d_coord[a], 4 * (size_t)n, cudaMemcpyDeviceToHost, s));
    }
    OW_CUDA(cudaMemcpyAsync(fc.data(), f->d_first_child, 4 * (size_t)n, cudaMemcpyDeviceToHost, s));
    OW_CUDA(cudaMemcpyAsync(marks.data(), f->d_marks, (size_t)n, cudaMemcpyDeviceToHost, s));
    OW_CUDA(cudaStreamSynchronize(s));
  }
  std::vector<int64_t> leaves;  // all_leaf_ids (forest.py:148-150): ascending
  for (int64_t i = 0; i < n; ++i)
    if (fc[(size_t)i] == -1) leaves.push_back(i);
  const int64_t nl = (int64_t)leaves.size();
  const int cp = D == 2 ? 4 : 8;
  // leaf boxes, FP64: lo = dmin + c * (ext / (root 2^L)), hi = lo + ext / (root 2^L)
  std::vector<double> lo((size_t)nl * D), hi((size_t)nl * D);
  for (int64_t k = 0; k < nl; ++k) {
    const int64_t i = leaves[(size_t)k];
    const int64_t L = level[(size_t)i];
    for (int a = 0; a < D; ++a) {
      const double den = (double)((int64_t)f->root[a] * ((int64_t)1 << L));
      const double q = f->dext[a] / den;
      const double o = f->dmin[a] + (double)coord[a][(size_t)i] * q;
      lo[(size_t)k * D + a] = o;
      hi[(size_t)k * D + a] = o + q;
    }
  }
  FILE* fp = fopen(path, "wb");
  if (!fp) {
    ow_set_error("cannot open %s for writing", path);
    return OW_ERR_INVALID;
  }
  std::string head = "# vtk DataFile Version 3.0\n";
  head += title ? title : "octowall leaf blocks";
  head += "\nASCII\nDATASET UNSTRUCTURED_GRID\n";
  char buf[256];
  snprintf(buf, sizeof(buf), "POINTS %lld float\n", (long long)(nl * cp));
  head += buf;
  fwrite(head.data(), 1, head.size(), fp);
  const std::string pts = format_parallel(nl * cp, [&](int64_t t, char* b) {
    const int64_t k = t / cp;
    const int ci = (int)(t % cp);
    const double* l = &lo[(size_t)k * D];
    const double* h = &hi[(size_t)k * D];
    double x, y, z;
    if (D == 2) {  // vtk_io.py:25-31: (lo,lo) (hi,lo) (hi,hi) (lo,hi)
      x = (ci == 1 || ci == 2) ? h[0] : l[0];
      y = (ci >= 2) ? h[1] : l[1];
      z = 0.0;
    } else {  // vtk_io.py:35-39
      x = (ci == 1 || ci == 2 || ci == 5 || ci == 6) ? h[0] : l[0];
      y = (ci == 2 || ci == 3 || ci == 6 || ci == 7) ? h[1] : l[1];
      z = ci >= 4 ? h[2] : l[2];
    }
    return snprintf(b, 256, "%.9g %.9g %.9g\n", x, y, z);
  });
  fwrite(pts.data(), 1, pts.size(), fp);
  snprintf(buf, sizeof(buf), "CELLS %lld %lld\n", (long long)nl, (long long)(nl * (cp + 1)));
  fputs(buf, fp);
  const std::string cells = format_parallel(nl, [&](int64_t k, char* b) {
    const long long base = (long long)k * cp;
    if (cp == 4) return snprintf(b, 256, "4 %lld %lld %lld %lld\n", base, base + 1, base + 2, base + 3);
    return snprintf(b, 256, "8 %lld %lld %lld %lld %lld %lld %lld %lld\n", base, base + 1, base + 2, base + 3,
                    base + 4, base + 5, base + 6, base + 7);
  });
  fwrite(cells.data(), 1, cells.size(), fp);
  snprintf(buf, sizeof(buf), "CELL_TYPES %lld\n", (long long)nl);
  fputs(buf, fp);
  const int ct = D == 2 ? VTK_QUAD : VTK_HEXAHEDRON;
  const std::string types = format_parallel(nl, [&](int64_t, char* b) { return snprintf(b, 256, "%d\n", ct); });
  fwrite(types.data(), 1, types.size(), fp);
  snprintf(buf, sizeof(buf), "CELL_DATA %lld\nSCALARS level int 1\nLOOKUP_TABLE default\n", (long long)nl);
  fputs(buf, fp);
  const std::string lv = format_parallel(
      nl, [&](int64_t k, char* b) { return snprintf(b, 256, "%d\n", (int)level[(size_t)leaves[(size_t)k]]); });
  fwrite(lv.data(), 1, lv.size(), fp);
  fputs("SCALARS marked int 1\nLOOKUP_TABLE default\n", fp);
  const std::string mk = format_parallel(nl, [&](int64_t k, char* b) {
    return snprintf(b, 256, "%d\n", marks[(size_t)leaves[(size_t)k]] == OW_MARKED ? 1 : 0);
  });
  fwrite(mk.data(), 1, mk.size(), fp);
  if (fclose(fp) != 0) {
    ow_set_error("write to %s failed", path);
    return OW_ERR_INTERNAL;
  }
  return OW_OK;
}
