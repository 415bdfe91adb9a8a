// Legacy ASCII VTK export of the forest's leaf blocks (export_vtk,
// vtk_io.py:17-69), written natively: one device->host copy of the block
// arrays, leaf boxes in FP64 with the reference's formula (forest.py:156-161,
// 207-215), text formatted in parallel host threads.  The file is byte-for-
// byte the reference's: corners "%.9g %.9g %.9g", quads (2D) / hexahedra (3D)
// with unwelded corner points, `level` and `marked` cell scalars.
#include <stdio.h>
#include <stdlib.h>
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

// ---------------------------------------------------------------------------
// ASCII STL (geometry.py:349-412) on the host: the whole parser, errors
// included.  Pure-ASCII text (the Python shim turns any other valid UTF-8
// into an equivalent ASCII token stream first); every number token is checked
// against Python's float() grammar (sign, digits with single underscores
// between digits, optional fraction and exponent, inf / infinity / nan)
// before a correctly rounded strtod, then rounded once to float32 like
// np.asarray(..., float32).  The accepting path tokenises and converts in
// parallel; on any failure a sequential walk finds the error the reference
// reports first (its token-by-token order) and returns it as
// err = {code, line, token offset, token length, expected keyword}:
//   1 unexpected end of file   2 expected <keyword>, got <token>
//   3 expected a number        4 expected 'facet' or 'endsolid'
//   5 <keyword> after endsolid 6 non-ASCII byte (the shim's job)
// Lines are numbered like str.splitlines() (\n, \r, \r\n, \v, \f, \x1c-\x1e).
// ---------------------------------------------------------------------------
namespace {

enum { PE_EOF = 1, PE_EXPECT, PE_NUMBER, PE_FACET, PE_AFTER, PE_NONASCII };
const char* const PE_KW[] = {"solid", "normal", "outer", "loop", "vertex", "endloop", "endfacet"};
enum { KW_SOLID, KW_NORMAL, KW_OUTER, KW_LOOP, KW_VERTEX, KW_ENDLOOP, KW_ENDFACET };

inline bool py_space(unsigned char c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }

inline bool ieq(const char* t, int n, const char* kw) {
  int i = 0;
  for (; i < n && kw[i]; ++i) {
    char c = t[i];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    if (c != kw[i]) return false;
  }
  return i == n && kw[i] == 0;
}

// Python float() grammar on an ASCII token; writes the underscore-free text
bool py_float(const char* t, int n, double* out) {
  char buf[128];
  if (n <= 0 || n >= (int)sizeof(buf)) return false;
  int i = 0, o = 0;
  if (t[i] == '+' || t[i] == '-') buf[o++] = t[i++];
  const char* r = t + i;
  const int rn = n - i;
  if (ieq(r, rn, "inf") || ieq(r, rn, "infinity")) {
    *out = (o && buf[0] == '-') ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(r, rn, "nan")) {
    *out = NAN;
    return true;
  }
  auto digitpart = [&](void) -> bool {  // digit (['_'] digit)*
    if (i >= n || t[i] < '0' || t[i] > '9') return false;
    buf[o++] = t[i++];
    while (i < n) {
      if (t[i] >= '0' && t[i] <= '9') {
        buf[o++] = t[i++];
      } else if (t[i] == '_' && i + 1 < n && t[i + 1] >= '0' && t[i + 1] <= '9') {
        ++i;
      } else {
        break;
      }
    }
    return true;
  };
  bool mant = false;
  if (i < n && t[i] >= '0' && t[i] <= '9') {
    digitpart();
    mant = true;
  }
  if (i < n && t[i] == '.') {
    buf[o++] = t[i++];
    if (i < n && t[i] >= '0' && t[i] <= '9') {
      digitpart();
      mant = true;
    }
  }
  if (!mant) return false;
  if (i < n && (t[i] == 'e' || t[i] == 'E')) {
    buf[o++] = t[i++];
    if (i < n && (t[i] == '+' || t[i] == '-')) buf[o++] = t[i++];
    if (!digitpart()) return false;
  }
  if (i != n) return false;
  buf[o] = 0;
  char* end = nullptr;
  *out = strtod(buf, &end);
  return end == buf + o;
}

struct Tok {
  const char* p;
  const char* end;
  const char* t;
  int n;
  bool next() {
    while (p < end && py_space((unsigned char)*p)) ++p;
    if (p >= end) return false;
    t = p;
    while (p < end && !py_space((unsigned char)*p)) ++p;
    n = (int)(p - t);
    return true;
  }
};

// 1-based line of byte offset `off` (str.splitlines() boundaries)
int64_t line_of(const char* data, int64_t off) {
  int64_t line = 1;
  for (int64_t i = 0; i < off; ++i) {
    const unsigned char c = (unsigned char)data[i];
    if (c == '\r') {
      if (i + 1 < off && data[i + 1] == '\n') ++i;
      ++line;
    } else if (c == '\n' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1e)) {
      ++line;
    }
  }
  return line;
}

// The reference's token-by-token walk (geometry.py:358-411), reporting the
// first error it meets; only run when the parallel path failed.
template <class TF, class NF>
void diagnose(const char* data, size_t ntok, TF T, NF N, int64_t* err) {
  size_t i = 0;
  auto set = [&](int code, size_t k, int kw) {
    err[0] = code;
    err[1] = ntok ? line_of(data, (int64_t)(T(k) - data)) : -1;
    err[2] = ntok ? (int64_t)(T(k) - data) : 0;
    err[3] = ntok ? N(k) : 0;
    err[4] = kw;
  };
  auto take = [&](int kw) -> bool {  // kw < 0: any token
    if (i >= ntok) {
      set(PE_EOF, ntok ? ntok - 1 : 0, -1);
      return false;
    }
    if (kw >= 0 && !ieq(T(i), N(i), PE_KW[kw])) {
      set(PE_EXPECT, i, kw);
      return false;
    }
    ++i;
    return true;
  };
  auto number = [&]() -> bool {
    if (i >= ntok) {
      set(PE_EOF, ntok ? ntok - 1 : 0, -1);
      return false;
    }
    double v;
    if (!py_float(T(i), N(i), &v)) {
      set(PE_NUMBER, i, -1);
      return false;
    }
    ++i;
    return true;
  };
  if (!take(KW_SOLID)) return;
  while (i < ntok && !ieq(T(i), N(i), "facet") && !ieq(T(i), N(i), "endsolid")) ++i;
  for (;;) {
    if (i >= ntok) {
      set(PE_EOF, ntok ? ntok - 1 : 0, -1);
      return;
    }
    if (ieq(T(i), N(i), "endsolid")) {
      ++i;
      break;
    }
    if (!ieq(T(i), N(i), "facet")) {
      set(PE_FACET, i, -1);
      return;
    }
    ++i;
    if (!take(KW_NORMAL) || !number() || !number() || !number() || !take(KW_OUTER) || !take(KW_LOOP)) return;
    for (int v = 0; v < 3; ++v)
      if (!take(KW_VERTEX) || !number() || !number() || !number()) return;
    if (!take(KW_ENDLOOP) || !take(KW_ENDFACET)) return;
  }
  for (; i < ntok; ++i)
    if (ieq(T(i), N(i), "facet") || ieq(T(i), N(i), "solid") || ieq(T(i), N(i), "vertex") ||
        ieq(T(i), N(i), "endsolid")) {
      set(PE_AFTER, i, -1);
      return;
    }
}

}  // namespace

extern "C" int ow_parse_ascii_stl(const char* data, int64_t len, float* tris, int64_t cap, int64_t* out_n,
                                  int64_t* err) {
  *out_n = 0;
  for (int k = 0; k < 5; ++k) err[k] = 0;
  // 1. tokenize in parallel chunks (boundaries moved to whitespace); any
  //    non-ASCII byte sends the file to the reference-faithful parser
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 4;
  if (nt > 32) nt = 32;
  if (len < (int64_t(1) << 20)) nt = 1;
  std::vector<int64_t> cut(nt + 1);
  cut[0] = 0;
  cut[nt] = len;
  for (unsigned t = 1; t < nt; ++t) {
    int64_t c = len * t / nt;
    if (c < cut[t - 1]) c = cut[t - 1];
    while (c < len && !py_space((unsigned char)data[c])) ++c;
    cut[t] = c;
  }
  std::vector<std::vector<std::pair<int64_t, int>>> part(nt);
  std::vector<int> bad(nt, 0);
  {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
      th.emplace_back([&, t]() {
        for (int64_t i = cut[t]; i < cut[t + 1]; ++i)
          if ((unsigned char)data[i] >= 0x80) {
            bad[t] = 1;
            return;
          }
        auto& v = part[t];
        v.reserve((size_t)((cut[t + 1] - cut[t]) / 6 + 16));
        Tok k{data + cut[t], data + cut[t + 1], nullptr, 0};
        while (k.next()) v.emplace_back((int64_t)(k.t - data), k.n);
      });
    for (auto& x : th) x.join();
  }
  for (unsigned t = 0; t < nt; ++t)
    if (bad[t]) {
      err[0] = PE_NONASCII;
      ow_set_error("ASCII STL: non-ASCII byte");
      return OW_ERR_PARSE;
    }
  size_t ntok = 0;
  for (auto& v : part) ntok += v.size();
  std::vector<std::pair<int64_t, int>> tok;
  tok.reserve(ntok);
  for (auto& v : part) tok.insert(tok.end(), v.begin(), v.end());
  auto T = [&](size_t i) { return data + tok[i].first; };
  auto N = [&](size_t i) { return tok[i].second; };
  auto fail = [&]() {
    diagnose(data, ntok, T, N, err);
    ow_set_error("ASCII STL: parse error (code %lld, line %lld)", (long long)err[0], (long long)err[1]);
    return OW_ERR_PARSE;
  };
  // 2. grammar walk (sequential); number tokens are only located here
  size_t i = 0;
  if (ntok == 0 || !ieq(T(0), N(0), "solid")) return fail();
  ++i;
  while (i < ntok && !ieq(T(i), N(i), "facet") && !ieq(T(i), N(i), "endsolid")) ++i;
  std::vector<size_t> facet_at;  // token index of each facet's "facet"
  while (true) {
    if (i >= ntok) return fail();  // unexpected end of file
    if (ieq(T(i), N(i), "endsolid")) break;
    // facet normal n n n outer loop (vertex x y z) x3 endloop endfacet: 21 tokens
    if (i + 21 > ntok) return fail();
    if (!ieq(T(i), N(i), "facet") || !ieq(T(i + 1), N(i + 1), "normal") || !ieq(T(i + 5), N(i + 5), "outer") ||
        !ieq(T(i + 6), N(i + 6), "loop") || !ieq(T(i + 7), N(i + 7), "vertex") ||
        !ieq(T(i + 11), N(i + 11), "vertex") || !ieq(T(i + 15), N(i + 15), "vertex") ||
        !ieq(T(i + 19), N(i + 19), "endloop") || !ieq(T(i + 20), N(i + 20), "endfacet"))
      return fail();
    facet_at.push_back(i);
    i += 21;
  }
  // trailing solid-name tokens are allowed, other keywords are not
  for (size_t j = i + 1; j < ntok; ++j)
    if (ieq(T(j), N(j), "facet") || ieq(T(j), N(j), "solid") || ieq(T(j), N(j), "vertex") ||
        ieq(T(j), N(j), "endsolid"))
      return fail();
  const int64_t nf = (int64_t)facet_at.size();
  if (nf > cap) return OW_ERR_CAPACITY;
  // 3. numbers in parallel: normals are validated, vertices converted
  std::vector<int> nbad(nt, 0);
  {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
      th.emplace_back([&, t]() {
        const int64_t a = nf * t / nt, b = nf * (t + 1) / nt;
        static const int num_at[12] = {2, 3, 4, 8, 9, 10, 12, 13, 14, 16, 17, 18};
        for (int64_t fct = a; fct < b; ++fct) {
          const size_t base = facet_at[(size_t)fct];
          for (int q = 0; q < 12; ++q) {
            double v;
            const size_t k = base + num_at[q];
            if (!py_float(T(k), N(k), &v)) {
              nbad[t] = 1;
              return;
            }
            if (q >= 3) tris[fct * 9 + (q - 3)] = (float)v;  // one rounding, as np.asarray(..., float32)
          }
        }
      });
    for (auto& x : th) x.join();
  }
  for (unsigned t = 0; t < nt; ++t)
    if (nbad[t]) return fail();
  *out_n = nf;
  return OW_OK;
}
