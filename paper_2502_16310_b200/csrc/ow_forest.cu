// Forest-of-octrees kernels: leaf listing, level histograms, cell centres,
// mark propagation, refinement with deterministic allocation and 2:1 balance.
//
// Reference: octowall/forest.py:143-205 (queries, cell centres), 224-285
// (face neighbours), 300-370 (split / refine_marked / _rebalance);
// octowall/nearwall.py:321-366 (propagate_marks).
//
// The reference resolves neighbours through a (level, coords) -> id dict; here
// a neighbour is found by descending from the root lattice with the child
// bits of its lattice coordinates (`locate`), which needs no hash table and
// touches <= level+1 first_child words per query.
#include "ow_scan.cuh"

namespace {

using ow::scan;
using ow::scan01;

__global__ void k_cell_centers(ForestC F, const int32_t* __restrict__ ids, int64_t n, float* out) {
  ow_pdl_wait();
  const int C = F.dim == 2 ? 16 : 64;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * C) return;
  int64_t i = t / C;
  int c = (int)(t % C);
  int id = ids[i];
  int L = F.level[id];
  for (int a = 0; a < F.dim; ++a) {
    double q = block_len(F, a, L);
    double o = DADD(F.dmin[a], DMUL((double)F.coord[a][id], q));
    int digit = (c >> (2 * a)) & 3;
    double u = ((double)digit + 0.5) / 4.0;  // exact
    out[t * F.dim + a] = __double2float_rn(DADD(o, DMUL(u, q)));
  }
}

__global__ void k_level_counts(ForestC F, int max_levels, unsigned long long* blocks, unsigned long long* leaves) {
  ow_pdl_wait();
  __shared__ unsigned long long sb[64], sl[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sb[i] = sl[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < F.n; i += (int64_t)gridDim.x * blockDim.x) {
    int L = F.level[i];
    if (L < max_levels) {
      atomicAdd(&sb[L], 1ull);
      if (F.first_child[i] < 0) atomicAdd(&sl[L], 1ull);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < max_levels; i += blockDim.x) {
    if (sb[i]) atomicAdd(&blocks[i], sb[i]);
    if (sl[i]) atomicAdd(&leaves[i], sl[i]);
  }
}

struct LeafLoad {
  const int16_t* level;
  const int32_t* fc;
  int L;
  __device__ int64_t operator()(int64_t i) const { return (level[i] == L) & (fc[i] < 0); }
};
struct CompactStore {
  int32_t* out;
  __device__ void operator()(int64_t i, int64_t e, int64_t v) const {
    if (v) out[e] = (int32_t)i;
  }
};

struct MarkCountLoad {
  ForestC F;
  int L, leaf_only, mark;
  __device__ int64_t operator()(int64_t i) const {
    return F.level[i] == L && (!leaf_only || F.first_child[i] < 0) && F.marks[i] == mark;
  }
};
struct NullStore {
  __device__ void operator()(int64_t, int64_t, int64_t) const {}
};

// MARKED leaves at L (flag 1) + INTERMEDIATE anywhere at L (side flag)
struct SplitLoad {
  ForestC F;
  int L;
  int64_t* inter_flag;
  __device__ int64_t operator()(int64_t i) const {
    // unconditional loads (issued together)
    const int lv = F.level[i];
    const int8_t m = F.marks[i];
    const int32_t fc = F.first_child[i];
    if (lv != L) return 0;
    if (m == OW_INTERMEDIATE) atomicExch((unsigned long long*)inter_flag, 1ull);
    return fc < 0 && m == OW_MARKED;
  }
};

struct FlagLoad {
  const uint8_t* flag;
  __device__ int64_t operator()(int64_t i) const { return flag[i] != 0; }
};

// Split list[0..m) (ascending ids): children ids base + 2^D * r + ci with
// coords 2c + bits(ci); parent mark reset (forest.py:300-329).
__global__ void k_split(ow_forest f, const int32_t* __restrict__ list, int64_t m, int64_t base) {
  ow_pdl_wait();
  const int nc = 1 << f.dim;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * nc) return;
  int64_t r = t / nc;
  int ci = (int)(t % nc);
  int p = list[r];
  int64_t id = base + t;
  f.d_level[id] = (int16_t)(f.d_level[p] + 1);
  for (int a = 0; a < f.dim; ++a) f.d_coord[a][id] = 2 * f.d_coord[a][p] + ((ci >> a) & 1);
  f.d_parent[id] = p;
  f.d_first_child[id] = -1;
  f.d_marks[id] = OW_NONE;
  if (ci == 0) {
    f.d_first_child[p] = (int32_t)(base + r * nc);
    f.d_marks[p] = OW_NONE;
  }
}

// 2:1 violators among the face-adjacent leaves of frontier blocks
// [f0, f1): a coarser leaf more than one level above (forest.py:351-370).
__global__ void k_violators(ForestC F, int64_t f0, int64_t f1, uint8_t* flag) {
  ow_pdl_wait();
  const int sides = 2 * F.dim;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (f1 - f0) * sides) return;
  int64_t id = f0 + t / sides;
  int s = (int)(t % sides);
  int lv = F.level[id];
  int32_t c[3] = {F.coord[0][id], F.dim > 1 ? F.coord[1][id] : 0, F.dim > 2 ? F.coord[2][id] : 0};
  int32_t nc[3];
  if (!side_target(F, lv, c, s, nc)) return;
  int depth;
  int node = locate(F, lv, nc, &depth);
  if (F.first_child[node] < 0 && depth < lv - 1) flag[node] = 1;
}

// a mark that counts as MARKED in a propagation round: MARKED, or a round tag
// of an earlier round of the device loop (3 <= m < below, ow_propagate_dev)
__device__ __forceinline__ bool counts_marked(int8_t m, int below) {
  return m == OW_MARKED || (m >= 3 && m < below);
}

// any MARKED leaf on the face of region (L, nc) facing the query block
__device__ bool side_has_marked(const ForestC& F, int L, const int32_t* nc, int s, int below = 0) {
  int depth;
  int node = locate(F, L, nc, &depth);
  if (F.first_child[node] < 0) return counts_marked(F.marks[node], below);
  const int ax = s >> 1;
  const int want = (s & 1) ? 0 : 1;  // neighbour on + side: its children on the min face
  int stack[64];
  int sp = 0;
  stack[sp++] = node;
  while (sp) {
    int b = stack[--sp];
    int fc = F.first_child[b];
    if (fc < 0) {
      if (counts_marked(F.marks[b], below)) return true;
      continue;
    }
    for (int ci = (1 << F.dim) - 1; ci >= 0; --ci)
      if (((ci >> ax) & 1) == want && sp < 64) stack[sp++] = fc + ci;
  }
  return false;
}

__global__ void k_prop_gather(ForestC F, const int32_t* __restrict__ leaves, int64_t n) {
  ow_pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int id = leaves[i];
  if (F.marks[id] != OW_NONE) return;
  int L = F.level[id];
  int32_t c[3] = {F.coord[0][id], F.dim > 1 ? F.coord[1][id] : 0, F.dim > 2 ? F.coord[2][id] : 0};
  for (int s = 0; s < 2 * F.dim; ++s) {
    int32_t nc[3];
    if (!side_target(F, L, c, s, nc)) continue;
    if (side_has_marked(F, L, nc, s)) {
      F.marks[id] = OW_INTERMEDIATE;
      return;
    }
  }
}

__global__ void k_prop_promote(int8_t* marks, const int32_t* __restrict__ leaves, int64_t n) {
  ow_pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int id = leaves[i];
  if (marks[id] == OW_INTERMEDIATE) marks[id] = OW_MARKED;
}

int split_list(ow_ctx* ctx, ow_forest* f, const int32_t* list, int64_t m, cudaStream_t s) {
  const int nc = 1 << f->dim;
  int64_t need = f->n_blocks + (int64_t)nc * m;
  if (need > (int64_t)INT32_MAX) {
    ow_set_error("forest exceeds 2^31 blocks");
    return OW_ERR_CAPACITY;
  }
  if (need > f->capacity) {
    if (!f->grow) {
      ow_set_error("forest capacity %lld < %lld and no grow callback", (long long)f->capacity, (long long)need);
      return OW_ERR_CAPACITY;
    }
    if (f->grow(f->grow_user, f, need) != 0 || f->capacity < need) {
      ow_set_error("forest grow callback failed (need %lld blocks)", (long long)need);
      return OW_ERR_INTERNAL;
    }
  }
  ow_launch(k_split, ow_blocks(m * nc, 256), 256, 0, s, *f, list, m, f->n_blocks);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  f->n_blocks = need;
  return OW_OK;
}

}  // namespace

extern "C" int ow_forest_leaves(ow_ctx* ctx, const ow_forest* f, int32_t level, int32_t* d_out, int64_t* out_n,
                                void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  OW_TRY(scan01(ctx, LeafLoad{f->d_level, f->d_first_child, level}, CompactStore{d_out}, f->n_blocks,
              ctx->d_small + 8, s));
  return ow_readback(ctx, ctx->d_small + 8, 1, out_n, s);
}

extern "C" int ow_forest_level_counts(ow_ctx* ctx, const ow_forest* f, int64_t* out_blocks, int64_t* out_leaves,
                                      int32_t max_levels, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (max_levels > 28) max_levels = 28;
  OW_CUDA(cudaMemsetAsync(ctx->d_small, 0, 64 * 8, s));
  ForestC F = make_forestc(f);
  ow_launch(k_level_counts, ow_blocks(F.n, 256, 2 * OW_SMS), 256, 0, s, F, max_levels, (unsigned long long*)ctx->d_small,
                                                                 (unsigned long long*)ctx->d_small + 32);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  int64_t h[64];
  OW_TRY(ow_readback(ctx, ctx->d_small, 64, h, s));
  for (int i = 0; i < max_levels; ++i) {
    out_blocks[i] = h[i];
    out_leaves[i] = h[32 + i];
  }
  return OW_OK;
}

extern "C" int ow_forest_count_marks(ow_ctx* ctx, const ow_forest* f, int32_t level, int32_t leaf_only,
                                     int32_t mark, int64_t* out_n, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  OW_TRY(scan01(ctx, MarkCountLoad{make_forestc(f), level, leaf_only, mark}, NullStore{}, f->n_blocks,
              ctx->d_small + 8, s));
  return ow_readback(ctx, ctx->d_small + 8, 1, out_n, s);
}

extern "C" int ow_forest_cell_centers(ow_ctx* ctx, const ow_forest* f, const int32_t* d_ids, int64_t n,
                                      float* d_out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) return OW_OK;
  const int C = f->dim == 2 ? 16 : 64;
  ow_launch(k_cell_centers, ow_blocks(n * C, 256), 256, 0, s, make_forestc(f), d_ids, n, d_out);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

extern "C" int ow_propagate_marks(ow_ctx* ctx, const ow_forest* f, const int32_t* d_leaves, int64_t n_leaves,
                                  int32_t rounds, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n_leaves <= 0 || rounds <= 0) return OW_OK;
  ForestC F = make_forestc(f);
  OW_PROF_BEGIN(ctx, PROF_PROP, s);
  for (int r = 0; r < rounds; ++r) {
    ow_launch(k_prop_gather, ow_blocks(n_leaves, 128), 128, 0, s, F, d_leaves, n_leaves);
    ow_launch(k_prop_promote, ow_blocks(n_leaves, 256), 256, 0, s, F.marks, d_leaves, n_leaves);
    ctx->launches += 2;
  }
  OW_PROF_END(ctx, PROF_PROP, s);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

static int refine_marked_impl(ow_ctx* ctx, ow_forest* f, int32_t level, int64_t* out_split, int64_t* out_marked,
                              cudaStream_t s);

extern "C" int ow_refine_marked(ow_ctx* ctx, ow_forest* f, int32_t level, int64_t* out_split, void* stream) {
  int64_t m;
  return ow_refine_marked_counted(ctx, f, level, out_split, &m, (cudaStream_t)stream);
}

int ow_refine_marked_counted(ow_ctx* ctx, ow_forest* f, int32_t level, int64_t* out_split, int64_t* out_marked,
                             cudaStream_t s) {
  OW_PROF_BEGIN(ctx, PROF_REFINE, s);
  int st = refine_marked_impl(ctx, f, level, out_split, out_marked, s);
  OW_PROF_END(ctx, PROF_REFINE, s);
  return st;
}

static int refine_marked_impl(ow_ctx* ctx, ow_forest* f, int32_t level, int64_t* out_split, int64_t* out_marked,
                              cudaStream_t s) {
  int64_t* small = ctx->d_small;
  void* pl;
  OW_TRY(ow_slot(ctx, SLOT_FOREST_LIST, 4 * (size_t)(f->n_blocks + 1), s, &pl));
  OW_CUDA(cudaMemsetAsync(small + 9, 0, 8, s));
  OW_TRY(scan01(ctx, SplitLoad{make_forestc(f), level, small + 9}, CompactStore{(int32_t*)pl}, f->n_blocks, small + 8, s));
  int64_t h[2];
  OW_TRY(ow_readback(ctx, small + 8, 2, h, s));
  if (h[1]) {
    ow_set_error("level %d still carries intermediate marks; finish propagation first", level);
    return OW_ERR_INVALID;
  }
  int64_t m = h[0], n_split = m;
  *out_split = 0;
  *out_marked = m;
  if (m == 0) return OW_OK;
  if (level >= f->max_level) {
    ow_set_error("refinement beyond max level %d", f->max_level);
    return OW_ERR_INVALID;
  }
  int64_t f0 = f->n_blocks;
  OW_TRY(split_list(ctx, f, (const int32_t*)pl, m, s));
  while (f->n_blocks > f0) {
    int64_t f1 = f->n_blocks;
    void* pf;
    OW_TRY(ow_slot(ctx, SLOT_FOREST_FLAG, (size_t)f->capacity, s, &pf));
    OW_CUDA(cudaMemsetAsync(pf, 0, (size_t)f1, s));
    ForestC F = make_forestc(f);
    ow_launch(k_violators, ow_blocks((f1 - f0) * 2 * f->dim, 256), 256, 0, s, F, f0, f1, (uint8_t*)pf);
    OW_LAUNCHED(ctx);
    OW_CHECK_LAUNCH();
    OW_TRY(ow_slot(ctx, SLOT_FOREST_LIST, 4 * (size_t)(f1 + 1), s, &pl));
    OW_TRY(scan01(ctx, FlagLoad{(const uint8_t*)pf}, CompactStore{(int32_t*)pl}, f1, small + 8, s));
    OW_TRY(ow_readback(ctx, small + 8, 1, h, s));
    int64_t v = h[0];
    if (v == 0) break;
    n_split += v;
    f0 = f1;
    OW_TRY(split_list(ctx, f, (const int32_t*)pl, v, s));
  }
  *out_split = n_split;
  return OW_OK;
}

// ---------------------------------------------------------------------------
// Device-driven variants for the native driver: counts stay in device memory
// (launches are sized from host upper bounds and read the exact count on the
// device), so a whole level runs without a host round trip.
// ---------------------------------------------------------------------------
namespace {

// refine state (int64, 64 words per pass): [0] intermediate-mark flag,
// [1] capacity overflow, [2] MARKED leaves split, [3] blocks split in total,
// [4] frontier start to resume from on the host, [5] MARKED list did not fit,
// [RS_NR + k] block count before split k, [RS_CR + k] length of split list k
// (layout constants RS_* in ow_common.cuh)

// refine state init (CTA 0) and the violator flags cleared (grid-stride, 16
// bytes per store: flag is 8-byte aligned scratch of cap + 8 bytes)
// (+ the deferred last promote of the level's propagation rounds: round tags
// of the leaves -> MARKED, ow_propagate_dev)
__global__ void k_rs_init(int64_t* st, int64_t n, const int64_t* nd, uint8_t* flag, int64_t cap,
                          int8_t* marks, const int32_t* __restrict__ promote_leaves, const int64_t* promote_n) {
  ow_pdl_wait();
  if (promote_leaves) {
    const int64_t pn = *promote_n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pn; i += (int64_t)gridDim.x * blockDim.x) {
      const int id = promote_leaves[i];
      if (marks[id] >= OW_INTERMEDIATE) marks[id] = OW_MARKED;
    }
  }
  if (blockIdx.x == 0) {
    if (nd) n = *nd;
    for (int i = threadIdx.x; i < RS_WORDS; i += blockDim.x) st[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      st[RS_NR] = n;
      st[RS_RESUME] = n;
    }
  }
  const int64_t words = (cap + 15) / 16;
  uint4* f4 = reinterpret_cast<uint4*>(flag);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
    f4[i] = make_uint4(0u, 0u, 0u, 0u);
}

// Split k of a device-driven refine: list k (length cnt[k]) splits into ids
// n[k] + 2^D r + ci; one thread publishes n[k+1].  A list that does not fit
// the capacity is dropped (n[k+1] = n[k]) and the frontier to resume from is
// recorded; the MARKED list (k = 0) is not split beyond max_level.
// next_leaves / next_count (device-resident loop, k = 0): the children of
// this split are exactly the leaves of level + 1 at the next marking pass, a
// contiguous id range in ascending order — written here, no compaction
__global__ void k_split_ring(ow_forest f, const int32_t* __restrict__ list, int64_t* st, int k, int beyond_max,
                             int64_t* nb_out, int32_t* next_leaves, int64_t* next_count) {
  ow_pdl_wait();
  const int nc = 1 << f.dim;
  const int64_t base = st[RS_NR + k];
  int64_t m = st[RS_CR + k];
  const bool over = st[RS_OVER] || base + nc * m > f.capacity;
  if (k == 0 && beyond_max) m = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (k == 0) st[RS_MARKED] = st[RS_CR];
    if (over) {
      if (m > 0 && !st[RS_OVER]) {
        st[RS_OVER] = 1;
        st[RS_OVER_FIRST] = k == 0;
        st[RS_RESUME] = k > 0 ? st[RS_NR + k - 1] : base;
      }
      st[RS_NR + k + 1] = base;
    } else {
      st[RS_NR + k + 1] = base + nc * m;
      st[RS_SPLITS] += m;
      st[RS_RESUME] = base;  // frontier of the newest children
    }
    if (nb_out) *nb_out = st[RS_NR + k + 1];
    if (next_count) *next_count = over ? 0 : nc * m;
  }
  if (over) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m * nc; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / nc;
    const int ci = (int)(t % nc);
    const int p = list[r];
    const int64_t id = base + t;
    if (next_leaves) next_leaves[t] = (int32_t)id;
    f.d_level[id] = (int16_t)(f.d_level[p] + 1);
    for (int a = 0; a < f.dim; ++a) f.d_coord[a][id] = 2 * f.d_coord[a][p] + ((ci >> a) & 1);
    f.d_parent[id] = p;
    f.d_first_child[id] = -1;
    f.d_marks[id] = OW_NONE;
    if (ci == 0) {
      f.d_first_child[p] = (int32_t)(base + r * nc);
      f.d_marks[p] = OW_NONE;
    }
  }
}

// 2:1 violators around the frontier [n[k-1], n[k]) read on the device (grid-stride)
// (scan_n: the length the following flag compaction scans, 0 when the
// previous sweep split nothing — then no block can be flagged)
__global__ void k_violators_dev(ForestC F, const int64_t* st, int k, uint8_t* flag, int64_t* scan_n) {
  ow_pdl_wait();
  const int sides = 2 * F.dim;
  const int64_t f0 = st[RS_NR + k - 1], f1 = st[RS_NR + k];
  if (blockIdx.x == 0 && threadIdx.x == 0) *scan_n = f1 > f0 ? f1 : 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (f1 - f0) * sides;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = f0 + t / sides;
    const int s = (int)(t % sides);
    const int lv = F.level[id];
    int32_t c[3] = {F.coord[0][id], F.dim > 1 ? F.coord[1][id] : 0, F.dim > 2 ? F.coord[2][id] : 0};
    int32_t nc[3];
    if (!side_target(F, lv, c, s, nc)) continue;
    int depth;
    const int node = locate(F, lv, nc, &depth);
    if (F.first_child[node] < 0 && depth < lv - 1) flag[node] = 1;
  }
}

struct FlagCompactClear {  // compaction that also clears the flags it consumed
  int32_t* out;
  uint8_t* flag;
  __device__ void operator()(int64_t i, int64_t e, int64_t v) const {
    if (v) {
      out[e] = (int32_t)i;
      flag[i] = 0;
    }
  }
};

// One propagation round of the device loop (nearwall.py:321-366) without
// its promote step: a NONE leaf with a face neighbour that counts as MARKED
// (MARKED, or tagged in an earlier round) gets this round's tag 3 + r, which
// the same round never counts — so every round sees exactly the marks the
// reference's round does, and one promote after the last round turns the
// tags into MARKED (rounds + 1 launches instead of 2 rounds).
// (levels of at most side_max leaves: a thread per (leaf, side), so a leaf's
// up to 2D neighbour descents run in parallel instead of one after another;
// every side that finds a marked neighbour writes the same tag, and
// counts_marked never counts this round's tag, so the result is the per-leaf
// loop's.  Larger levels keep a thread per leaf: they fill the GPU anyway
// and the per-leaf early exit saves descents)
__global__ void k_prop_gather_dev(ForestC F, const int32_t* __restrict__ leaves, const int64_t* n, int tag,
                                  int below, int64_t side_max) {
  ow_pdl_wait();
  const int64_t nn = *n;
  if (nn <= side_max) {
    const int ns = 2 * F.dim;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn * ns;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int id = leaves[i / ns];
      const int sd = (int)(i % ns);
      if (F.marks[id] != OW_NONE) continue;
      const int L = F.level[id];
      int32_t c[3] = {F.coord[0][id], F.dim > 1 ? F.coord[1][id] : 0, F.dim > 2 ? F.coord[2][id] : 0};
      int32_t nc[3];
      if (!side_target(F, L, c, sd, nc)) continue;
      if (side_has_marked(F, L, nc, sd, below)) F.marks[id] = (int8_t)tag;
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
    const int id = leaves[i];
    if (F.marks[id] != OW_NONE) continue;
    const int L = F.level[id];
    int32_t c[3] = {F.coord[0][id], F.dim > 1 ? F.coord[1][id] : 0, F.dim > 2 ? F.coord[2][id] : 0};
    for (int s = 0; s < 2 * F.dim; ++s) {
      int32_t nc[3];
      if (!side_target(F, L, c, s, nc)) continue;
      if (side_has_marked(F, L, nc, s, below)) {
        F.marks[id] = (int8_t)tag;
        break;
      }
    }
  }
}

__global__ void k_prop_promote_dev(int8_t* marks, const int32_t* __restrict__ leaves, const int64_t* n) {
  ow_pdl_wait();
  const int64_t nn = *n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
    const int id = leaves[i];
    if (marks[id] >= OW_INTERMEDIATE) marks[id] = OW_MARKED;  // (INTERMEDIATE or this level's round tags)
  }
}

}  // namespace

// leaves at `level` into d_out, count into *d_count (device; no readback)
// (d_nb: the block count lives on the device; the scan then covers the capacity)
int ow_forest_leaves_dev(ow_ctx* ctx, const ow_forest* f, int32_t level, int32_t* d_out, int64_t* d_count,
                         cudaStream_t s, const int64_t* d_nb) {
  if (d_nb)
    return scan01(ctx, LeafLoad{f->d_level, f->d_first_child, level}, CompactStore{d_out}, f->capacity, d_count, s,
                  d_nb);
  return scan01(ctx, LeafLoad{f->d_level, f->d_first_child, level}, CompactStore{d_out}, f->n_blocks, d_count, s);
}

// largest level whose propagation gather runs a thread per (leaf, side)
// (OW_PROP_SIDES_MAX, A/B; 0: always per leaf).  tools/ab_prop.sh on one
// B200, per (leaf, side) on every level vs per leaf: C1 0.287 -> 0.252 ms,
// C2 0.320 -> 0.311, C3 1.454 -> 1.431, C4 2.050 -> 2.034, but C5 (levels of
// 262 144 and 178 112 leaves) 3.559 -> 3.574
static int64_t prop_side_max() {
  static const int64_t v = [] {
    const char* e = getenv("OW_PROP_SIDES_MAX");
    return e ? (int64_t)atoll(e) : (int64_t)131072;
  }();
  return v;
}

int ow_propagate_dev(ow_ctx* ctx, const ow_forest* f, const int32_t* d_leaves, const int64_t* d_n, int64_t n_bound,
                     int32_t rounds, cudaStream_t s, bool tags, bool defer_promote) {
  if (n_bound <= 0 || rounds <= 0) return OW_OK;
  ForestC F = make_forestc(f);
  OW_PROF_BEGIN(ctx, PROF_PROP, s);
  // tags (a fresh forest, no INTERMEDIATE marks before the level's marking):
  // round tags 3 .. 3 + rounds - 1 stay inside int8 (a promote every 100
  // rounds restarts them; the reference's rounds are 1 + floor(d / block
  // length)).  Else the reference's round as is: INTERMEDIATE, then promote.
  for (int r = 0; r < rounds; ++r) {
    const int tag = tags ? 3 + r % 100 : OW_INTERMEDIATE;
    ow_launch(k_prop_gather_dev, ow_blocks(n_bound * 2 * f->dim, 128, 16 * OW_SMS), 128, 0, s, F, d_leaves, d_n, tag,
              tags ? tag : 0, prop_side_max());
    ctx->launches += 1;
    if (!tags || r % 100 == 99 || (r + 1 == rounds && !defer_promote)) {
      ow_launch(k_prop_promote_dev, ow_blocks(n_bound, 256, 8 * OW_SMS), 256, 0, s, F.marks, d_leaves, d_n);
      ctx->launches += 1;
    }
  }
  OW_PROF_END(ctx, PROF_PROP, s);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

// refine_marked + 2:1 rebalance (forest.py:300-370) without host round trips:
// split the MARKED leaves at `level`, then `iters` violator sweeps (each
// splits the coarser leaves more than one level above a new block).  The host
// reads d_st afterwards: intermediate marks / beyond-max-level are errors; an
// overflow or violators left after the last sweep are finished by
// ow_rebalance_host from st[RS_RESUME] (or by a synchronous refine when the
// MARKED list itself did not fit).
//
// d_nb (device-resident level loop): the block count is read from and the
// final count written back to *d_nb, so f->n_blocks is stale until the caller
// reads it.
int ow_refine_dev(ow_ctx* ctx, ow_forest* f, int32_t level, int32_t iters, int64_t* d_st, cudaStream_t s,
                  int64_t* d_nb, int32_t* next_leaves, int64_t* next_count, const int32_t* promote_leaves,
                  const int64_t* promote_n) {
  if (iters > RS_MAX_ITERS) iters = RS_MAX_ITERS;
  const int nc = 1 << f->dim;
  const int64_t n = f->n_blocks, cap = f->capacity;
  void *pl, *pf;
  OW_TRY(ow_slot(ctx, SLOT_FOREST_LIST, 4 * (size_t)(cap + 1), s, &pl));
  OW_TRY(ow_slot(ctx, SLOT_FOREST_FLAG, (size_t)cap + 16, s, &pf));
  OW_PROF_BEGIN(ctx, PROF_REFINE, s);
  ow_launch(k_rs_init, ow_blocks((cap + 15) / 16, 256, 2 * OW_SMS), 256, 0, s, d_st, n, d_nb, (uint8_t*)pf, cap,
            f->d_marks, promote_leaves, promote_n);
  OW_TRY(scan01(ctx, SplitLoad{make_forestc(f), level, d_st + RS_INTER}, CompactStore{(int32_t*)pl},
                d_nb ? cap : n, d_st + RS_CR, s, d_nb));
  const ow_forest fv = *f;
  const int sg = ow_blocks(cap * nc, 256, 8 * OW_SMS);
  ow_launch(k_split_ring, sg, 256, 0, s, fv, (const int32_t*)pl, d_st, 0, level >= f->max_level,
            iters == 0 ? d_nb : nullptr, next_leaves, next_count);
  ctx->launches += 2;
  ForestC F = make_forestc(f);
  F.n = cap;
  for (int k = 1; k <= iters; ++k) {
    int64_t* scan_n = ctx->d_small + 53;
    ow_launch(k_violators_dev, ow_blocks(cap * 2 * f->dim, 256, 8 * OW_SMS), 256, 0, s, F, d_st, k, (uint8_t*)pf,
              scan_n);
    // violator flags of blocks [0, n[k]) (n[k] on the device; 0 after a sweep without splits)
    OW_TRY(scan01(ctx, FlagLoad{(const uint8_t*)pf}, FlagCompactClear{(int32_t*)pl, (uint8_t*)pf}, cap,
                  d_st + RS_CR + k, s, scan_n));
    ow_launch(k_split_ring, sg, 256, 0, s, fv, (const int32_t*)pl, d_st, k, 0, k == iters ? d_nb : nullptr,
              (int32_t*)nullptr, (int64_t*)nullptr);
    ctx->launches += 2;
  }
  OW_PROF_END(ctx, PROF_REFINE, s);
  OW_CHECK_LAUNCH();
  return OW_OK;
}

// finish a rebalance on the host loop from frontier [f0, n_blocks) (fallback of
// ow_refine_dev after an overflow or a cascade deeper than its sweeps)
int ow_rebalance_host(ow_ctx* ctx, ow_forest* f, int64_t f0, int64_t* n_split, cudaStream_t s) {
  int64_t* small = ctx->d_small;
  int64_t h[1];
  while (f->n_blocks > f0) {
    const int64_t f1 = f->n_blocks;
    void *pf, *pl;
    OW_TRY(ow_slot(ctx, SLOT_FOREST_FLAG, (size_t)f->capacity + 8, s, &pf));
    OW_CUDA(cudaMemsetAsync(pf, 0, (size_t)f1, s));
    ForestC F = make_forestc(f);
    ow_launch(k_violators, ow_blocks((f1 - f0) * 2 * f->dim, 256), 256, 0, s, F, f0, f1, (uint8_t*)pf);
    OW_LAUNCHED(ctx);
    OW_CHECK_LAUNCH();
    OW_TRY(ow_slot(ctx, SLOT_FOREST_LIST, 4 * (size_t)(f1 + 1), s, &pl));
    OW_TRY(scan01(ctx, FlagLoad{(const uint8_t*)pf}, CompactStore{(int32_t*)pl}, f1, small + 8, s));
    OW_TRY(ow_readback(ctx, small + 8, 1, h, s));
    if (h[0] == 0) break;
    *n_split += h[0];
    f0 = f1;
    OW_TRY(split_list(ctx, f, (const int32_t*)pl, h[0], s));
  }
  return OW_OK;
}
