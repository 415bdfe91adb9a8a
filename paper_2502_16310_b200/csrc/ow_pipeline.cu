// Native per-level near-wall driver (refine_near_wall, nearwall.py:430-491)
// and root-grid initialisation (init_root_grid, forest.py:48-81, 405-409).
//
// The reference drives the level loop from Python; the B200 build runs it in
// C++ over the same library entry points, so a whole geometry-to-grid pass is
// one host call: bins (once per (geometry, grid); the reference rebuilds an
// identical structure every level) -> per level {leaves, marking, propagation,
// refinement} with device-event stage timings.  The only host round trips are
// the scalars the algorithm needs to size the next step (leaf count, marks,
// split / violator counts).
#include <math.h>
#include <stddef.h>
#include <string.h>

#include "ow_scan.cuh"

namespace {

using ow::scan;

__global__ void k_root_init(ow_forest f, int64_t r, int64_t* face_summary) {
  ow_pdl_wait();
  if (face_summary && blockIdx.x == 0 && threadIdx.x == 0) ow_face_summary_init_words(face_summary);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r) return;
  int64_t rem = i;
  for (int a = 0; a < f.dim; ++a) {
    f.d_coord[a][i] = (int32_t)(rem % f.root[a]);
    rem /= f.root[a];
  }
  f.d_level[i] = 0;
  f.d_parent[i] = -1;
  f.d_first_child[i] = -1;
  f.d_marks[i] = 0;
}

struct StageEvents {
  cudaEvent_t ev[OW_MAX_PASSES][5];
  bool used[OW_MAX_PASSES][5];
};

int record(StageEvents* se, int lv, int k, cudaStream_t s, bool skip = false) {
  if (skip) return OW_OK;
  if (!se->ev[lv][k]) OW_CUDA(cudaEventCreate(&se->ev[lv][k]));
  OW_CUDA(cudaEventRecord(se->ev[lv][k], s));
  se->used[lv][k] = true;
  return OW_OK;
}

// batch_ranges (binning.py:190-197) running totals: first batch whose total
// overflows the capacity, for the reference's CapacityError message
int64_t overflow_total(const int32_t* h_counts, int64_t n_bins, int64_t bin_fraction, int64_t capacity) {
  int64_t bf = bin_fraction < n_bins ? bin_fraction : n_bins;
  if (bf < 1) bf = 1;
  const int64_t per = (n_bins + bf - 1) / bf;
  int64_t acc = 0;
  for (int64_t s0 = 0; s0 < n_bins; s0 += per) {
    const int64_t s1 = s0 + per < n_bins ? s0 + per : n_bins;
    for (int64_t b = s0; b < s1; ++b) acc += h_counts[b];
    if (acc > capacity) break;
  }
  return acc;
}

// the level loop's statistics cleared and (device-resident loop) the block
// count set, one launch
// (+ the device-sized pass's bin counts and count words, k_bins_init's work)
__global__ void k_loop_init(unsigned long long* stats, int n_stats, int64_t* d_nb, int64_t nb, int32_t* counts,
                            int64_t n_bins, int64_t* small) {
  ow_pdl_wait();
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < n_stats; i += blockDim.x) stats[i] = 0ull;
    if (threadIdx.x == 0 && d_nb) *d_nb = nb;
    if (small && threadIdx.x < 8) small[threadIdx.x] = (threadIdx.x == 1 || threadIdx.x == 3) ? -1 : 0;
  }
  if (counts)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_bins; i += (int64_t)gridDim.x * blockDim.x)
      counts[i] = 0;
}

// ---- multi-GPU marking shards ("balanced by work") --------
// Work of a leaf block: 1 + the faces of the bin holding its centre (the
// marking cost per cell is the size of its bin's face list; the centre's bin
// stands for the block's 4^D cells).  The exclusive prefix of the weights
// splits the level's leaves into `world` contiguous slices of equal work.
struct LeafWork {
  ForestC F;
  GridC g;
  const int32_t* leaves;
  const int32_t* counts;  // null: naive strategy (every block weighs the same)
  const int64_t* d_n;
  int level;
  __device__ int64_t operator()(int64_t i) const {
    if (i >= *d_n) return 0;
    if (!counts) return 1;
    const int id = leaves[i];
    int64_t bin = 0, mul = 1;
    for (int a = 0; a < F.dim; ++a) {
      const double q = block_len(F, a, level);
      const float c = __double2float_rn(DADD(F.dmin[a], DMUL(DADD((double)F.coord[a][id], 0.5), q)));
      bin += (int64_t)bin_axis(c, g.min32[a], g.len32[a], g.B) * mul;
      mul *= g.B;
    }
    return 1 + counts[bin];
  }
};
struct WorkPrefix {
  int64_t* e;
  const int64_t* d_n;
  __device__ void operator()(int64_t i, int64_t ex, int64_t) const {
    if (i < *d_n) e[i] = ex;
  }
};
// slice[0..1) of `rank`: positions whose work prefix lies in
// [total rank / world, total (rank + 1) / world) (the same formula on every
// rank, so the slices tile the leaves)
__global__ void k_slice_bounds(const int64_t* __restrict__ e, const int64_t* d_n, const int64_t* d_total, int rank,
                               int world, int64_t* slice) {
  ow_pdl_wait();
  if (threadIdx.x != 0) return;
  const int64_t n = *d_n, total = *d_total;
  auto first_geq = [&](int64_t t) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (e[mid] < t) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  slice[0] = rank == 0 ? 0 : first_geq(total * rank / world);
  slice[1] = rank == world - 1 ? n : first_geq(total * (rank + 1) / world);
}

// Device-resident level loop: per pass, the words the host needs from the
// refine ring state and the marking stats, gathered for one readback.
constexpr int SUM_W = 13;  // [0..6) RS_INTER..RS_OVER_FIRST, [6] final blocks, [7] last sweep's list, [8..13) stats
constexpr int DRV_RETRY = 1000;  // internal: rerun the pass with per-level host sync

// the SUM_W summary words of pass p from its ring state and statistics
template <class Out>
__device__ __forceinline__ void drv_summary_pass(const int64_t* drv, const unsigned long long* stats, int p, Out o) {
  const int64_t* rs = drv + 72 * p + 8;
  const int it = refine_sweeps(p);
  for (int k = 0; k < 6; ++k) o[k] = rs[k];
  o[6] = rs[RS_NR + it + 1];
  o[7] = refine_sweeps_exact(p) ? 0 : rs[RS_CR + it];  // (a cascade the sweeps may not have finished)
  for (int k = 0; k < 5; ++k) o[8 + k] = (int64_t)stats[MARK_STATS * p + k];
}

__global__ void k_drv_summary(const int64_t* drv, const unsigned long long* stats, int passes, int64_t* sum) {
  ow_pdl_wait();
  for (int p = threadIdx.x; p < passes; p += blockDim.x) drv_summary_pass(drv, stats, p, sum + SUM_W * p);
}

}  // namespace

namespace {
// root grid (+ the fused pass's face summary words initialised in the same launch)
int init_root(ow_ctx* ctx, ow_forest* f, void* stream, int64_t* face_summary) {
  cudaStream_t s = (cudaStream_t)stream;
  int64_t r = 1;
  for (int a = 0; a < f->dim; ++a) r *= f->root[a];
  if (f->dim < 2 || f->dim > 3 || r < 1 || r > f->capacity) {
    ow_set_error("init_root_grid: bad root grid or capacity (%lld roots, capacity %lld)", (long long)r,
                 (long long)f->capacity);
    return OW_ERR_INVALID;
  }
  ow_launch(k_root_init, ow_blocks(r, 256), 256, 0, s, *f, r, face_summary);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  f->n_blocks = r;
  return OW_OK;
}
}  // namespace

extern "C" int ow_forest_init_root(ow_ctx* ctx, ow_forest* f, void* stream) {
  return init_root(ctx, f, stream, nullptr);
}

namespace {
// the device-resident loop's summary words (SUM_W per pass + the deepest
// level's leaf count): host checks and results; DRV_RETRY when the forest
// outgrew its capacity or a 2:1 cascade outran the device sweeps
int drv_apply(ow_ctx* ctx, ow_forest* f, const int64_t* h, int passes, ow_nearwall_result* out) {
  for (int level = 0; level < passes; ++level) {
    const int64_t* w = h + SUM_W * level;
    if (w[RS_INTER]) {
      ow_set_error("level %d still carries intermediate marks; finish propagation first", level);
      return OW_ERR_INVALID;
    }
    if (w[RS_MARKED] > 0 && level >= f->max_level) {
      ow_set_error("refinement beyond max level %d", f->max_level);
      return OW_ERR_INVALID;
    }
    if (w[RS_OVER] || w[7] > 0) return DRV_RETRY;
    f->n_blocks = w[6];
    out->marked_refined[level] = w[RS_MARKED];
    out->n_split[level] = w[RS_SPLITS];
    out->marked_detected[level] = w[8];
    out->tests[level] = w[9];
    out->evaluated[level] = w[10];
    out->sphere_tests[level] = w[11];
    out->box_culls[level] = w[12];
  }
  ctx->drv_spec_nl = h[SUM_W * passes];
  return OW_OK;
}

// The level loop.  dev = false: the block count returns to the host after each
// refinement (exact launch sizes; capacity overflows and deep 2:1 cascades are
// finished on the host path, which grows the forest).  dev = true (fused pass
// from a fresh root grid, one rank): every launch is sized by the forest
// capacity and reads the live block count from the device, so the whole loop
// runs without a host round trip; one readback at the end checks it, and an
// overflow or cascade returns DRV_RETRY (the caller re-initialises the root
// grid and reruns with dev = false).  In dev mode the leaves of the deepest
// level are compacted too (ctx->drv_spec_nl; -1 when not available).
int refine_driver(ow_ctx* ctx, ow_forest* f, const float* d_coords, int64_t n_faces, int64_t geom_key,
                  const ow_grid* grid, const ow_nearwall_params* p, int32_t* d_bin_ids, int64_t bin_ids_capacity,
                  int32_t* d_bin_counts, int32_t* d_bin_offsets, ow_nearwall_result* out, cudaStream_t s, bool dev) {
  ctx->drv_spec_nl = -1;
  // device-sized fused pass (g2g_device): bins are counted and emitted with
  // their entry count on the device and nothing is read back here
  const bool devpass = dev && ctx->dev_pass;
  ow_comm* comm = p->world > 1 ? p->comm : nullptr;
  if (p->world > 1 && !comm) dev = false;  // (the host exchange hook needs the leaf count on the host)
  if (comm && (comm->world != p->world || comm->rank != p->rank || !comm->open)) {
    ow_set_error("refine_near_wall: the exchange (rank %d of %d) does not match rank %d of %d or is not open",
                 comm->rank, comm->world, p->rank, p->world);
    return OW_ERR_INVALID;
  }
  memset(out, 0, sizeof(*out));
  if (p->n_levels < 1 || p->n_levels - 1 > OW_MAX_PASSES) {
    ow_set_error("n_levels must be in [1, %d], got %d", OW_MAX_PASSES + 1, p->n_levels);
    return OW_ERR_INVALID;
  }
  if (p->binned && (!grid || grid->dim != f->dim || !d_bin_ids || !d_bin_counts || !d_bin_offsets)) {
    ow_set_error("refine_near_wall: binned strategy needs a matching bin grid and bin buffers");
    return OW_ERR_INVALID;
  }
  if (!ctx->stage_events) {
    ctx->stage_events = calloc(1, sizeof(StageEvents));
    if (!ctx->stage_events) {
      ow_set_error("refine_near_wall: out of host memory");
      return OW_ERR_INTERNAL;
    }
  }
  StageEvents* se = (StageEvents*)ctx->stage_events;
  memset(se->used, 0, sizeof(se->used));
  int64_t n_bins = 1;
  if (grid)
    for (int a = 0; a < grid->dim; ++a) n_bins *= grid->bins_per_axis;
  bool have_bins = false;
  int64_t E = 0;
  const int passes = p->n_levels - 1;
  void *stats, *drv;
  OW_TRY(ow_slot(ctx, SLOT_DRV_STATS, 8 * MARK_STATS * (size_t)passes, s, &stats));
  // [72 * pass] ring state | [72 * passes] device block count | summary
  OW_TRY(ow_slot(ctx, SLOT_DRV_STATE, 8 * (72 * (size_t)passes + 16 + SUM_W * (size_t)passes), s, &drv));
  // the bin count of fill_bins with its host checks (one readback: the entry
  // count sizes the emission); in the device-resident loop it runs before the
  // loop so the loop itself has no host round trip
  auto count_bins = [&]() -> int {
    int64_t outside = -1;
    OW_TRY(ow_fill_bins_count(ctx, grid, d_coords, n_faces, p->spacing, d_bin_counts, &E, &outside, s));
    if (outside >= 0) {
      ow_set_error("face sample outside binning domain (face %lld)", (long long)outside);
      return OW_ERR_INVALID;
    }
    const int64_t capacity = p->overlap_factor * n_faces;
    if (E > capacity || E > bin_ids_capacity) {
      int32_t* h = (int32_t*)malloc(4 * (size_t)n_bins);
      if (!h) {
        ow_set_error("refine_near_wall: out of host memory");
        return OW_ERR_INTERNAL;
      }
      cudaError_t e = cudaMemcpyAsync(h, d_bin_counts, 4 * (size_t)n_bins, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      const int64_t acc = e == cudaSuccess ? overflow_total(h, n_bins, p->bin_fraction, capacity) : E;
      free(h);
      OW_CUDA(e);
      ow_set_error("bin assignment overflow: %lld face-bin entries exceed capacity %lld (= %lld x %lld faces); "
                   "raise overlap_factor, or raise bin_fraction to shrink the per-batch indicator",
                   (long long)acc, (long long)capacity, (long long)p->overlap_factor, (long long)n_faces);
      return OW_ERR_CAPACITY;
    }
    return OW_OK;
  };
  int64_t* d_nb = dev ? (int64_t*)drv + 72 * passes : nullptr;
  int64_t* d_sum = (int64_t*)drv + 72 * passes + 8;
  // device-resident loop: its only host round trips (the bin count, the
  // face summary) happen first, so everything below runs without one and can
  // be replayed as a CUDA graph (ow_graph.cu)
  bool pre_counted = false;
  if (devpass) {
    E = ctx->dev_e_cap;  // (the bound; the count stays on the device)
  } else if (dev && p->binned && p->reuse_bins) {
    OW_TRY(record(se, 0, 0, s, ctx->no_stage_events));
    OW_TRY(count_bins());
    pre_counted = true;
  } else if (dev && ctx->faces_pending) {
    OW_TRY(ow_faces_settle(ctx, nullptr, s));
  }
  auto device_part = [&]() -> int {
  bool bins_counted = pre_counted;
  have_bins = false;
  const bool init_bins = devpass && p->binned;  // (fill_dev then skips its own init)
  ow_launch(k_loop_init, init_bins ? ow_blocks(n_bins, 256, 4 * OW_SMS) : 1, init_bins ? 256 : 128, 0, s,
            (unsigned long long*)stats, MARK_STATS * passes, dev ? d_nb : nullptr, f->n_blocks,
            init_bins ? d_bin_counts : nullptr, n_bins, init_bins ? ctx->d_small : nullptr);
  OW_LAUNCHED(ctx);
  for (int level = 0; level < passes; ++level) {
    // ---- bin_setup
    if (!(pre_counted && level == 0)) OW_TRY(record(se, level, 0, s, ctx->no_stage_events));
    bool fresh_bins = level == 0;  // chunk boxes of the bins (marking) need a rebuild
    if (p->binned && (!have_bins || !p->reuse_bins)) {
      fresh_bins = true;
      if (devpass) {
        OW_TRY(ow_fill_bins_dev(ctx, grid, d_coords, n_faces, p->spacing, d_bin_counts, d_bin_ids, d_bin_offsets, E,
                                s, level > 0 || !init_bins));
      } else {
        if (!bins_counted) OW_TRY(count_bins());
        bins_counted = false;
        OW_TRY(ow_fill_bins_emit(ctx, grid, d_bin_ids, d_bin_counts, d_bin_offsets, s));
      }
      have_bins = true;
      out->bin_entries = E;
      out->bins_built += 1;
    }
    // ---- face_detection
    if (ctx->faces_pending) OW_TRY(ow_faces_settle(ctx, nullptr, s));  // (naive strategy: no bin readback)
    OW_TRY(record(se, level, 1, s, ctx->no_stage_events));
    const int64_t n_host = dev ? f->capacity : f->n_blocks;  // bound on this level's leaves
    void* pl;
    OW_TRY(ow_slot(ctx, SLOT_DRV_LEAVES, 4 * (size_t)(n_host + 1), s, &pl));
    int64_t* dn = (int64_t*)drv + 72 * level;  // [0] leaves at level, [8..72) refine state
    int64_t* rs = dn + 8;
    unsigned long long* dst = (unsigned long long*)stats + MARK_STATS * level;
    if (comm) {
      // sharded marking on the device: slices balanced by per-leaf work, the
      // rank marks its slice, then the marks and the statistics are exchanged
      // over peer memory (ow_comm.cu) — no host round trip
      // (device-resident loop: the leaves of level >= 1 were written by the
      // previous level's split, ow_refine_dev next_leaves)
      if (level == 0 || !dev) OW_TRY(ow_forest_leaves_dev(ctx, f, level, (int32_t*)pl, dn, s, d_nb));
      void* psl;
      OW_TRY(ow_slot(ctx, SLOT_DRV_SLICE, 8 * (size_t)(n_host + 8), s, &psl));
      int64_t* wpre = (int64_t*)psl + 8;
      int64_t* slice = (int64_t*)psl;  // [0..1) slice, [2] total work
      LeafWork lw{make_forestc(f), p->binned ? make_gridc(grid) : GridC{}, (const int32_t*)pl,
                  p->binned ? d_bin_counts : nullptr, dn, level};
      OW_TRY(scan(ctx, lw, WorkPrefix{wpre, dn}, n_host, slice + 2, s));
      ow_launch(k_slice_bounds, 1, 32, 0, s, (const int64_t*)wpre, (const int64_t*)dn, (const int64_t*)(slice + 2),
                p->rank, p->world, slice);
      OW_LAUNCHED(ctx);
      OW_TRY(ow_mark_launch(ctx, f, (const int32_t*)pl, n_host, d_coords, n_faces, geom_key,
                            p->binned ? grid : nullptr, p->binned ? d_bin_ids : nullptr,
                            p->binned ? d_bin_counts : nullptr, p->binned ? d_bin_offsets : nullptr,
                            p->binned ? E : 0, p->d_spec, p->reach, dst, s, dn, !fresh_bins, slice, nullptr, level));
      OW_TRY(ow_comm_exchange_marks(ctx, comm, (const int32_t*)pl, f->d_marks, slice, dn, n_host, dst, 5, s));
    } else if (p->world > 1) {
      // sharded marking: each rank marks a contiguous slice, then the exchange
      // callback all-gathers the marks (the slice needs the leaf count on the host)
      int64_t n_leaves = 0;
      OW_TRY(ow_forest_leaves(ctx, f, level, (int32_t*)pl, &n_leaves, s));
      OW_CUDA(cudaMemcpyAsync(dn, &ctx->h_pinned[0], 8, cudaMemcpyHostToDevice, s));  // h_pinned[0] = n_leaves
      const int64_t per = (n_leaves + p->world - 1) / p->world;
      const int64_t lo = per * p->rank < n_leaves ? per * p->rank : n_leaves;
      const int64_t hi = per * (p->rank + 1) < n_leaves ? per * (p->rank + 1) : n_leaves;
      OW_TRY(ow_mark_launch(ctx, f, (const int32_t*)pl + lo, hi - lo, d_coords, n_faces, geom_key,
                            p->binned ? grid : nullptr, p->binned ? d_bin_ids : nullptr,
                            p->binned ? d_bin_counts : nullptr, p->binned ? d_bin_offsets : nullptr,
                            p->binned ? E : 0, p->d_spec, p->reach, dst, s, nullptr, !fresh_bins, nullptr, nullptr,
                            level));
      if (!p->exchange) {
        ow_set_error("refine_near_wall: world > 1 needs an exchange callback");
        return OW_ERR_INVALID;
      }
      int64_t st[3];
      OW_TRY(ow_readback(ctx, (const int64_t*)dst, 3, st, s));
      if (p->exchange(p->exchange_user, level, (const int32_t*)pl, n_leaves, lo, hi, st) != 0) {
        ow_set_error("refine_near_wall: mark exchange failed at level %d", level);
        return OW_ERR_INTERNAL;
      }
      for (int k = 0; k < 3; ++k) ctx->h_pinned[k] = st[k];
      OW_CUDA(cudaMemcpyAsync(dst, ctx->h_pinned, 24, cudaMemcpyHostToDevice, s));
      OW_CUDA(cudaStreamSynchronize(s));
    } else {
      // leaf count stays on the device: marking is launched for n_host blocks
      // (an upper bound) and every warp checks the exact count (the leaves of
      // level >= 1 were written by the previous level's split)
      if (level == 0 || !dev) OW_TRY(ow_forest_leaves_dev(ctx, f, level, (int32_t*)pl, dn, s, d_nb));
      OW_TRY(ow_mark_launch(ctx, f, (const int32_t*)pl, n_host, d_coords, n_faces, geom_key,
                            p->binned ? grid : nullptr, p->binned ? d_bin_ids : nullptr,
                            p->binned ? d_bin_counts : nullptr, p->binned ? d_bin_offsets : nullptr,
                            p->binned ? E : 0, p->d_spec, p->reach, dst, s, dn, !fresh_bins, nullptr,
                            devpass ? ctx->d_small + 5 : nullptr, level));
    }
    // ---- propagation (binned only): 1 + floor(d / min block length)
    OW_TRY(record(se, level, 2, s, ctx->no_stage_events));
    int rounds = 0;
    if (p->binned) {
      double bl = INFINITY;
      for (int a = 0; a < f->dim; ++a) {
        const double b = f->dext[a] / (double)((int64_t)f->root[a] << level);
        bl = b < bl ? b : bl;
      }
      rounds = 1 + (int)floor(p->d_spec64 / bl);
      // (the device-resident loop starts from a fresh root grid: round tags)
      // (its last promote is deferred into the refine's init kernel)
      OW_TRY(ow_propagate_dev(ctx, f, (const int32_t*)pl, dn, n_host, rounds, s, dev, dev));
    }
    // ---- refinement on the device; one readback of its state per level
    OW_TRY(record(se, level, 3, s, ctx->no_stage_events));
    // splits that would not fit the current capacity are detected on the device
    // and finished below on the host path, which grows the forest
    // a cascade of splits descends at least one level per sweep
    const int iters = refine_sweeps(level);
    // device-resident loop: the split of this level's MARKED leaves writes the
    // next level's leaf list (its children, a contiguous id range) and count
    int64_t* next_count = !dev ? nullptr : (level + 1 < passes ? (int64_t*)drv + 72 * (level + 1) : d_sum + SUM_W * passes);
    OW_TRY(ow_refine_dev(ctx, f, level, iters, rs, s, d_nb, dev ? (int32_t*)pl : nullptr, next_count,
                         dev && p->binned && rounds > 0 ? (const int32_t*)pl : nullptr, dn));
    OW_TRY(record(se, level, 4, s, ctx->no_stage_events));
    if (dev) {
      out->n_passes = level + 1;
      continue;
    }
    int64_t h[64];
    OW_TRY(ow_readback(ctx, rs, 64, h, s));
    if (h[0]) {
      ow_set_error("level %d still carries intermediate marks; finish propagation first", level);
      return OW_ERR_INVALID;
    }
    if (h[2] > 0 && level >= f->max_level) {
      ow_set_error("refinement beyond max level %d", f->max_level);
      return OW_ERR_INVALID;
    }
    int64_t n_split = h[3], n_marked = h[2];
    const int64_t n_final = h[8 + iters + 1], last_cnt = refine_sweeps_exact(level) ? 0 : h[36 + iters];
    if (h[1] && h[5]) {
      // the MARKED list itself did not fit: refine synchronously (grows the forest)
      OW_TRY(ow_refine_marked_counted(ctx, f, level, &n_split, &n_marked, s));
    } else {
      f->n_blocks = n_final;
      if (h[1] || last_cnt > 0)  // capacity overflow or a cascade deeper than the device sweeps
        OW_TRY(ow_rebalance_host(ctx, f, h[4], &n_split, s));
    }
    out->marked_refined[level] = n_marked;
    out->n_split[level] = n_split;
    out->n_passes = level + 1;
  }
  if (dev && passes > 0) {
    // (the leaves of the deepest level, the lattice level whenever the last
    // pass split, were written by that pass's split into SLOT_DRV_LEAVES; a
    // device-sized pass forms the summary in its own last kernel)
    if (!devpass) {
      ow_launch(k_drv_summary, 1, 32, 0, s, (const int64_t*)drv, (const unsigned long long*)stats, passes, d_sum);
      OW_LAUNCHED(ctx);
    }
  }
  return OW_OK;
  };  // device_part
  if (dev) {
    // replay / capture / run of the device-resident loop (graph eligible only
    // without host-side events, profiling or a multi-GPU exchange)
    const bool graph_ok = p->binned && p->reuse_bins && ctx->no_stage_events && !comm &&
                          !(ctx->prof && ctx->prof->enabled);
    GraphKey key;
    make_loop_key(&key, ctx, f, d_coords, n_faces, grid, p, d_bin_ids, d_bin_counts, d_bin_offsets, E, stats, drv);
    const int gs = ow_loop_graph(ctx, graph_ok, &key, &s, device_part);
    OW_TRY(gs < 0 ? OW_OK : gs);
    if (gs < 0) {  // replayed: the host-side bookkeeping of the loop
      out->n_passes = passes;
      if (p->binned) {
        out->bin_entries = E;
        out->bins_built = 1;
      }
    }
  } else {
    OW_TRY(device_part());
  }
  if (devpass) {
    // (the caller reads the summary with its other words after the lattice work)
  } else if (dev && passes > 0) {
    int64_t h[SUM_W * OW_MAX_PASSES + 1];
    OW_TRY(ow_readback(ctx, d_sum, SUM_W * passes + 1, h, s));
    OW_TRY(drv_apply(ctx, f, h, passes, out));
  } else if (passes > 0) {
    int64_t h[MARK_STATS * OW_MAX_PASSES];
    OW_TRY(ow_readback(ctx, (const int64_t*)stats, MARK_STATS * passes, h, s));
    for (int level = 0; level < out->n_passes; ++level) {
      out->marked_detected[level] = h[MARK_STATS * level];
      out->tests[level] = h[MARK_STATS * level + 1];
      out->evaluated[level] = h[MARK_STATS * level + 2];
      out->sphere_tests[level] = h[MARK_STATS * level + 3];
      out->box_culls[level] = h[MARK_STATS * level + 4];
    }
  }
  if (!ctx->defer_stage_times) return ow_stage_times(ctx, out);
  return OW_OK;
}
}  // namespace

extern "C" int ow_refine_near_wall(ow_ctx* ctx, ow_forest* f, const float* d_coords, int64_t n_faces, int64_t geom_key,
                                   const ow_grid* grid, const ow_nearwall_params* p, int32_t* d_bin_ids,
                                   int64_t bin_ids_capacity, int32_t* d_bin_counts, int32_t* d_bin_offsets,
                                   ow_nearwall_result* out, void* stream) {
  return refine_driver(ctx, f, d_coords, n_faces, geom_key, grid, p, d_bin_ids, bin_ids_capacity, d_bin_counts,
                       d_bin_offsets, out, (cudaStream_t)stream, false);
}

// stage times of the last driver pass from its CUDA events (all recorded
// events precede the driver's final readback, so they are complete)
int ow_stage_times(ow_ctx* ctx, ow_nearwall_result* out) {
  StageEvents* se = (StageEvents*)ctx->stage_events;
  if (!se) return OW_OK;
  for (int level = 0; level < out->n_passes; ++level)
    for (int k = 0; k < 4; ++k) {
      float ms = 0.0f;
      if (se->used[level][k] && se->used[level][k + 1])
        OW_CUDA(cudaEventElapsedTime(&ms, se->ev[level][k], se->ev[level][k + 1]));
      out->stage_ms[level][k] = ms;
    }
  return OW_OK;
}

// ---------------------------------------------------------------------------
// One geometry-to-grid pass in one host call: import (binary STL records ->
// SoA) -> face validation / bounding box -> root grid -> refine_near_wall ->
// lattice links on the finest level.  Output buffers whose size is only known
// on the device (finest leaves, flags, boundary cells, q) are requested from
// the caller through `alloc`, so the caller's allocator (PyTorch) owns them.
// ---------------------------------------------------------------------------
namespace {
int out_buffer(const ow_g2g_params* p, int what, int64_t bytes, void** out) {
  if (p->out_buf[what] && p->out_cap[what] >= bytes) {
    *out = p->out_buf[what];
    return 0;
  }
  return p->alloc(p->alloc_user, what, bytes, out);
}

__global__ void k_widen(const int32_t* __restrict__ in, int64_t n, int64_t* out) {
  ow_pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}
}  // namespace

struct FacesState {
  ow_g2g_result* out;
  const ow_forest* f;
  ow_nearwall_params* nw;
  int64_t n_faces;
};

int ow_faces_settle(ow_ctx* ctx, const int64_t* h6, cudaStream_t s) {
  if (!ctx->faces_pending) return OW_OK;
  int64_t h[6];
  if (h6) {
    memcpy(h, h6, sizeof(h));
  } else {
    OW_TRY(ow_readback(ctx, ctx->faces_pending, 6, h, s));
  }
  ctx->faces_pending = nullptr;
  FacesState* fs = (FacesState*)ctx->faces_state;
  ow_g2g_result* out = fs->out;
  const ow_forest* f = fs->f;
  const int D = f->dim;
  ow_face_summary_from(h, fs->n_faces, &out->faces);
  if (out->faces.first_nonfinite >= 0) {
    ow_set_error("geometry has non-finite coordinates");
    return OW_ERR_INVALID;
  }
  if (out->faces.first_degenerate >= 0) {
    ow_set_error(D == 2 ? "degenerate edge (identical endpoints) at face %lld"
                        : "degenerate triangle (zero area) at face %lld",
                 (long long)out->faces.first_degenerate);
    return OW_ERR_INVALID;
  }
  double scale = 0.0;  // nearwall.py:31-35: max |coordinate| of domain and geometry
  for (int a = 0; a < D; ++a) {
    const double lo = f->dmin[a], hi = f->dmin[a] + f->dext[a], tol = 1e-6 * f->dext[a];
    if ((double)out->faces.bbox_min[a] < lo - tol || (double)out->faces.bbox_max[a] > hi + tol) {
      out->outside_domain = 1;
      ow_set_error("geometry outside the forest domain");
      return OW_ERR_INVALID;
    }
    scale = fmax(scale, fmax(fabs(lo), fabs(hi)));
  }
  scale = fmax(scale, (double)out->faces.abs_max);
  ow_nearwall_params* nw = fs->nw;
  if (!(nw->reach > 0.0)) nw->reach = nw->d_spec64 + 1e-3 * fmax(1.0, fmax(scale, nw->d_spec64));  // nearwall.py:38-40
  return OW_OK;
}

namespace {
int g2g_sync(ow_ctx* ctx, const uint8_t* d_records, float* d_coords, int64_t n_faces, int64_t geom_key, ow_forest* f,
             const ow_grid* grid, const ow_g2g_params* p, int32_t* d_bin_ids, int64_t bin_ids_capacity,
             int32_t* d_bin_counts, int32_t* d_bin_offsets, ow_g2g_result* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  memset(out, 0, sizeof(*out));
  out->faces.first_degenerate = out->faces.first_nonfinite = -1;
  const int D = f->dim;
  if (n_faces <= 0) {
    ow_set_error("cannot refine around empty geometry");
    return OW_ERR_INVALID;
  }
  // deferred host copies of this caller's previous pass still read its
  // outputs: the device waits for them before anything is rewritten
  if (p->copy_done) OW_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)p->copy_done, 0));
  // the face check's summary is read with the first bin-count readback (one
  // host round trip less) and validated there, before anything depends on it
  // (with STL records: fused into the record -> SoA pass)
  if (d_records && D == 3) OW_TRY(ow_stl_to_soa_checked(ctx, d_records, n_faces, d_coords, ctx->d_small + 56, s));
  else OW_TRY(ow_face_check_launch(ctx, D, d_coords, n_faces, ctx->d_small + 56, s));
  OW_TRY(ow_forest_init_root(ctx, f, stream));
  ow_nearwall_params nw = p->nw;
  FacesState fs_state{out, f, &nw, n_faces};
  ctx->faces_state = &fs_state;
  ctx->faces_pending = ctx->d_small + 56;
  ctx->defer_stage_times = true;  // read the stage events after the lattice work is queued
  ctx->no_stage_events = p->no_stage_times != 0;
  int st = refine_driver(ctx, f, d_coords, n_faces, geom_key, grid, &nw, d_bin_ids, bin_ids_capacity, d_bin_counts,
                         d_bin_offsets, &out->nw, s, true);
  if (st == OW_OK && ctx->faces_pending) st = ow_faces_settle(ctx, nullptr, s);  // (no pass read it)
  ctx->faces_pending = nullptr;
  ctx->faces_state = nullptr;
  if (out->faces.first_nonfinite >= 0 || out->faces.first_degenerate >= 0 || out->outside_domain) {
    ctx->defer_stage_times = false;
    ctx->no_stage_events = false;
    return OW_ERR_INVALID;  // (the message was set by ow_faces_settle)
  }
  if (st == DRV_RETRY) {  // the forest outgrew its capacity (or a deep cascade): per-level host path
    out->reran = 1;
    OW_TRY(ow_forest_init_root(ctx, f, stream));
    st = refine_driver(ctx, f, d_coords, n_faces, geom_key, grid, &nw, d_bin_ids, bin_ids_capacity, d_bin_counts,
                       d_bin_offsets, &out->nw, s, false);
  }
  ctx->defer_stage_times = false;
  ctx->no_stage_events = false;
  OW_TRY(st);
  int finest = 0;
  for (int l = 0; l < out->nw.n_passes; ++l)
    if (out->nw.n_split[l] > 0) finest = l + 1;
  out->finest_level = finest;
  // the forest is final: stream its arrays to the host on the side stream
  // while the lattice work runs on `s`
  const int64_t nbk = f->n_blocks;
  bool side = false;
  if (p->host_level && p->host_block_cap >= nbk) {
    if (!ctx->copy_stream) {
      OW_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      OW_CUDA(cudaEventCreateWithFlags(&ctx->copy_ev[0], cudaEventDisableTiming));
      OW_CUDA(cudaEventCreateWithFlags(&ctx->copy_ev[1], cudaEventDisableTiming));
    }
    cudaStream_t cs = ctx->copy_stream;
    OW_CUDA(cudaEventRecord(ctx->copy_ev[0], s));
    OW_CUDA(cudaStreamWaitEvent(cs, ctx->copy_ev[0], 0));
    OW_CUDA(cudaMemcpyAsync(p->host_level, f->d_level, 2 * (size_t)nbk, cudaMemcpyDeviceToHost, cs));
    for (int a = 0; a < D; ++a)
      OW_CUDA(cudaMemcpyAsync(p->host_coord[a], f->d_coord[a], 4 * (size_t)nbk, cudaMemcpyDeviceToHost, cs));
    OW_CUDA(cudaMemcpyAsync(p->host_parent, f->d_parent, 4 * (size_t)nbk, cudaMemcpyDeviceToHost, cs));
    OW_CUDA(cudaMemcpyAsync(p->host_first_child, f->d_first_child, 4 * (size_t)nbk, cudaMemcpyDeviceToHost, cs));
    OW_CUDA(cudaMemcpyAsync(p->host_marks, f->d_marks, (size_t)nbk, cudaMemcpyDeviceToHost, cs));
    OW_CUDA(cudaEventRecord(ctx->copy_ev[1], cs));
    out->host_copied |= 1;
    side = true;
  }
  // from here on every return path (errors included) joins the side stream
  // into `s` — the caller may reuse the forest storage on `s` as soon as the
  // call returns, and the copies still read it — or, with deferred copies,
  // records copy_done after them (the caller's next pass waits for it)
  struct JoinCopies {
    ow_ctx* ctx;
    cudaStream_t s;
    cudaEvent_t done;
    bool on;
    ~JoinCopies() {
      if (!on) return;
      if (done) cudaEventRecord(done, ctx->copy_stream);
      else cudaStreamWaitEvent(s, ctx->copy_ev[1], 0);
    }
  } join{ctx, s, (cudaEvent_t)p->copy_done, side};
  if (p->lattice_q < 2 || !p->alloc) return ow_stage_times(ctx, &out->nw);
  void* pl;
  OW_TRY(ow_slot(ctx, SLOT_DRV_LEAVES, 4 * (size_t)(f->n_blocks + 1), s, &pl));
  int64_t nl = ctx->drv_spec_nl;  // compacted by the device-resident loop
  if (nl < 0 || finest != out->nw.n_passes) OW_TRY(ow_forest_leaves(ctx, f, finest, (int32_t*)pl, &nl, stream));
  out->n_finest_leaves = nl;
  const int C = D == 3 ? 64 : 16;
  void *leaves64, *flags;
  if (out_buffer(p, OW_OUT_LEAVES, 8 * nl, &leaves64) || out_buffer(p, OW_OUT_FLAGS, 4 * nl * C, &flags)) {
    ow_set_error("geometry_to_grid: output allocation failed");
    return OW_ERR_INTERNAL;
  }
  if (nl > 0) {
    ow_launch(k_widen, ow_blocks(nl, 256), 256, 0, s, (const int32_t*)pl, nl, (int64_t*)leaves64);
    OW_LAUNCHED(ctx);
    OW_CHECK_LAUNCH();
  }
  int64_t nb = 0;
  ctx->lat_mean_extent = out->faces.mean_extent;  // shapes the face pass
  // multi-GPU: each rank sweeps an equal slice of the finest leaves; flag
  // words and q rows are all-gathered over peer memory inside the lattice calls
  const bool shard = p->nw.world > 1 && p->nw.comm;
  ctx->lat_comm = shard ? p->nw.comm : nullptr;
  const int64_t pos_lo = shard ? nl * p->nw.rank / p->nw.world : 0;
  const int64_t pos_hi = shard ? nl * (p->nw.rank + 1) / p->nw.world : nl;
  const int lst = ow_lattice_links_count_range(ctx, f, finest, (const int32_t*)pl, nl, pos_lo, pos_hi, d_coords,
                                               n_faces, geom_key, grid, p->lattice_dirs, p->lattice_q,
                                               (uint32_t*)flags, &nb, stream);
  ctx->lat_mean_extent = 0.0f;
  if (lst != OW_OK) ctx->lat_comm = nullptr;
  OW_TRY(lst);
  out->n_boundary = nb;
  void *cells, *q;
  if (out_buffer(p, OW_OUT_CELLS, 8 * nb, &cells) || out_buffer(p, OW_OUT_Q, 4 * nb * p->lattice_q, &q)) {
    ow_set_error("geometry_to_grid: output allocation failed");
    return OW_ERR_INTERNAL;
  }
  int64_t n_links = 0;
  OW_TRY(ow_lattice_links_n_links(ctx, &n_links));
  out->n_links = n_links;
  const bool packed = p->host_rows && p->host_q_packed && p->host_row_cap >= nb && p->host_link_cap >= n_links &&
                      nb > 0;
  uint32_t* d_rows = nullptr;
  float* d_qp = nullptr;
  // deferred copies need staging buffers of the caller's own (the next pass
  // of another plan reuses the context's scratch while these copies run)
  const bool deferred = p->copy_done && side && packed && p->dev_rows && p->dev_q_packed &&
                        p->dev_row_cap >= nb && p->dev_link_cap >= n_links;
  if (deferred) {
    d_rows = (uint32_t*)p->dev_rows;
    d_qp = (float*)p->dev_q_packed;
  } else if (packed) {
    void *pr, *pq;
    OW_TRY(ow_slot(ctx, SLOT_LAT_RFLAGS, 8 * (size_t)nb, s, &pr));
    OW_TRY(ow_slot(ctx, SLOT_LAT_QPACK, 4 * (size_t)n_links, s, &pq));
    d_rows = (uint32_t*)pr;
    d_qp = (float*)pq;
  }
  const int est = ow_lattice_links_emit_packed(ctx, (int64_t*)cells, (float*)q, d_rows, d_qp, stream);
  ctx->lat_comm = nullptr;
  OW_TRY(est);
  if (deferred) {  // the packed rows travel on the copy stream, after the forest arrays
    join.on = false;
    OW_CUDA(cudaEventRecord(ctx->copy_ev[0], s));
    OW_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_ev[0], 0));
    OW_CUDA(cudaMemcpyAsync(p->host_rows, d_rows, 8 * (size_t)nb, cudaMemcpyDeviceToHost, ctx->copy_stream));
    OW_CUDA(cudaMemcpyAsync(p->host_q_packed, d_qp, 4 * (size_t)n_links, cudaMemcpyDeviceToHost, ctx->copy_stream));
    OW_CUDA(cudaEventRecord((cudaEvent_t)p->copy_done, ctx->copy_stream));
    out->host_copied |= 4 | 8;
  } else if (packed) {  // (8 + 4 popc) bytes per row instead of 8 + 4 Q: the host tail is the transfer
    OW_CUDA(cudaMemcpyAsync(p->host_rows, d_rows, 8 * (size_t)nb, cudaMemcpyDeviceToHost, s));
    OW_CUDA(cudaMemcpyAsync(p->host_q_packed, d_qp, 4 * (size_t)n_links, cudaMemcpyDeviceToHost, s));
    out->host_copied |= 4;
  } else if (p->host_cells && p->host_q && p->host_row_cap >= nb && nb > 0) {
    OW_CUDA(cudaMemcpyAsync(p->host_cells, cells, 8 * (size_t)nb, cudaMemcpyDeviceToHost, s));
    OW_CUDA(cudaMemcpyAsync(p->host_q, q, 4 * (size_t)nb * p->lattice_q, cudaMemcpyDeviceToHost, s));
    out->host_copied |= 2;
  }
  if (side && !deferred) {  // results complete on `s`
    join.on = false;
    OW_CUDA(cudaStreamWaitEvent(s, ctx->copy_ev[1], 0));
    if (p->copy_done) OW_CUDA(cudaEventRecord((cudaEvent_t)p->copy_done, s));
  }
  OW_TRY(ow_lattice_stats(ctx, out->lattice_stats, stream));
  return ow_stage_times(ctx, &out->nw);  // host work overlapping the emit kernels
}
}  // namespace (g2g_sync)

// ---------------------------------------------------------------------------
// Device-sized pass: the whole geometry-to-grid pass is enqueued without a
// host round trip — bins counted and emitted with their entry count on the
// device, the level loop device-resident (a CUDA graph when replayable), the
// lattice stage sized by the deepest level's leaf count on the device, emit
// kernels striding over the candidate-block count — and ONE readback at the
// end carries every count the host needs.  Launch sizes come from capacities
// (the forest capacity, the caller's output buffers, the bin-entry and
// lattice-row estimates of earlier passes); every kernel bounds its writes by
// them.  The host then checks, in the reference's error order, the face
// summary, the bin counts, the driver summary and the lattice counts; a pass
// whose capacity or assumption (no slow bin faces, the near-wall reach
// predicted from the domain, every level split) did not hold is re-run on the
// synchronous path (g2g_sync), which also learns the larger capacities.
// ---------------------------------------------------------------------------
namespace {
constexpr int G2G_RETRY = 1001;
constexpr int G2G_WORDS = 34;  // [0, 8) bins, [8, 28) lattice (d_small 33..52), [28, 34) face summary

// every word the host needs, written straight into mapped pinned host memory
// (no copy-engine transfer after the last kernel): the driver summary, then
// the bin, lattice and face words
__global__ void k_g2g_summary(const int64_t* __restrict__ small, const int64_t* __restrict__ drv,
                              const unsigned long long* __restrict__ stats, int passes, volatile int64_t* dst) {
  ow_pdl_wait();
  for (int p = threadIdx.x; p < passes; p += blockDim.x) drv_summary_pass(drv, stats, p, dst + SUM_W * p);
  const int n_sum = SUM_W * passes + 1;
  if (threadIdx.x == 0) dst[n_sum - 1] = drv[72 * passes + 8 + SUM_W * passes];  // the deepest level's leaves
  volatile int64_t* t = dst + n_sum;
  const int k = threadIdx.x;
  if (k < 8) t[k] = small[k];
  if (k < 20) t[8 + k] = small[33 + k];
  if (k < 6) t[28 + k] = small[56 + k];
}

// near-wall reach (nearwall.py:31-40) from the domain alone: equal to the
// reference's value whenever no coordinate of the geometry exceeds the
// domain's largest |bound| (checked against the face summary afterwards)
double predicted_reach(const ow_forest* f, const ow_nearwall_params* nw) {
  if (nw->reach > 0.0) return nw->reach;
  double scale = 0.0;
  for (int a = 0; a < f->dim; ++a) scale = fmax(scale, fmax(fabs(f->dmin[a]), fabs(f->dmin[a] + f->dext[a])));
  return nw->d_spec64 + 1e-3 * fmax(1.0, fmax(scale, nw->d_spec64));
}

// One device-sized pass in flight: what its finish step needs besides the
// caller's arguments (the capacities the pass was launched with, its summary
// area and the event after its last kernel)
struct G2GTicket {
  int used;
  cudaEvent_t ev;       // recorded after k_g2g_summary
  int passes;
  int64_t n_faces, e_cap, nl_cap, row_cap, link_cap, lat_row_cap, lat_unit_cap, lat_ihit_cap;
  bool packed, host_forest, deferred;
  uint32_t* d_rows;
  float* d_qp;
  double reach_pred;
  int64_t* area;        // pinned summary words (host view)
};
constexpr int G2G_TICKETS = 8;
constexpr int G2G_AREA = 512;  // int64 words per summary area

// enqueue the whole pass; no host round trip
int g2g_submit(ow_ctx* ctx, const uint8_t* d_records, float* d_coords, int64_t n_faces, int64_t geom_key,
               ow_forest* f, const ow_grid* grid, const ow_g2g_params* p, int32_t* d_bin_ids,
               int64_t bin_ids_capacity, int32_t* d_bin_counts, int32_t* d_bin_offsets, ow_g2g_result* out,
               cudaStream_t s, G2GTicket* t) {
  const int D = f->dim, C = D == 3 ? 64 : 16, Q = p->lattice_q;
  const int passes = p->nw.n_levels - 1;
  static_assert(SUM_W * OW_MAX_PASSES + 1 + G2G_WORDS <= G2G_AREA, "summary area");
  // capacities of this pass
  const int64_t e_cap = ctx->dev_e_cap < bin_ids_capacity ? ctx->dev_e_cap : bin_ids_capacity;
  int64_t nl_cap = f->capacity;
  nl_cap = p->out_cap[OW_OUT_FLAGS] / (4 * C) < nl_cap ? p->out_cap[OW_OUT_FLAGS] / (4 * C) : nl_cap;
  nl_cap = p->out_cap[OW_OUT_LEAVES] / 8 < nl_cap ? p->out_cap[OW_OUT_LEAVES] / 8 : nl_cap;
  int64_t row_cap = p->out_cap[OW_OUT_CELLS] / 8;
  row_cap = p->out_cap[OW_OUT_Q] / (4 * (int64_t)Q) < row_cap ? p->out_cap[OW_OUT_Q] / (4 * (int64_t)Q) : row_cap;
  const bool packed = p->host_rows && p->host_q_packed && p->host_row_cap > 0 && p->host_link_cap > 0;
  const bool host_forest = p->host_level && p->host_block_cap > 0;
  const bool deferred = p->copy_done && packed && host_forest && p->dev_rows && p->dev_q_packed &&
                        p->dev_row_cap > 0 && p->dev_link_cap > 0;
  int64_t link_cap = INT64_MAX;
  uint32_t* d_rows = nullptr;
  float* d_qp = nullptr;
  if (packed) {
    row_cap = p->host_row_cap < row_cap ? p->host_row_cap : row_cap;
    link_cap = p->host_link_cap;
    if (deferred) {
      row_cap = p->dev_row_cap < row_cap ? p->dev_row_cap : row_cap;
      link_cap = p->dev_link_cap < link_cap ? p->dev_link_cap : link_cap;
      d_rows = (uint32_t*)p->dev_rows;
      d_qp = (float*)p->dev_q_packed;
    } else {
      void *pr, *pq;
      OW_TRY(ow_slot(ctx, SLOT_LAT_RFLAGS, 8 * (size_t)row_cap, s, &pr));
      OW_TRY(ow_slot(ctx, SLOT_LAT_QPACK, 4 * (size_t)link_cap, s, &pq));
      d_rows = (uint32_t*)pr;
      d_qp = (float*)pq;
    }
  }
  if (e_cap < 1 || nl_cap < 1 || row_cap < 1) return G2G_RETRY;
  if (!t->ev) OW_CUDA(cudaEventCreateWithFlags(&t->ev, cudaEventDisableTiming));
  t->passes = passes;
  t->n_faces = n_faces;
  t->e_cap = e_cap;
  t->nl_cap = nl_cap;
  t->row_cap = row_cap;
  t->link_cap = link_cap;
  t->packed = packed;
  t->host_forest = host_forest;
  t->deferred = deferred;
  t->d_rows = d_rows;
  t->d_qp = d_qp;
  // ---- the pass, enqueued without a host round trip
  if (p->copy_done) OW_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)p->copy_done, 0));
  if (d_records && D == 3) {  // root grid + face summary words in one launch, then the fused import
    OW_TRY(init_root(ctx, f, s, ctx->d_small + 56));
    OW_TRY(ow_stl_to_soa_checked(ctx, d_records, n_faces, d_coords, ctx->d_small + 56, s, false));
  } else {
    OW_TRY(ow_face_check_launch(ctx, D, d_coords, n_faces, ctx->d_small + 56, s));
    OW_TRY(ow_forest_init_root(ctx, f, s));
  }
  ow_nearwall_params nw = p->nw;
  nw.reach = predicted_reach(f, &p->nw);
  t->reach_pred = nw.reach;
  ctx->faces_pending = nullptr;
  ctx->defer_stage_times = true;
  ctx->no_stage_events = p->no_stage_times != 0;
  ctx->dev_pass = true;
  ctx->dev_e_cap = e_cap;  // (read by refine_driver)
  int st = refine_driver(ctx, f, d_coords, n_faces, geom_key, grid, &nw, d_bin_ids, bin_ids_capacity, d_bin_counts,
                         d_bin_offsets, &out->nw, s, true);
  ctx->dev_pass = false;
  if (st != OW_OK) return st;
  void* drv = ctx->slot_ptr[SLOT_DRV_STATE];
  int64_t* d_sum = (int64_t*)drv + 72 * passes + 8;
  const int64_t* d_nl = d_sum + SUM_W * passes;  // the deepest level's leaf count (refine_driver)
  const int32_t* leaves = (const int32_t*)ctx->slot_ptr[SLOT_DRV_LEAVES];
  int64_t* leaves64 = (int64_t*)p->out_buf[OW_OUT_LEAVES];
  uint32_t* flags = (uint32_t*)p->out_buf[OW_OUT_FLAGS];
  ctx->lat_mean_extent = ctx->dev_mean_extent;
  ctx->lat_comm = nullptr;
  // (k_lat_pos also writes the int64 leaf output)
  st = ow_lattice_dev_count(ctx, f, passes, leaves, d_nl, nl_cap, d_coords, n_faces, p->lattice_dirs, Q, flags, s,
                            leaves64);
  ctx->lat_mean_extent = 0.0f;
  OW_TRY(st);
  // (the caps the finish step checks against: the lattice lists as sized now)
  t->lat_row_cap = ctx->lat_row_cap;
  t->lat_unit_cap = ctx->lat_unit_cap;
  t->lat_ihit_cap = ctx->lat_ihit_cap;
  const int64_t ncb_grid = ctx->dev_ncb > 0 ? ctx->dev_ncb : 4 * OW_SMS;
  OW_TRY(ow_lattice_dev_emit(ctx, (int64_t*)p->out_buf[OW_OUT_CELLS], (float*)p->out_buf[OW_OUT_Q], row_cap, d_rows,
                             d_qp, link_cap, ncb_grid, s));
  // ---- every count the host needs, stored into this pass's pinned area
  ow_launch(k_g2g_summary, 1, 128, 0, s, (const int64_t*)ctx->d_small, (const int64_t*)drv,
            (const unsigned long long*)ctx->slot_ptr[SLOT_DRV_STATS], passes,
            (volatile int64_t*)(ctx->g2g_ring_dev + (t->area - ctx->g2g_ring)));
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  OW_CUDA(cudaEventRecord(t->ev, s));
  return OW_OK;
}

// wait for the pass's summary, check it in the reference's error order, and
// stream the host copies; G2G_RETRY: re-run on the synchronous path
int g2g_finish(ow_ctx* ctx, ow_forest* f, const ow_g2g_params* p, ow_g2g_result* out, cudaStream_t s,
               G2GTicket* t) {
  const int D = f->dim, Q = p->lattice_q, passes = t->passes;
  const int n_sum = SUM_W * passes + 1;
  OW_CUDA(cudaEventSynchronize(t->ev));
  int64_t h[SUM_W * OW_MAX_PASSES + 1], w[G2G_WORDS];
  memcpy(h, t->area, 8 * (size_t)n_sum);
  memcpy(w, t->area + n_sum, sizeof(w));
  // faces first (the reference's import order), then bins, driver, lattice
  ow_nearwall_params nw_true = p->nw;
  FacesState fs_state{out, f, &nw_true, t->n_faces};
  ctx->faces_state = &fs_state;
  ctx->faces_pending = ctx->d_small + 56;
  int st = ow_faces_settle(ctx, w + 28, s);
  ctx->faces_state = nullptr;
  ctx->faces_pending = nullptr;
  if (st != OW_OK) return st;
  if (w[1] >= 0) {
    ow_set_error("face sample outside binning domain (face %lld)", (long long)w[1]);
    return OW_ERR_INVALID;
  }
  if (w[2]) {
    ow_set_error("fill_bins: a face sample escaped its padded bin range (internal)");
    return OW_ERR_INTERNAL;
  }
  const int64_t E = w[5];
  ctx->dev_mean_extent = out->faces.mean_extent;
  if (E > t->e_cap && ctx->dev_e_cap < E + E / 4 + 1024) ctx->dev_e_cap = E + E / 4 + 1024;
  if (w[0] > 0 || E > t->e_cap || E > p->nw.overlap_factor * t->n_faces || nw_true.reach != t->reach_pred)
    return G2G_RETRY;  // slow bin faces, short pair buffers, a capacity error or another reach
  st = drv_apply(ctx, f, h, passes, &out->nw);
  if (st == DRV_RETRY) return G2G_RETRY;
  if (st != OW_OK) return st;
  out->nw.n_passes = passes;
  out->nw.bin_entries = E;
  out->nw.bins_built = 1;
  int finest = 0;
  for (int l = 0; l < passes; ++l)
    if (out->nw.n_split[l] > 0) finest = l + 1;
  const int64_t nl = h[SUM_W * passes];
  if (finest != passes || nl > t->nl_cap) return G2G_RETRY;
  const int64_t* L = w + 8;  // d_small[33 + i]
  const int64_t n_cb = L[0], nb = L[2], n_links = L[18];
  const int64_t n_rows = (int64_t)((uint64_t)L[15] & ((1ull << 28) - 1)), n_units = (int64_t)((uint64_t)L[15] >> 28);
  if (n_rows > t->lat_row_cap || n_units > t->lat_unit_cap || L[16] > t->lat_ihit_cap) {
    // the sync path grows the row / hit lists (and re-runs the sweep)
    return G2G_RETRY;
  }
  if (nb > t->row_cap || n_links > t->link_cap) return G2G_RETRY;
  // ---- results
  out->finest_level = finest;
  out->n_finest_leaves = nl;
  out->n_boundary = nb;
  out->n_links = n_links;
  ctx->lat_ncb = n_cb;
  ctx->lat_rows = n_rows + (int64_t)((uint64_t)L[17] & ((1ull << 28) - 1));
  ctx->lat_units = n_units + (int64_t)((uint64_t)L[17] >> 28);
  ctx->lat_boundary = nb;
  ctx->lat_links = n_links;
  ctx->dev_ncb = n_cb;
  out->lattice_stats[0] = n_cb;
  out->lattice_stats[1] = ctx->lat_rows;
  out->lattice_stats[2] = ctx->lat_units;
  // host copies: on the copy stream after this pass's last kernel for a
  // deferred caller (later passes may already be queued on `s`), else on `s`
  const int64_t nbk = f->n_blocks;
  const bool fc = t->host_forest && p->host_block_cap >= nbk;
  const bool rows_fit = t->packed && nb > 0;
  if (fc || rows_fit || (!t->packed && p->host_cells && p->host_q && p->host_row_cap >= nb && nb > 0)) {
    cudaStream_t cs = s;
    if (t->deferred) {
      if (!ctx->copy_stream) {
        OW_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        OW_CUDA(cudaEventCreateWithFlags(&ctx->copy_ev[0], cudaEventDisableTiming));
        OW_CUDA(cudaEventCreateWithFlags(&ctx->copy_ev[1], cudaEventDisableTiming));
      }
      cs = ctx->copy_stream;
      OW_CUDA(cudaStreamWaitEvent(cs, t->ev, 0));
    }
    if (fc) {
      OW_CUDA(cudaMemcpyAsync(p->host_level, f->d_level, 2 * (size_t)nbk, cudaMemcpyDeviceToHost, cs));
      for (int a = 0; a < D; ++a)
        OW_CUDA(cudaMemcpyAsync(p->host_coord[a], f->d_coord[a], 4 * (size_t)nbk, cudaMemcpyDeviceToHost, cs));
      OW_CUDA(cudaMemcpyAsync(p->host_parent, f->d_parent, 4 * (size_t)nbk, cudaMemcpyDeviceToHost, cs));
      OW_CUDA(cudaMemcpyAsync(p->host_first_child, f->d_first_child, 4 * (size_t)nbk, cudaMemcpyDeviceToHost, cs));
      OW_CUDA(cudaMemcpyAsync(p->host_marks, f->d_marks, (size_t)nbk, cudaMemcpyDeviceToHost, cs));
      out->host_copied |= 1;
    }
    if (rows_fit) {
      OW_CUDA(cudaMemcpyAsync(p->host_rows, t->d_rows, 8 * (size_t)nb, cudaMemcpyDeviceToHost, cs));
      OW_CUDA(cudaMemcpyAsync(p->host_q_packed, t->d_qp, 4 * (size_t)n_links, cudaMemcpyDeviceToHost, cs));
      out->host_copied |= t->deferred ? 4 | 8 : 4;
    } else if (!t->packed && p->host_cells && p->host_q && p->host_row_cap >= nb && nb > 0) {
      OW_CUDA(cudaMemcpyAsync(p->host_cells, p->out_buf[OW_OUT_CELLS], 8 * (size_t)nb, cudaMemcpyDeviceToHost, cs));
      OW_CUDA(cudaMemcpyAsync(p->host_q, p->out_buf[OW_OUT_Q], 4 * (size_t)nb * Q, cudaMemcpyDeviceToHost, cs));
      out->host_copied |= 2;
    }
    if (t->deferred) OW_CUDA(cudaEventRecord((cudaEvent_t)p->copy_done, cs));
  }
  if (p->copy_done && !t->deferred) OW_CUDA(cudaEventRecord((cudaEvent_t)p->copy_done, s));
  return ow_stage_times(ctx, &out->nw);
}

int ticket_get(ow_ctx* ctx, G2GTicket** out) {
  if (!ctx->g2g_tickets) {
    ctx->g2g_tickets = calloc(G2G_TICKETS, sizeof(G2GTicket));
    if (!ctx->g2g_tickets) {
      ow_set_error("geometry_to_grid: out of host memory");
      return OW_ERR_INTERNAL;
    }
    OW_CUDA(cudaHostAlloc((void**)&ctx->g2g_ring, 8 * (size_t)G2G_AREA * G2G_TICKETS, cudaHostAllocMapped));
    OW_CUDA(cudaHostGetDevicePointer((void**)&ctx->g2g_ring_dev, ctx->g2g_ring, 0));
  }
  G2GTicket* T = (G2GTicket*)ctx->g2g_tickets;
  for (int i = 0; i < G2G_TICKETS; ++i)
    if (!T[i].used) {
      T[i].used = 1;
      T[i].area = ctx->g2g_ring + (size_t)G2G_AREA * i;
      *out = &T[i];
      return OW_OK;
    }
  ow_set_error("geometry_to_grid: more than %d passes in flight on one context", G2G_TICKETS);
  return OW_ERR_INVALID;
}

void g2g_reset_state(ow_ctx* ctx) {
  ctx->dev_pass = false;
  ctx->faces_pending = nullptr;
  ctx->faces_state = nullptr;
  ctx->defer_stage_times = false;
  ctx->no_stage_events = false;
}

bool g2g_device_eligible(const ow_ctx* ctx, const ow_forest* f, const ow_g2g_params* p) {
  static const bool env_off = [] {
    const char* e = getenv("OW_DEVICE_PASS");
    return e && e[0] == '0';
  }();
  if (env_off || ctx->dev_disabled || ctx->dev_e_cap <= 0) return false;
  if (p->nw.world > 1 || !p->nw.binned || !p->nw.reuse_bins || p->nw.n_levels < 2) return false;
  if (p->lattice_q < 2 || !p->alloc) return false;
  for (int k = 0; k < 4; ++k)
    if (!p->out_buf[k] || p->out_cap[k] <= 0) return false;
  if (ctx->prof && ctx->prof->enabled) return false;  // (profiled passes keep per-stage brackets)
  return f->capacity > 0;
}
}  // namespace

// (ow_ctx_destroy) the in-flight table and the pinned summary areas
void ow_g2g_release(ow_ctx* ctx) {
  if (ctx->g2g_tickets) {
    G2GTicket* T = (G2GTicket*)ctx->g2g_tickets;
    for (int i = 0; i < G2G_TICKETS; ++i)
      if (T[i].ev) cudaEventDestroy(T[i].ev);
    free(ctx->g2g_tickets);
    ctx->g2g_tickets = nullptr;
  }
  if (ctx->g2g_ring) cudaFreeHost(ctx->g2g_ring);
  ctx->g2g_ring = ctx->g2g_ring_dev = nullptr;
}

extern "C" int ow_set_device_pass(ow_ctx* ctx, int32_t enable) {
  ctx->dev_disabled = enable ? 0 : 1;
  return OW_OK;
}

extern "C" int ow_device_pass_stats(ow_ctx* ctx, int64_t* out2) {
  out2[0] = ctx->dev_passes;
  out2[1] = ctx->dev_fallbacks;
  return OW_OK;
}

namespace {
// the synchronous pass, after a device-sized attempt (fell_back) or instead of one
int g2g_sync_learn(ow_ctx* ctx, const uint8_t* d_records, float* d_coords, int64_t n_faces, int64_t geom_key,
                   ow_forest* f, const ow_grid* grid, const ow_g2g_params* p, int32_t* d_bin_ids,
                   int64_t bin_ids_capacity, int32_t* d_bin_counts, int32_t* d_bin_offsets, ow_g2g_result* out,
                   void* stream, bool fell_back) {
  if (fell_back) {
    ctx->dev_fallbacks++;
    d_records = nullptr;  // (records already converted: the synchronous pass starts from the coordinates)
  }
  const int st = g2g_sync(ctx, d_records, d_coords, n_faces, geom_key, f, grid, p, d_bin_ids, bin_ids_capacity,
                          d_bin_counts, d_bin_offsets, out, stream);
  if (st == OW_OK) {  // capacities for the next device-sized pass
    const int64_t E = out->nw.bin_entries;
    const int64_t want = E + E / 4 + 1024;
    if (ctx->dev_e_cap < want) ctx->dev_e_cap = want;
    ctx->dev_ncb = out->lattice_stats[0];
    ctx->dev_mean_extent = out->faces.mean_extent;
    out->device_sized = fell_back ? 2 : 0;
  }
  return st;
}

void g2g_out_init(ow_g2g_result* out) {
  memset(out, 0, sizeof(*out));
  out->faces.first_degenerate = out->faces.first_nonfinite = -1;
}
}  // namespace

// Submit a pass without waiting for it (device-sized when eligible and no
// stage events are requested): *ticket > 0 identifies the pass in flight and
// ow_geometry_to_grid_finish completes it; *ticket = 0: the pass ran
// synchronously and `out` is final.  Between submit and finish the caller
// keeps every argument alive and unchanged and may submit passes of other
// plans (other forests, parameters and outputs) on the same stream.
extern "C" int ow_geometry_to_grid_submit(ow_ctx* ctx, const uint8_t* d_records, float* d_coords, int64_t n_faces,
                                          int64_t geom_key, ow_forest* f, const ow_grid* grid, const ow_g2g_params* p,
                                          int32_t* d_bin_ids, int64_t bin_ids_capacity, int32_t* d_bin_counts,
                                          int32_t* d_bin_offsets, ow_g2g_result* out, void* stream, int64_t* ticket) {
  *ticket = 0;
  g2g_out_init(out);
  bool fell_back = false;
  if (n_faces > 0 && g2g_device_eligible(ctx, f, p)) {
    G2GTicket* t;
    OW_TRY(ticket_get(ctx, &t));
    const int st = g2g_submit(ctx, d_records, d_coords, n_faces, geom_key, f, grid, p, d_bin_ids, bin_ids_capacity,
                              d_bin_counts, d_bin_offsets, out, (cudaStream_t)stream, t);
    g2g_reset_state(ctx);
    if (st == OW_OK) {
      *ticket = 1 + (t - (G2GTicket*)ctx->g2g_tickets);
      return OW_OK;
    }
    t->used = 0;
    if (st != G2G_RETRY) return st;
    fell_back = true;
  }
  return g2g_sync_learn(ctx, d_records, d_coords, n_faces, geom_key, f, grid, p, d_bin_ids, bin_ids_capacity,
                        d_bin_counts, d_bin_offsets, out, stream, fell_back);
}

extern "C" int ow_geometry_to_grid_finish(ow_ctx* ctx, int64_t ticket, float* d_coords, int64_t n_faces,
                                          int64_t geom_key, ow_forest* f, const ow_grid* grid, const ow_g2g_params* p,
                                          int32_t* d_bin_ids, int64_t bin_ids_capacity, int32_t* d_bin_counts,
                                          int32_t* d_bin_offsets, ow_g2g_result* out, void* stream) {
  if (ticket <= 0) return OW_OK;  // (completed by the submit)
  if (ticket > G2G_TICKETS || !ctx->g2g_tickets || !((G2GTicket*)ctx->g2g_tickets)[ticket - 1].used) {
    ow_set_error("geometry_to_grid: unknown pass ticket %lld", (long long)ticket);
    return OW_ERR_INVALID;
  }
  G2GTicket* t = (G2GTicket*)ctx->g2g_tickets + (ticket - 1);
  const int st = g2g_finish(ctx, f, p, out, (cudaStream_t)stream, t);
  t->used = 0;
  g2g_reset_state(ctx);
  if (st == OW_OK) {
    ctx->dev_passes++;
    out->device_sized = 1;
    return OW_OK;
  }
  if (st != G2G_RETRY) return st;
  g2g_out_init(out);
  return g2g_sync_learn(ctx, nullptr, d_coords, n_faces, geom_key, f, grid, p, d_bin_ids, bin_ids_capacity,
                        d_bin_counts, d_bin_offsets, out, stream, true);
}

extern "C" int ow_geometry_to_grid(ow_ctx* ctx, const uint8_t* d_records, float* d_coords, int64_t n_faces,
                                   int64_t geom_key, ow_forest* f, const ow_grid* grid, const ow_g2g_params* p,
                                   int32_t* d_bin_ids, int64_t bin_ids_capacity, int32_t* d_bin_counts,
                                   int32_t* d_bin_offsets, ow_g2g_result* out, void* stream) {
  int64_t ticket = 0;
  OW_TRY(ow_geometry_to_grid_submit(ctx, d_records, d_coords, n_faces, geom_key, f, grid, p, d_bin_ids,
                                    bin_ids_capacity, d_bin_counts, d_bin_offsets, out, stream, &ticket));
  return ow_geometry_to_grid_finish(ctx, ticket, d_coords, n_faces, geom_key, f, grid, p, d_bin_ids,
                                    bin_ids_capacity, d_bin_counts, d_bin_offsets, out, stream);
}
