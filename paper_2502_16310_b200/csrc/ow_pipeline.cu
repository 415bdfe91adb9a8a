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
#include <string.h>

#include "ow_scan.cuh"

namespace {

__global__ void k_root_init(ow_forest f, int64_t r) {
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

int record(StageEvents* se, int lv, int k, cudaStream_t s) {
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

}  // namespace

extern "C" int ow_forest_init_root(ow_ctx* ctx, ow_forest* f, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int64_t r = 1;
  for (int a = 0; a < f->dim; ++a) r *= f->root[a];
  if (f->dim < 2 || f->dim > 3 || r < 1 || r > f->capacity) {
    ow_set_error("init_root_grid: bad root grid or capacity (%lld roots, capacity %lld)", (long long)r,
                 (long long)f->capacity);
    return OW_ERR_INVALID;
  }
  k_root_init<<<ow_blocks(r, 256), 256, 0, s>>>(*f, r);
  OW_LAUNCHED(ctx);
  OW_CHECK_LAUNCH();
  f->n_blocks = r;
  return OW_OK;
}

extern "C" int ow_refine_near_wall(ow_ctx* ctx, ow_forest* f, const float* d_coords, int64_t n_faces, int64_t geom_key,
                                   const ow_grid* grid, const ow_nearwall_params* p, int32_t* d_bin_ids,
                                   int64_t bin_ids_capacity, int32_t* d_bin_counts, int32_t* d_bin_offsets,
                                   ow_nearwall_result* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
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
  for (int level = 0; level < passes; ++level) {
    // ---- bin_setup
    OW_TRY(record(se, level, 0, s));
    if (p->binned && (!have_bins || !p->reuse_bins)) {
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
      OW_TRY(ow_fill_bins_emit(ctx, grid, d_bin_ids, d_bin_counts, d_bin_offsets, s));
      have_bins = true;
      out->bin_entries = E;
      out->bins_built += 1;
    }
    // ---- face_detection
    OW_TRY(record(se, level, 1, s));
    void* pl;
    OW_TRY(ow_slot(ctx, SLOT_DRV_LEAVES, 4 * (size_t)(f->n_blocks + 1), s, &pl));
    int64_t n_leaves = 0;
    OW_TRY(ow_forest_leaves(ctx, f, level, (int32_t*)pl, &n_leaves, s));
    int64_t lo = 0, hi = n_leaves;
    if (p->world > 1) {  // contiguous count-balanced slice (parallel.partition)
      const int64_t per = (n_leaves + p->world - 1) / p->world;
      lo = per * p->rank < n_leaves ? per * p->rank : n_leaves;
      hi = per * (p->rank + 1) < n_leaves ? per * (p->rank + 1) : n_leaves;
    }
    int64_t st[3] = {0, 0, 0};
    OW_TRY(ow_mark_near_wall(ctx, f, (const int32_t*)pl + lo, hi - lo, d_coords, n_faces, geom_key,
                             p->binned ? grid : nullptr, p->binned ? d_bin_ids : nullptr,
                             p->binned ? d_bin_counts : nullptr, p->binned ? d_bin_offsets : nullptr,
                             p->binned ? E : 0, p->d_spec, p->reach, &st[0], &st[1], &st[2], s));
    if (p->world > 1) {
      if (!p->exchange) {
        ow_set_error("refine_near_wall: world > 1 needs an exchange callback");
        return OW_ERR_INVALID;
      }
      if (p->exchange(p->exchange_user, level, (const int32_t*)pl, n_leaves, lo, hi, st) != 0) {
        ow_set_error("refine_near_wall: mark exchange failed at level %d", level);
        return OW_ERR_INTERNAL;
      }
    }
    out->marked_detected[level] = st[0];
    out->tests[level] = st[1];
    out->evaluated[level] = st[2];
    // ---- propagation (binned only): 1 + floor(d / min block length)
    OW_TRY(record(se, level, 2, s));
    if (p->binned && n_leaves > 0) {
      double bl = INFINITY;
      for (int a = 0; a < f->dim; ++a) {
        const double b = f->dext[a] / (double)((int64_t)f->root[a] << level);
        bl = b < bl ? b : bl;
      }
      const int rounds = 1 + (int)floor(p->d_spec64 / bl);
      OW_TRY(ow_propagate_marks(ctx, f, (const int32_t*)pl, n_leaves, rounds, s));
    }
    // ---- refinement: MARKED leaves at level = the split count of this pass
    OW_TRY(record(se, level, 3, s));
    int64_t n_split = 0, n_marked = 0;
    OW_TRY(ow_refine_marked_counted(ctx, f, level, &n_split, &n_marked, s));
    out->marked_refined[level] = n_marked;
    out->n_split[level] = n_split;
    OW_TRY(record(se, level, 4, s));
    out->n_passes = level + 1;
  }
  OW_CUDA(cudaStreamSynchronize(s));
  for (int level = 0; level < out->n_passes; ++level)
    for (int k = 0; k < 4; ++k) {
      float ms = 0.0f;
      if (se->used[level][k] && se->used[level][k + 1])
        OW_CUDA(cudaEventElapsedTime(&ms, se->ev[level][k], se->ev[level][k + 1]));
      out->stage_ms[level][k] = ms;
    }
  return OW_OK;
}
