// Shared host/device infrastructure for libowb200: context, errors, scratch
// slots, launch accounting, and the exact float32/float64 arithmetic helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <functional>
#include <utility>

#include "../../include/owb200.h"

#define OW_SMS 148  // B200 SM count: persistent grids are sized in multiples of it
#define OW_PINNED_WORDS 512

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
void ow_set_error(const char* fmt, ...);

#define OW_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t _e = (call);                                                                   \
    if (_e != cudaSuccess) {                                                                   \
      ow_set_error("CUDA error %s at %s:%d", cudaGetErrorString(_e), __FILE__, __LINE__);       \
      return OW_ERR_INTERNAL;                                                                  \
    }                                                                                          \
  } while (0)

#define OW_TRY(call)              \
  do {                            \
    int _s = (call);              \
    if (_s != OW_OK) return _s;   \
  } while (0)

// ---------------------------------------------------------------------------
// context: persistent scratch slots (stream-ordered growth) + pinned readback
// ---------------------------------------------------------------------------
enum ow_slot {
  SLOT_SCAN_STATUS = 0,
  SLOT_SCAN_AUX,
  SLOT_FACE_PREP,      // predicate payload cache
  SLOT_FACE_BOX,       // float32 face boxes (lo[D], hi[D])
  SLOT_FACE_SPHERE,    // float4 bounding spheres (reach dependent)
  SLOT_BIN_MASK,       // per-face bin bitmask (fill_bins)
  SLOT_BIN_NB,         // per-face distinct-bin count
  SLOT_BIN_FOFF,       // per-face pair offset
  SLOT_BIN_SLOW,       // slow-path face list
  SLOT_BIN_SLOWOFF,    // slow-path bitmap offsets
  SLOT_BIN_BITMAP,     // slow-path bitmaps
  SLOT_PAIR_KEY0,      // radix sort ping-pong
  SLOT_PAIR_VAL0,
  SLOT_PAIR_KEY1,
  SLOT_PAIR_VAL1,
  SLOT_RADIX_HIST,
  SLOT_FOREST_LIST,    // split / violator lists
  SLOT_FOREST_FLAG,    // violator flags
  SLOT_LINK_CNT,       // per-cell link counts
  SLOT_LINK_OFF,
  SLOT_LINK_CELLOFF,
  SLOT_LINK_LEAVES,
  SLOT_LAT_BCOUNT,     // boundary cells per candidate block
  SLOT_LAT_BOFFS,      // boundary-row offsets per candidate block
  SLOT_LAT_LEAVES,     // candidate-block leaf positions
  SLOT_LAT_RANK,       // candidate-block rank per leaf position
  SLOT_LAT_POS,        // leaf position per block id
  SLOT_LAT_HAS,        // leaf has at least one candidate row
  SLOT_LAT_CEN,        // per-leaf float32 cell-centre coordinates [D][4]
  SLOT_LAT_REC,        // packed face records (v0, e1, e2)
  SLOT_LAT_ROWS,       // (leaf, face, block, direction|cell ranges) rows
  SLOT_LAT_ROWOFF,     // units per row -> unit offsets
  SLOT_LAT_TILEROW,    // first row of each intersection tile
  SLOT_LAT_HITS,       // hit list (flat cell, t bits)
  SLOT_LAT_HITDIR,     // hit list directions
  SLOT_LAT_TILEHITS,   // hits per intersection tile
  SLOT_BIN_MID,        // faces whose bins need the sample walk
  SLOT_LAT_IHITS,      // hit list of the rows swept inline by k_lat_faces (flat cell, t bits)
  SLOT_LAT_IHITDIR,    // ... and their directions
  SLOT_LAT_BMASK,      // boundary-cell mask per candidate block
  SLOT_MARK_CBOX,      // union boxes of 32-entry bin chunks (marking cull)
  SLOT_MARK_ITEMS,     // (block, chunk, bin) marking items
  SLOT_MARK_HIT,       // per-leaf hit words of a marking pass
  SLOT_DRV_LEAVES,     // native driver: leaves of the current level
  SLOT_DRV_STATS,      // native driver: per-pass marking statistics
  SLOT_DRV_STATE,      // native driver: per-pass leaf count + refine state
  SLOT_LAT_HCOUNT,     // boundary links (set flag bits) per candidate block
  SLOT_LAT_HOFFS,      // packed-q offsets per candidate block
  SLOT_LAT_RFLAGS,     // (cell id, flag word) per boundary row (packed host output)
  SLOT_LAT_QPACK,      // q of the set flag bits, row-major (packed host output)
  SLOT_LAT_GRID,       // dense finest-level lattice -> leaf position
  SLOT_DRV_SLICE,      // native driver, multi-GPU: per-leaf work prefix + slice bounds
  SLOT_SCAN_STATUS_G,  // look-back status words of scans inside a CUDA graph (ow_graph.cu)
  SLOT_MISC,
  SLOT_COUNT
};

// optional per-kernel CUDA-event timing (bench.py roofline instrumentation)
enum { PROF_MARK = 0, PROF_LATTICE, PROF_BINS, PROF_REFINE, PROF_PROP, PROF_LINKS, PROF_STL, PROF_PREP,
       PROF_LAT_SWEEP, PROF_N };
#define PROF_MAX 256
struct ow_prof {
  int enabled;
  int n[PROF_N];
  cudaEvent_t ev[PROF_N][PROF_MAX][2];
};

struct GraphKey;
struct ow_ctx {
  int device;
  ow_prof* prof;
  void* slot_ptr[SLOT_COUNT];
  size_t slot_bytes[SLOT_COUNT];
  int64_t* h_pinned;  // OW_PINNED_WORDS int64 of pinned host memory for readbacks
  int64_t* h_pinned_dev;  // the same memory mapped into the device (lazily resolved)
  int64_t* d_small;   // 64 int64 of device scalars (counters, flags)
  int64_t launches;
  int64_t scan_epoch;  // epoch of the last scan (status words are epoch-tagged)
  // face prep cache key
  int64_t prep_key;
  float prep_d;
  double prep_reach;
  int64_t prep_faces;
  int32_t prep_dim;
  // fill_bins phase state
  int64_t bins_faces, bins_entries, bins_slow;
  int32_t bins_dim, bins_B;
  float bins_h;
  const float* bins_coords;
  // cell-face link phase state
  int64_t link_cells, link_total, link_leaves;
  int32_t link_dim, link_nbins;
  const float* link_coords;
  const int32_t *link_bin_ids, *link_bin_counts, *link_bin_offsets;
  const int32_t* link_leaves_ptr;
  int64_t link_key, link_faces;
  float link_d;
  double link_reach;
  ow_forest link_forest;
  ow_grid link_grid;
  // lattice phase state
  int64_t lat_leaves, lat_boundary, lat_faces, lat_ncb, lat_rows, lat_units, lat_links;
  int64_t lat_row_cap, lat_unit_cap, lat_ihit_cap;
  int32_t lat_inline_units;
  bool lat_inline_set;
  float lat_mean_extent;
  int32_t lat_fpw;  // faces per warp of the face pass (0: chosen per call)  // mean largest face side when known (geometry_to_grid), else 0
  int64_t lat_pos_lo, lat_pos_hi;  // leaf-position slice of the last count call  // capacities of the single-pass row / unit lists
  int32_t lat_dirs, lat_level;
  bool lat_grid_on;  // the last count call built the dense finest-lattice table
  ow_comm* lat_comm;  // multi-GPU lattice stage: flags / q rows of the position slice exchanged
  int8_t lat_dir[27 * 3];
  const float* lat_coords;
  const int32_t* lat_leaves_ptr;
  uint32_t* lat_flags;
  ow_forest lat_forest;
  void* stage_events;  // native driver CUDA events
  cudaStream_t copy_stream;       // side stream for result copies (lazily created)
  cudaEvent_t copy_ev[2];         // [0] forest final, [1] copies done
  bool defer_stage_times;
  bool no_stage_events;  // fused pass without stage-timing events (ow_g2g_params.no_stage_times)
  // fused pass: the face check's summary words on the device, not yet read
  // (ow_faces_settle reads them with the next readback and validates)
  const int64_t* faces_pending;
  void* faces_state;  // the fused call's (result, forest, parameters) for ow_faces_settle
  int64_t drv_spec_nl;  // leaves of the deepest level compacted by the device-resident driver (-1: none)
  // CUDA graph of the device-resident level loop (ow_graph.cu)
  bool capturing;                      // stream capture in progress: scratch must not grow
  bool capture_failed;
  int graph_site;                      // scans recorded in the current capture
  unsigned long long* d_graph_epoch;   // device epoch base of the scans inside the graph
  // a few graphs per context (a stream of passes may alternate plans)
  cudaGraphExec_t loop_exec[4];
  GraphKey* loop_key[4];               // inputs of each captured loop
  int64_t loop_launches[4];            // kernels per replay
  GraphKey* eager_key[4];              // inputs of recent eager passes
  int loop_next, eager_next;           // round-robin victims
  cudaStream_t capture_stream;         // private stream the loop is recorded on (the caller's may be the
                                       // legacy default stream, which cannot be captured)
  // device-sized fused pass (ow_pipeline.cu: g2g_device): capacities learnt
  // from earlier passes, one readback per pass
  bool dev_pass;                       // refine_driver runs inside a device-sized pass
  int dev_disabled;                    // ow_set_device_pass(ctx, 0): always the synchronous path
  int64_t dev_e_cap;                   // bin entries (0: no estimate yet)
  int64_t dev_ncb;                     // candidate blocks of the last pass (emit grid)
  float dev_mean_extent;               // face summary of the last pass (face-pass shape)
  int64_t dev_passes, dev_fallbacks;   // statistics
  void* g2g_tickets;                   // passes in flight (ow_geometry_to_grid_submit / _finish)
  int64_t* g2g_ring;                   // their summary areas: mapped pinned host memory ...
  int64_t* g2g_ring_dev;               // ... and its device alias
};

// host-side inputs of the device-resident loop (a replay is valid only when
// they are all unchanged)
struct GraphKey {
  ow_forest f;
  ow_grid g;
  ow_nearwall_params p;
  const void* coords;
  int64_t n_faces;
  const void *ids, *counts, *offsets;
  int64_t E;
  const void *stats, *drv;
  int dev;  // captured inside a device-sized pass (bins counted on the device)
  void* slot_ptr[SLOT_COUNT];
  size_t slot_bytes[SLOT_COUNT];
};
void make_loop_key(GraphKey* k, const ow_ctx* ctx, const ow_forest* f, const float* d_coords, int64_t n_faces,
                   const ow_grid* grid, const ow_nearwall_params* p, const int32_t* ids, const int32_t* counts,
                   const int32_t* offsets, int64_t E, const void* stats, const void* drv);
int ow_loop_graph(ow_ctx* ctx, bool ok, const GraphKey* key, cudaStream_t* ps, const std::function<int()>& body);

// multi-GPU exchange over peer memory (ow_comm.cu)
struct ow_comm {
  int device, rank, world, open;
  int64_t area_bytes;           // bytes of each of the two data areas
  void* local;                  // this rank's symmetric buffer (header + 2 areas)
  uint8_t* peer[OW_COMM_MAX];   // every rank's buffer mapped here (peer[rank] = local)
  int64_t epoch;                // exchanges so far (identical sequence on every rank)
  int64_t* d_err;               // device error word: a peer missed the timeout
  unsigned* d_counter;          // CTAs done of the current put
};
size_t ow_comm_area(const ow_comm* c, int64_t epoch);
int ow_comm_check(ow_comm* c, int64_t bytes, const char* what);
// all-gather of disjoint 32-bit word ranges: [lo, hi) from d_range (device
// int64[2]) or the host values; n (or *d_n) words in the array
int ow_comm_allgather_words(ow_ctx* ctx, ow_comm* c, uint32_t* d_data, const int64_t* d_range, int64_t lo, int64_t hi,
                            const int64_t* d_n, int64_t n, cudaStream_t s);
// marks of leaf positions d_slice[0..1) of d_leaves + n_stats u64 statistics
// (summed over ranks into d_stats)
int ow_comm_exchange_marks(ow_ctx* ctx, ow_comm* c, const int32_t* d_leaves, int8_t* d_marks, const int64_t* d_slice,
                           const int64_t* d_n, int64_t n_bound, unsigned long long* d_stats, int n_stats,
                           cudaStream_t s);

// marking statistics per pass: [0] marked, [1] tests T, [2] evaluated,
// [3] sphere tests, [4] box culls, [5] the pass's (block, chunk) item counter
constexpr int MARK_STATS = 8;  // marked, T, evaluated, spheres, culls, items, block-pass counter, -

// one marking pass without a host round trip: stats accumulate in d_out[0..5)
// (d_out[5]: the item counter, zero on entry like the statistics)
int ow_mark_launch(ow_ctx* ctx, ow_forest* f, const int32_t* d_leaves, int64_t n_leaves, const float* d_coords,
                   int64_t n_faces, int64_t geom_key, const ow_grid* grid, const int32_t* d_bin_ids,
                   const int32_t* d_bin_counts, const int32_t* d_bin_offsets, int64_t n_bin_entries, float d_spec,
                   double reach, unsigned long long* d_out, cudaStream_t s,
                   const int64_t* d_n_leaves = nullptr, bool chunk_boxes_ready = false,
                   const int64_t* d_slice = nullptr, const int64_t* d_bin_entries = nullptr, int level = -1);

// device-sized lattice stage of the fused pass (ow_lattice.cu)
int ow_lattice_dev_count(ow_ctx* ctx, const ow_forest* f, int32_t level, const int32_t* d_leaves, const int64_t* d_nl,
                         int64_t nl_cap, const float* d_coords, int64_t n_faces, const int8_t* h_dirs, int32_t n_dirs,
                         uint32_t* d_flags, cudaStream_t s, int64_t* d_leaves64);
int ow_lattice_dev_emit(ow_ctx* ctx, int64_t* d_cells, float* d_q, int64_t row_cap, uint32_t* d_rows,
                        float* d_q_packed, int64_t link_cap, int64_t ncb_grid, cudaStream_t s);

void ow_g2g_release(ow_ctx* ctx);  // passes-in-flight table (ow_pipeline.cu)

// fill_bins with the entry count left on the device (ow_binning.cu: fill_dev)
int ow_fill_bins_dev(ow_ctx* ctx, const ow_grid* grid, const float* d_coords, int64_t n_faces, float spacing,
                     int32_t* d_counts, int32_t* d_ids, int32_t* d_offsets, int64_t e_cap, cudaStream_t s,
                     bool init = true);

int ow_stage_times(ow_ctx* ctx, ow_nearwall_result* out);

// device-driven forest steps of the native driver (ow_forest.cu); refine
// ring state per pass (int64 words, see ow_refine_dev)
enum { RS_INTER = 0, RS_OVER, RS_MARKED, RS_SPLITS, RS_RESUME, RS_OVER_FIRST, RS_NR = 8, RS_CR = 36, RS_WORDS = 64 };
constexpr int RS_MAX_ITERS = 26;
// 2:1 violator sweeps after splitting the MARKED leaves of `level` (children
// at level + 1): a violator of a block at depth c has depth < c - 1, and the
// children of a violator at depth v are at depth v + 1, so sweep k (k >= 1) can
// only find leaves at depth <= level - k.  `level` sweeps therefore finish
// every cascade (none at level 0: no leaf is shallower than 0); only a level
// past RS_MAX_ITERS needs the last sweep's list checked (then the host path
// finishes the cascade).
__host__ __device__ __forceinline__ int refine_sweeps(int level) {
  return level < RS_MAX_ITERS ? level : RS_MAX_ITERS;
}
__host__ __device__ __forceinline__ bool refine_sweeps_exact(int level) { return level < RS_MAX_ITERS; }
// device-driven forest steps of the native driver (ow_forest.cu)
int ow_forest_leaves_dev(ow_ctx* ctx, const ow_forest* f, int32_t level, int32_t* d_out, int64_t* d_count,
                         cudaStream_t s, const int64_t* d_nb = nullptr);
int ow_propagate_dev(ow_ctx* ctx, const ow_forest* f, const int32_t* d_leaves, const int64_t* d_n, int64_t n_bound,
                     int32_t rounds, cudaStream_t s, bool tags = false, bool defer_promote = false);
int ow_refine_dev(ow_ctx* ctx, ow_forest* f, int32_t level, int32_t iters, int64_t* d_st, cudaStream_t s,
                  int64_t* d_nb = nullptr, int32_t* next_leaves = nullptr, int64_t* next_count = nullptr,
                  const int32_t* promote_leaves = nullptr, const int64_t* promote_n = nullptr);
int ow_rebalance_host(ow_ctx* ctx, ow_forest* f, int64_t f0, int64_t* n_split, cudaStream_t s);

// refine_marked returning the MARKED-leaf count of the split pass as well
int ow_refine_marked_counted(ow_ctx* ctx, ow_forest* f, int32_t level, int64_t* out_split, int64_t* out_marked,
                             cudaStream_t s);

// Scratch slot of at least `bytes`; contents are preserved across calls unless
// the slot grows (then it is reallocated, stream-ordered, uninitialised).
int ow_slot(ow_ctx* ctx, int slot, size_t bytes, cudaStream_t s, void** out);

// cudaMemsetAsync semantics as a PDL kernel (hot paths)
int ow_fill_async(ow_ctx* ctx, void* p, int value, size_t bytes, cudaStream_t s);

// Copy n int64 device values to host and synchronise.
int ow_readback(ow_ctx* ctx, const int64_t* d_src, int n, int64_t* h_dst, cudaStream_t s);
// the pending face summary (ctx->faces_pending): validate it (errors of the
// reference's import order) and derive the near-wall reach.  h6 = the words
// if they were already read with another readback, else null (reads them).
int ow_faces_settle(ow_ctx* ctx, const int64_t* h6, cudaStream_t s);
void ow_face_summary_from(const int64_t* h, int64_t n, ow_face_summary* out);
int ow_face_check_launch(ow_ctx* ctx, int32_t dim, const float* d_coords, int64_t n, int64_t* dst, cudaStream_t s);
int ow_stl_to_soa_checked(ow_ctx* ctx, const uint8_t* d_records, int64_t n, float* d_coords, int64_t* dst,
                          cudaStream_t s, bool init_summary = true);
// the face summary's initial words (as k_face_check_init), for a kernel that
// initialises them itself (the fused pass's first kernel)
__device__ __forceinline__ void ow_face_summary_init_words(int64_t* small) {
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

// bracket device work of kernel family `id` with events when profiling is on
void ow_prof_mark(ow_ctx* ctx, int id, int end, cudaStream_t s);
#define OW_PROF_BEGIN(ctx, id, s) \
  do {                            \
    if ((ctx)->prof && (ctx)->prof->enabled) ow_prof_mark(ctx, id, 0, s); \
  } while (0)
#define OW_PROF_END(ctx, id, s) \
  do {                          \
    if ((ctx)->prof && (ctx)->prof->enabled) ow_prof_mark(ctx, id, 1, s); \
  } while (0)

#define OW_LAUNCHED(ctx) ((ctx)->launches++)
#define OW_CHECK_LAUNCH()                                                                        \
  do {                                                                                           \
    cudaError_t _e = cudaGetLastError();                                                         \
    if (_e != cudaSuccess) {                                                                     \
      ow_set_error("kernel launch failed: %s at %s:%d", cudaGetErrorString(_e), __FILE__, __LINE__); \
      return OW_ERR_INTERNAL;                                                                    \
    }                                                                                            \
  } while (0)

static inline int ow_blocks(int64_t n, int threads, int64_t cap = 1 << 30) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

// ---- programmatic dependent launch (PDL) ------------------------------------
// Every kernel is launched with programmatic stream serialization: its CTAs may
// be scheduled while the previous kernel on the stream drains, and the kernel's
// first statement, ow_pdl_wait() (griddepcontrol.wait), blocks until that
// kernel has completed and its memory is visible.  Back-to-back dependent
// launches (the level loop is a chain of ~60 short kernels) then overlap their
// launch latency with the predecessor's tail instead of serialising it.
// OW_PDL=0 in the environment launches without the attribute (A/B timing).
// (no explicit griddepcontrol.launch_dependents: the implicit trigger at CTA
// exit measured faster than triggering at kernel start, C2 0.62 vs 0.64 ms)
__device__ __forceinline__ void ow_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool ow_pdl_enabled();

template <typename... KArgs, typename... Args>
static inline void ow_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = ow_pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// exact arithmetic: explicit round-to-nearest intrinsics never contract to FMA
// ---------------------------------------------------------------------------
#define FADD(a, b) __fadd_rn((a), (b))
#define FSUB(a, b) __fsub_rn((a), (b))
#define FMUL(a, b) __fmul_rn((a), (b))
#define FDIV(a, b) __fdiv_rn((a), (b))
#define FSQRT(a) __fsqrt_rn(a)
#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DMUL(a, b) __dmul_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))

// ((a0*b0 + a1*b1) + a2*b2) in float32, left to right
__device__ __forceinline__ float dot3f(float a0, float a1, float a2, float b0, float b1, float b2) {
  return FADD(FADD(FMUL(a0, b0), FMUL(a1, b1)), FMUL(a2, b2));
}

// ---------------------------------------------------------------------------
// grid constants on device
// ---------------------------------------------------------------------------
struct GridC {
  int dim, B;
  float min32[3], len32[3];
  double lo_tol[3], hi_tol[3];  // domain +- 1e-6 * extent (binning.py:71-77)
};

static inline GridC make_gridc(const ow_grid* g) {
  GridC c;
  c.dim = g->dim;
  c.B = g->bins_per_axis;
  for (int a = 0; a < 3; ++a) {
    c.min32[a] = g->min32[a];
    c.len32[a] = g->len32[a];
    double ext = g->dmax[a] - g->dmin[a];
    double tol = 1e-6 * ext;
    c.lo_tol[a] = g->dmin[a] - tol;
    c.hi_tol[a] = g->dmax[a] + tol;
  }
  return c;
}

// floor((p - min32) / len32) -> int64 -> clip [0, B-1]  (binning.py:78-79)
__device__ __forceinline__ int bin_axis(float p, float mn, float ln, int B) {
  float f = floorf(FDIV(FSUB(p, mn), ln));
  if (!(f >= 0.0f)) return 0;  // negative (NaN impossible for finite input)
  if (f >= (float)(B - 1)) return B - 1;
  return (int)f;
}

__device__ __forceinline__ bool outside_domain(const GridC& g, const float* p) {
  for (int a = 0; a < g.dim; ++a) {
    double v = (double)p[a];
    if (v < g.lo_tol[a] || v > g.hi_tol[a]) return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// forest device view + helpers
// ---------------------------------------------------------------------------
constexpr int OW_QLEV = 16;  // block edges of levels 0..15 precomputed on the host
struct ForestC {
  int dim, max_level;
  int root[3];
  double dmin[3], dext[3];
  double qlev[OW_QLEV][3];  // extent / (root * 2^level): the same IEEE division as block_len
  int64_t n;
  const int16_t* level;
  const int32_t* coord[3];
  const int32_t* parent;
  const int32_t* first_child;
  int8_t* marks;
};

static inline ForestC make_forestc(const ow_forest* f) {
  ForestC c;
  c.dim = f->dim;
  c.max_level = f->max_level;
  for (int a = 0; a < 3; ++a) {
    c.root[a] = f->root[a];
    c.dmin[a] = f->dmin[a];
    c.dext[a] = f->dext[a];
    c.coord[a] = f->d_coord[a];
  }
  for (int l = 0; l < OW_QLEV; ++l)
    for (int a = 0; a < 3; ++a)
      c.qlev[l][a] = a < f->dim ? f->dext[a] / (double)((int64_t)f->root[a] << l) : 1.0;
  c.n = f->n_blocks;
  c.level = f->d_level;
  c.parent = f->d_parent;
  c.first_child = f->d_first_child;
  c.marks = f->d_marks;
  return c;
}

// block edge per axis: extent / (root * 2^level)   (forest.py:152-161)
__device__ __forceinline__ double block_len(const ForestC& F, int ax, int level) {
  // (a table lookup for the usual levels: an FP64 division per block and axis
  // was the heaviest part of the marking / links prologues)
  if (level < OW_QLEV) return F.qlev[level][ax];
  return DDIV(F.dext[ax], (double)((int64_t)F.root[ax] << level));
}

// Deepest existing block on the path from the root lattice to lattice cell
// (level, nc): the block itself if it exists, else the coarser leaf covering
// it.  Replaces the (level, coords) dictionary walk of forest.py:246-261.
__device__ __forceinline__ int locate(const ForestC& F, int level, const int32_t* nc, int* out_depth) {
  int node = 0, stride = 1;
  for (int a = 0; a < F.dim; ++a) {
    node += (nc[a] >> level) * stride;
    stride *= F.root[a];
  }
  int depth = 0;
  while (depth < level) {
    int fc = F.first_child[node];
    if (fc < 0) break;
    int sh = level - 1 - depth, ci = 0;
    for (int a = 0; a < F.dim; ++a) ci |= ((nc[a] >> sh) & 1) << a;
    node = fc + ci;
    ++depth;
  }
  *out_depth = depth;
  return node;
}

// Lattice neighbour of block (level, c) across side s = 2*axis + (step>0);
// returns false at the domain boundary.
__device__ __forceinline__ bool side_target(const ForestC& F, int level, const int32_t* c, int s,
                                            int32_t* nc) {
  int ax = s >> 1, step = (s & 1) ? 1 : -1;
  for (int a = 0; a < 3; ++a) nc[a] = (a < F.dim) ? c[a] : 0;
  nc[ax] += step;
  int64_t dimax = (int64_t)F.root[ax] << level;
  return nc[ax] >= 0 && nc[ax] < dimax;
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
