/*
 * owb200.h — C ABI of libowb200.so, the sm_100a geometry-to-grid hot path.
 *
 * Drop-in boundary for the reference package `octowall`
 * (/root/reference/pkg/src/octowall).  The reference is pure Python, so it has
 * no FFI of its own; each entry point below replaces one reference function
 * and is what a ctypes / cffi binding of that function binds (see
 * INTEGRATION.md).  The Python host package paper_2502_16310_b200 mirrors the
 * reference API on top of these calls.
 *
 * Conventions
 *  - Every pointer named d_* is DEVICE memory owned by the caller (PyTorch
 *    tensors in the Python package); the library owns only scratch inside an
 *    ow_ctx.  Sizes are element counts.  `stream` is a cudaStream_t.
 *  - Calls are stream-ordered.  A call that returns a host scalar through an
 *    out_* pointer synchronises `stream` before returning.
 *  - Return value: OW_OK or an error code mirroring octowall/errors.py:4-41
 *    (exit codes 2/3/4); ow_last_error() returns the thread-local message.
 *  - Arithmetic: float32 with the reference's operation order, IEEE div/sqrt,
 *    no FMA contraction (compiled -fmad=false), float64 where the reference
 *    uses float64 (cell centres, face boxes, degeneracy test).
 */
#ifndef OWB200_H
#define OWB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OW_OK = 0,
  OW_ERR_INTERNAL = 1, /* CUDA / library failure                     (OctowallError)          */
  OW_ERR_INVALID = 2,  /* bad parameter, degenerate face, outside domain (InvalidParameterError) */
  OW_ERR_PARSE = 3,    /* malformed STL                             (GeometryParseError)     */
  OW_ERR_CAPACITY = 4  /* bin / link capacity exceeded              (CapacityError)          */
};

enum { OW_NONE = 0, OW_MARKED = 1, OW_INTERMEDIATE = 2 }; /* forest.py:24-27 RefineMark */

typedef struct ow_ctx ow_ctx;

/* Regular bin grid, binning.py:34-60 (BinGrid).  min32/len32 are the float32
 * constants the reference derives (_min32 = f32(min), _len32 = f32(extent/B)). */
typedef struct {
  int32_t dim;
  int32_t bins_per_axis;
  double dmin[3];
  double dmax[3];
  float min32[3];
  float len32[3];
} ow_grid;

/* Forest-of-octrees SoA view, forest.py:47-81.  Arrays are caller-owned device
 * memory of `capacity` entries; n_blocks entries are valid.  The library grows
 * the forest through `grow`, a caller callback that must reallocate every
 * array to at least `need` entries, copy the first n_blocks entries, update
 * the pointers/capacity in *f and return 0. */
typedef struct ow_forest ow_forest;
typedef int (*ow_grow_fn)(void* user, ow_forest* f, int64_t need);
struct ow_forest {
  int32_t dim;
  int32_t max_level;
  int32_t root[3];
  int32_t _pad;
  double dmin[3];
  double dext[3];
  int64_t n_blocks;
  int64_t capacity;
  int16_t* d_level;
  int32_t* d_coord[3]; /* lattice coordinates per axis at the block's level */
  int32_t* d_parent;
  int32_t* d_first_child;
  int8_t* d_marks;
  ow_grow_fn grow;
  void* grow_user;
};

/* ---- context --------------------------------------------------------------- */
int ow_ctx_create(int device, ow_ctx** out);
int ow_ctx_destroy(ow_ctx* ctx);
const char* ow_last_error(void);
int ow_version(void);
/* kernels launched by this ctx since creation (instrumentation for bench.py) */
int64_t ow_launch_count(ow_ctx* ctx);
/* Optional CUDA-event timing of kernel families (bench.py roofline):
 * ids 0 mark, 1 lattice, 2 fill_bins, 3 refine, 4 propagate, 5 links,
 * 6 STL import, 7 face prep, 8 lattice sweep kernel alone.
 * ow_profile(ctx, 1) enables and resets. */
int ow_profile(ow_ctx* ctx, int enable);
int ow_profile_read(ow_ctx* ctx, int kernel_id, double* total_ms, int64_t* launches);

/* ---- geometry import (geometry.py) ----------------------------------------- */
/* Binary STL records (50 B each, after the 84-byte header) -> coords (3,3,F)
 * float32 SoA [vertex slot][component][face].  Replaces _parse_binary_stl +
 * _tris_to_geometry, geometry.py:415-436. */
int ow_stl_binary_to_soa(ow_ctx* ctx, const uint8_t* d_records, int64_t n_faces, float* d_coords,
                         void* stream);
/* Pure gather coords[j][c][k] = vertices[faces[k][j]][c]; index_to_coords,
 * geometry.py:262-273. */
int ow_index_to_coords(ow_ctx* ctx, int32_t dim, const float* d_vertices, const int32_t* d_faces,
                       int64_t n_faces, float* d_coords, void* stream);

/* One pass over all faces: first degenerate face (validate_faces,
 * geometry.py:276-299), first non-finite face, float32 bounding box
 * (bounding_box, geometry.py:302-308) and max |coordinate|. */
typedef struct {
  int64_t first_degenerate; /* -1 if none */
  int64_t first_nonfinite;  /* -1 if none */
  float bbox_min[3];
  float bbox_max[3];
  float abs_max;
  float mean_extent;        /* mean largest bounding-box side per face (approximate:
                               unordered float sum; shapes work, never results) */
} ow_face_summary;
int ow_face_check(ow_ctx* ctx, int32_t dim, const float* d_coords, int64_t n_faces,
                  ow_face_summary* out, void* stream);

/* ---- binning (binning.py:200-266, fill_bins) ------------------------------- */
/* Phase 1: sample every face (spacing h), count distinct (bin, face) pairs.
 * Writes d_counts[n_bins] and returns the entry total.  *out_outside is the
 * first face with a sample outside the domain (-1 if none; binning.py:74-77). */
int ow_fill_bins_count(ow_ctx* ctx, const ow_grid* grid, const float* d_coords, int64_t n_faces,
                       float spacing, int32_t* d_counts, int64_t* out_entries, int64_t* out_outside,
                       void* stream);
/* Phase 2 (after a successful phase 1 on the same ctx): d_ids[entries] grouped
 * by bin, ascending face id within each bin; d_offsets = exclusive scan. */
int ow_fill_bins_emit(ow_ctx* ctx, const ow_grid* grid, int32_t* d_ids, const int32_t* d_counts,
                      int32_t* d_offsets, void* stream);

/* ---- forest (forest.py) ----------------------------------------------------- */
/* Ascending ids of childless blocks at `level` (leaf_blocks_at, forest.py:143). */
int ow_forest_leaves(ow_ctx* ctx, const ow_forest* f, int32_t level, int32_t* d_out, int64_t* out_n,
                     void* stream);
/* Per-level block and leaf histograms (blocks_per_level / leaves_per_level). */
int ow_forest_level_counts(ow_ctx* ctx, const ow_forest* f, int64_t* out_blocks, int64_t* out_leaves,
                           int32_t max_levels, void* stream);
/* Count blocks at `level` carrying mark `mark` (leaves only if leaf_only). */
int ow_forest_count_marks(ow_ctx* ctx, const ow_forest* f, int32_t level, int32_t leaf_only,
                          int32_t mark, int64_t* out_n, void* stream);
/* Cell centres (n, 4^D, D) float32 of blocks `d_ids`, FP64 then one rounding
 * (cell_centers_many, forest.py:187-205). */
int ow_forest_cell_centers(ow_ctx* ctx, const ow_forest* f, const int32_t* d_ids, int64_t n,
                           float* d_out, void* stream);
/* Split MARKED leaves at `level` in ascending id, then restore 2:1 face
 * balance (refine_marked, forest.py:331-370).  *out_split = blocks split. */
int ow_refine_marked(ow_ctx* ctx, ow_forest* f, int32_t level, int64_t* out_split, void* stream);

/* Fill the root grid: blocks 0..R-1 at level 0, x-fastest lattice coordinates
 * (init_root_grid, forest.py:48-81, 405-409); sets f->n_blocks = R. */
int ow_forest_init_root(ow_ctx* ctx, ow_forest* f, void* stream);

/* ---- near-wall detection (nearwall.py) ------------------------------------- */
/* Mark leaves `d_leaves` (ascending, at one level) whose cell centres pass the
 * FP32 near-face predicate at d_spec for a candidate face: every face (naive,
 * d_bin_ids == NULL; mark_near_wall_naive nearwall.py:217) or the faces of the
 * cell's bin (mark_near_wall_binned nearwall.py:253; n_bin_entries = length of
 * d_bin_ids).  `reach` is the
 * reference's conservative cull radius (nearwall.py:38-40).  Outputs:
 * *out_marked newly MARKED blocks; *out_tests the algorithmic cell-face test
 * count T; *out_evaluated the pairs that reached the full
 * predicate.  geom_key identifies the immutable geometry for prep caching. */
int ow_mark_near_wall(ow_ctx* ctx, ow_forest* f, const int32_t* d_leaves, int64_t n_leaves,
                      const float* d_coords, int64_t n_faces, int64_t geom_key, const ow_grid* grid,
                      const int32_t* d_bin_ids, const int32_t* d_bin_counts, const int32_t* d_bin_offsets,
                      int64_t n_bin_entries, float d_spec, double reach, int64_t* out_marked, int64_t* out_tests,
                      int64_t* out_evaluated, void* stream);
/* `rounds` two-pass dilation rounds over leaves `d_leaves` (propagate_marks,
 * nearwall.py:321-366). */
int ow_propagate_marks(ow_ctx* ctx, const ow_forest* f, const int32_t* d_leaves, int64_t n_leaves,
                       int32_t rounds, void* stream);

/* ---- native per-level driver (refine_near_wall, nearwall.py:430-491) -------- */
#define OW_MAX_PASSES 26
/* Multi-GPU hook: after a rank marked leaves [lo, hi) of d_leaves (all
 * n_leaves leaves of `level`, ascending), make every rank's forest marks of
 * all n_leaves leaves identical and sum stats[3] (marked, tests, evaluated)
 * over ranks.  Return 0 on success. */
typedef int (*ow_exchange_fn)(void* user, int32_t level, const int32_t* d_leaves, int64_t n_leaves, int64_t lo,
                              int64_t hi, int64_t* stats3);
/* Device-side exchange between the ranks of one node (ow_comm.cu): one
 * symmetric device buffer per rank, mapped by the others through CUDA IPC;
 * exchanges are stream-ordered put / get kernels over peer memory (no host
 * round trip, no NCCL).  Collective setup: every rank calls ow_comm_create
 * (which writes its 64-byte IPC handle), the handles are all-gathered by the
 * caller (torch.distributed), then every rank calls ow_comm_open. */
#define OW_COMM_MAX 8
typedef struct ow_comm ow_comm;
int ow_comm_create(int device, int32_t rank, int32_t world, int64_t area_bytes, ow_comm** out, void* handle64);
int ow_comm_open(ow_comm* comm, const void* handles /* world x 64 bytes */);
int ow_comm_destroy(ow_comm* comm);
/* 1 when a peer missed an exchange's timeout (the exchange then gave up). */
int ow_comm_status(ow_comm* comm, int64_t* out_error);
/* All-gather of disjoint ranges: this rank's words [lo, hi) of the n words at
 * d_data reach every rank; afterwards every rank's array is whole. */
int ow_comm_allgather_u32(ow_ctx* ctx, ow_comm* comm, uint32_t* d_data, int64_t lo, int64_t hi, int64_t n,
                          void* stream);

typedef struct {
  float d_spec;           /* float32(d_spec): predicate distance */
  int32_t n_levels;       /* NearWallParams.n_levels */
  double d_spec64;        /* Python float d_spec: propagation rounds */
  double reach;           /* conservative cull reach (nearwall.py:38-40) */
  int32_t binned;         /* strategy: 1 "binned", 0 "naive" */
  int32_t reuse_bins;     /* 1: build the bin CSR once (identical every level) */
  float spacing;          /* fill_bins sample spacing h */
  int32_t rank, world;    /* marking shard of this process (world <= 1: all) */
  int64_t overlap_factor; /* fill_bins capacity = overlap_factor * n_faces */
  int64_t bin_fraction;   /* B_f (only shapes the capacity-error message) */
  ow_exchange_fn exchange;
  void* exchange_user;
  ow_comm* comm;          /* world > 1: device-side exchange (the level loop then runs with no
                             host round trip; marking slices are balanced by per-leaf work) */
} ow_nearwall_params;
typedef struct {
  int32_t n_passes;
  int32_t bins_built;
  int64_t bin_entries;
  int64_t marked_detected[OW_MAX_PASSES];
  int64_t marked_refined[OW_MAX_PASSES];
  int64_t n_split[OW_MAX_PASSES];
  int64_t tests[OW_MAX_PASSES];     /* algorithmic cell-face tests T */
  int64_t evaluated[OW_MAX_PASSES];    /* pairs that reached the full predicate */
  int64_t sphere_tests[OW_MAX_PASSES]; /* (cell, face) bounding-sphere prefilter tests */
  int64_t box_culls[OW_MAX_PASSES];    /* FP64 block-box culls (bin chunks + faces) */
  float stage_ms[OW_MAX_PASSES][4]; /* bin_setup, face_detection, propagation, refinement (CUDA events) */
} ow_nearwall_result;
/* The whole level loop in one call: per level L in 0..n_levels-2, bins (binned;
 * built into the caller's d_bin_* buffers, d_bin_ids of bin_ids_capacity
 * entries) -> mark leaves at L -> propagate (binned) -> refine.  Geometry
 * validation (degenerate faces, domain) is the caller's, as in the reference
 * it precedes the loop.  Errors carry the reference's messages. */
int ow_refine_near_wall(ow_ctx* ctx, ow_forest* f, const float* d_coords, int64_t n_faces, int64_t geom_key,
                        const ow_grid* grid, const ow_nearwall_params* params, int32_t* d_bin_ids,
                        int64_t bin_ids_capacity, int32_t* d_bin_counts, int32_t* d_bin_offsets,
                        ow_nearwall_result* out, void* stream);

/* ---- one native geometry-to-grid pass -------------------------------------- */
/* Output allocator: return 0 and set *out to `bytes` of device memory owned by
 * the caller (kept alive by it), for output `what`. */
typedef int (*ow_alloc_fn)(void* user, int32_t what, int64_t bytes, void** out);
enum { OW_OUT_LEAVES = 0, OW_OUT_FLAGS = 1, OW_OUT_CELLS = 2, OW_OUT_Q = 3 };
typedef struct {
  ow_nearwall_params nw;    /* reach <= 0: derived as nearwall.py:31-40 */
  int32_t lattice_q;        /* directions of the lattice (0: no lattice links) */
  int8_t lattice_dirs[27 * 3];
  ow_alloc_fn alloc;
  void* alloc_user;
  void* out_buf[4];         /* optional caller buffers per OW_OUT_*: used when */
  int64_t out_cap[4];       /* out_cap (bytes) covers the need, else alloc() */
  /* optional pinned host destinations of the results: the forest arrays are
   * copied on a side stream while the lattice work runs, the boundary rows
   * (cells, q) after it; the call's stream waits for both copies, so a
   * synchronisation of `stream` makes them visible.  A destination whose
   * capacity is too small is skipped (ow_g2g_result.host_copied says which). */
  void* host_level;         /* int16[host_block_cap] */
  void* host_coord[3];      /* int32[host_block_cap] per axis */
  void* host_parent;        /* int32[host_block_cap] */
  void* host_first_child;   /* int32[host_block_cap] */
  void* host_marks;         /* int8[host_block_cap] */
  int64_t host_block_cap;
  void* host_cells;         /* int64[host_row_cap] */
  void* host_q;             /* float32[host_row_cap * lattice_q] (dense rows; unused when the
                               packed destinations below are given and fit) */
  int64_t host_row_cap;
  /* packed boundary rows (preferred over host_cells / host_q when they fit):
   * per boundary row its flat cell id (uint32: finest cells < 2^32 is checked)
   * and flag word, and the q of the set bits only, rows in order and
   * directions ascending within a row — the dense q row is -1 where a bit is
   * clear, so the pair is the whole result at (8 + 4 popc) bytes per row */
  void* host_rows;          /* uint32[2 * host_row_cap]: (cell id, flag word) per row */
  void* host_q_packed;      /* float32[host_link_cap] */
  int64_t host_link_cap;
  /* Deferred host copies (a stream of passes whose transfers overlap the
   * next pass's device work): with copy_done (a cudaEvent_t of the caller)
   * and device staging buffers of its own for the packed rows (dev_rows,
   * dev_q_packed: one pair per caller-side plan), every D2H copy of the pass
   * runs on the library's copy stream, copy_done is recorded after the last
   * one and the call's stream does NOT wait for it; the next call with the
   * same copy_done waits for it on the device before it reuses the outputs.
   * The host results are valid once copy_done has completed. */
  void* copy_done;
  void* dev_rows;           /* uint32[2 * dev_row_cap] */
  void* dev_q_packed;       /* float32[dev_link_cap] */
  int64_t dev_row_cap, dev_link_cap;
  int32_t no_stage_times;   /* 1: no stage-timing events in the level loop (an event between two
                               kernels stops their programmatic overlap); stage_ms reads 0 */
} ow_g2g_params;
typedef struct {
  ow_face_summary faces;
  int32_t outside_domain;   /* 1: the bounding box left the forest domain */
  int32_t finest_level;
  ow_nearwall_result nw;
  int64_t n_finest_leaves;
  int64_t n_boundary;
  int64_t lattice_stats[3];
  int32_t host_copied;      /* bit 0: forest arrays, bit 1: boundary rows (cells + dense q),
                               bit 2: boundary rows packed (rows + packed q) */
  int32_t reran;            /* 1: the device-resident level loop outgrew the forest capacity
                               and the pass reran with a host round trip per level */
  int64_t n_links;          /* boundary links = set flag bits = packed-q length */
  int32_t device_sized;     /* 1: one device-sized pass (a single readback at its end); 2: a
                               device-sized attempt fell back to the synchronous pass; 0: synchronous */
  int32_t reserved;
} ow_g2g_result;
/* Binary STL records (or, with d_records NULL, coords already in d_coords) ->
 * validated SoA geometry -> root grid in `f` (capacity preallocated, grown
 * through f->grow) -> refine_near_wall -> finest-level leaves (int64), lattice
 * flags, boundary cells and q through `alloc`.  Errors carry the reference's
 * messages (degenerate face, outside domain, bin capacity). */
int ow_geometry_to_grid(ow_ctx* ctx, const uint8_t* d_records, float* d_coords, int64_t n_faces, int64_t geom_key,
                        ow_forest* f, const ow_grid* grid, const ow_g2g_params* params, int32_t* d_bin_ids,
                        int64_t bin_ids_capacity, int32_t* d_bin_counts, int32_t* d_bin_offsets,
                        ow_g2g_result* out, void* stream);

/* The same pass in two steps, so a stream of passes never waits for the host
 * between passes: submit enqueues it (device-sized when eligible) and returns
 * *ticket > 0 while it is in flight, or 0 when it already ran synchronously
 * (`out` final); finish waits for its summary, checks it (the reference's
 * errors), streams the host copies and fills `out` (a failed capacity or
 * assumption re-runs the pass synchronously there).  Between the two calls
 * the caller keeps every argument alive and unchanged; passes of other
 * forests / outputs may be submitted meanwhile (at most 8 in flight). */
int ow_geometry_to_grid_submit(ow_ctx* ctx, const uint8_t* d_records, float* d_coords, int64_t n_faces,
                               int64_t geom_key, ow_forest* f, const ow_grid* grid, const ow_g2g_params* params,
                               int32_t* d_bin_ids, int64_t bin_ids_capacity, int32_t* d_bin_counts,
                               int32_t* d_bin_offsets, ow_g2g_result* out, void* stream, int64_t* ticket);
int ow_geometry_to_grid_finish(ow_ctx* ctx, int64_t ticket, float* d_coords, int64_t n_faces, int64_t geom_key,
                               ow_forest* f, const ow_grid* grid, const ow_g2g_params* params, int32_t* d_bin_ids,
                               int64_t bin_ids_capacity, int32_t* d_bin_counts, int32_t* d_bin_offsets,
                               ow_g2g_result* out, void* stream);

/* Device-sized fused passes (on by default once a pass has sized the caller's
 * output buffers): enable = 0 keeps ow_geometry_to_grid on the synchronous
 * path (a host round trip per size it needs).  Stats: [0] device-sized passes,
 * [1] device-sized attempts that fell back to the synchronous path. */
int ow_set_device_pass(ow_ctx* ctx, int32_t enable);
int ow_device_pass_stats(ow_ctx* ctx, int64_t* out2);

/* Cell-face links (build_cell_face_links, nearwall.py:522-594), two phases.
 * Count: per leaf cell the faces of its bin within d_link.  On overflow of
 * `capacity` returns OW_ERR_CAPACITY with the reference's message naming the
 * first overflowing (block, bin, cell).  Emit writes the CSR. */
int ow_cell_face_links_count(ow_ctx* ctx, const ow_forest* f, const int32_t* d_leaves, int64_t n_leaves,
                             const float* d_coords, int64_t n_faces, int64_t geom_key, const ow_grid* grid,
                             const int32_t* d_bin_ids, const int32_t* d_bin_counts,
                             const int32_t* d_bin_offsets, float d_link, double reach, int64_t capacity,
                             int64_t* out_cells, int64_t* out_links, void* stream);
int ow_cell_face_links_emit(ow_ctx* ctx, int64_t* d_block_ids, int64_t* d_cell_indices, int64_t* d_offsets,
                            int32_t* d_face_ids, void* stream);

/* ---- lattice boundary links (north-star extension) -------------- */
/* Q directions d_dirs[Q][dim] (int8) of a DnQm lattice; links of every cell of
 * leaves `d_leaves` (all at `level`, the finest level) tested with FP32
 * Moller-Trumbore (3D) / segment-segment (2D) against every face whose float32
 * AABB meets the link's AABB.  `grid` is optional and unused (kept for ABI
 * stability: candidates come from the forest itself).  Phase 1 writes d_flags
 * [n_leaves * 4^D] (bit i = link i hits) and returns the boundary-cell count;
 * phase 2 writes d_cells (flat cell index, ascending) and d_q [nb][Q] = min t
 * (-1 for no hit). */
int ow_lattice_links_count(ow_ctx* ctx, const ow_forest* f, int32_t level, const int32_t* d_leaves,
                           int64_t n_leaves, const float* d_coords, int64_t n_faces, int64_t geom_key,
                           const ow_grid* grid, const int8_t* h_dirs, int32_t n_dirs, uint32_t* d_flags,
                           int64_t* out_boundary, void* stream);
/* Same, for the leaf positions [pos_lo, pos_hi) only (multi-GPU slice): the
 * flags of other positions stay 0 and only this slice's boundary rows are
 * emitted; ranks all-gather the slices (parallel.Shard). */
int ow_lattice_links_count_range(ow_ctx* ctx, const ow_forest* f, int32_t level, const int32_t* d_leaves,
                                 int64_t n_leaves, int64_t pos_lo, int64_t pos_hi, const float* d_coords,
                                 int64_t n_faces, int64_t geom_key, const ow_grid* grid, const int8_t* h_dirs,
                                 int32_t n_dirs, uint32_t* d_flags, int64_t* out_boundary, void* stream);
int ow_lattice_links_emit(ow_ctx* ctx, int64_t* d_cells, float* d_q, void* stream);
/* Emit plus the packed form: d_rows[2 * n_boundary] = (cell id as uint32, flag
 * word) per boundary row, d_q_packed[n_links] = q of the set bits (rows in
 * order, directions ascending).  Both null = ow_lattice_links_emit. */
int ow_lattice_links_emit_packed(ow_ctx* ctx, int64_t* d_cells, float* d_q, uint32_t* d_rows,
                                 float* d_q_packed, void* stream);
/* Boundary links (set flag bits over the boundary rows) of the last count. */
int ow_lattice_links_n_links(ow_ctx* ctx, int64_t* out);
/* Tuning / testing knobs of the lattice sweep (results never depend on them):
 * rows of more than `inline_units` cells are tested by the unit-balanced
 * k_lat_mt pass, the others inside the face pass (default 64: all inline);
 * faces_per_warp (1, 2, 4, 8, 16 or 32; 3D) fixes the face pass's lane groups (default: chosen
 * from the mean face size against the finest block).  Negative = default. */
int ow_lattice_tune(ow_ctx* ctx, int32_t inline_units, int32_t faces_per_warp);

/* Work counters of the last ow_lattice_links_count: [0] candidate blocks,
 * [1] (block, face, direction) rows, [2] Moller-Trumbore / segment tests. */
int ow_lattice_stats(ow_ctx* ctx, int64_t* out3, void* stream);

/* ---- output ------------------------------------------------------------------ */
/* Legacy ASCII VTK of the leaf blocks, byte-identical to export_vtk
 * (vtk_io.py:17-69): quads / hexahedra, `level` and `marked` scalars. */
int ow_export_vtk(ow_ctx* ctx, const ow_forest* f, const char* path, const char* title, void* stream);

/* ---- predicate probe (parity tests) ---------------------------------------- */
/* out[i] = near(point i, face i, d[i]) for n independent pairs; points (n, D),
 * faces (D, D, n) SoA, d float32 (n).  The device predicate used by marking. */
int ow_near_pairs(ow_ctx* ctx, int32_t dim, const float* d_points, const float* d_faces, const float* d_d,
                  int64_t n, uint8_t* d_out, void* stream);

/* ASCII STL parser (host, replaces _parse_ascii_stl geometry.py:349-412):
 * pure-ASCII STL text -> tris[n][3][3] float32 (Python float() grammar, then
 * one float32 rounding).  OW_ERR_PARSE with err[5] = {code, line, token
 * offset, token length, expected keyword index} describing the first error
 * in the reference's token order (codes: 1 end of file, 2 expected keyword
 * err[4] of {solid, normal, outer, loop, vertex, endloop, endfacet}, 3
 * expected a number, 4 expected 'facet' or 'endsolid', 5 keyword after
 * endsolid, 6 non-ASCII byte); OW_ERR_CAPACITY when more than `cap` facets. */
int ow_parse_ascii_stl(const char* data, int64_t len, float* tris, int64_t cap, int64_t* out_n, int64_t* err);

/* Predicate-vs-referee sampling (validate.py:98-141): out_mask[i] = FP32
 * near(point i, face i, f32(d[i])); out_exact[i] = FP64 exact distance of the
 * point to the closed face (distance.py:260-345, same double op order). */
int ow_referee_pairs(ow_ctx* ctx, int32_t dim, const float* d_points, const float* d_faces, const double* d_d,
                     int64_t n, double* d_exact, uint8_t* d_mask, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* OWB200_H */
