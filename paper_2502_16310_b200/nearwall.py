"""Near-wall refinement on the GPU: marking, propagation, per-level driver,
cell-face links.  Mirrors octowall/nearwall.py (names, signatures, defaults,
return values, error messages) on top of libowb200:

    mark_near_wall_naive / _binned -> ow_mark_near_wall     (nearwall.py:217, 253)
    propagate_marks                -> ow_propagate_marks    (nearwall.py:321)
    Forest.refine_marked           -> ow_refine_marked      (forest.py:331)
    build_cell_face_links          -> ow_cell_face_links_*  (nearwall.py:522)

Every host scalar the reference returns (blocks marked, entries, splits) is a
stream synchronisation point; everything else stays on the device.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, backends
from .binning import BinGrid, BinnedFaces, auto_bin_fraction, default_spacing, fill_bins
from .errors import InvalidParameterError
from .forest import Forest, RefineMark
from .geometry import CoordListGeometry, bounding_box, validate_faces


def _coordinate_scale(forest, geom):
    """nearwall.py:31-35 (|coords| max from the GPU face summary)."""
    s = max(float(np.abs(forest.domain.min).max()), float(np.abs(forest.domain.max).max()))
    if geom.n_faces:
        s = max(s, float(np.float32(geom.summary().abs_max)))
    return s


def _cull_reach(d_spec, scale):
    return d_spec + 1e-3 * max(1.0, scale, d_spec)


def _check_marking_inputs(forest, geom, d_spec):
    if geom.dim != forest.dim:
        raise InvalidParameterError(f"geometry is {geom.dim}D but forest is {forest.dim}D")
    if geom.n_faces == 0:
        raise InvalidParameterError("cannot mark near-wall blocks with empty geometry")
    if d_spec <= 0:
        raise InvalidParameterError(f"near-wall distance must be positive, got {d_spec}")
    validate_faces(geom)


@dataclass
class MarkStats:
    """Per marking pass: blocks newly marked, algorithmic tests T, pairs evaluated."""

    marked: int
    tests: int
    evaluated: int


def _mark(forest, level, geom, d_spec, bins, grid, leaves=None):
    if leaves is None:
        leaves = forest._leaves(level)
    n = int(leaves.numel())
    m, t, e = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    reach = _cull_reach(d_spec, _coordinate_scale(forest, geom))
    g = grid.c_struct() if grid is not None else None
    _lib.call("ow_mark_near_wall", _lib.ctx(), C.byref(forest.view()), _lib.ptr(leaves), n, _lib.ptr(geom.coords),
              geom.n_faces, geom.key, C.byref(g) if g is not None else None,
              _lib.ptr(bins.ids) if bins is not None else None,
              _lib.ptr(bins.counts) if bins is not None else None,
              _lib.ptr(bins.offsets) if bins is not None else None,
              int(bins.ids.numel()) if bins is not None else 0, float(np.float32(d_spec)), float(reach), C.byref(m), C.byref(t), C.byref(e), _lib.stream())
    return MarkStats(int(m.value), int(t.value), int(e.value))


def mark_near_wall_naive(forest: Forest, level, geom: CoordListGeometry, d_spec, backend=backends.SERIAL,
                         stats=False):
    """Mark leaves at ``level`` with a cell centre within d_spec of any face."""
    backends.validate_backend(backend)
    _check_marking_inputs(forest, geom, d_spec)
    s = _mark(forest, level, geom, d_spec, None, None)
    return s if stats else s.marked


def mark_near_wall_binned(forest: Forest, level, geom: CoordListGeometry, bins: BinnedFaces, grid: BinGrid,
                          d_spec, backend=backends.SERIAL, stats=False):
    """Each cell tests only the faces stored in the bin holding its centre."""
    backends.validate_backend(backend)
    _check_marking_inputs(forest, geom, d_spec)
    if bins.n_bins != grid.n_bins:
        raise InvalidParameterError("bin structure does not match the bin grid")
    s = _mark(forest, level, geom, d_spec, bins, grid)
    return s if stats else s.marked


def propagation_rounds(d_spec, block_length):
    if d_spec <= 0 or block_length <= 0:
        raise InvalidParameterError("d_spec and block_length must be positive")
    return 1 + math.floor(d_spec / block_length)


def propagate_marks(forest: Forest, level, d_spec, backend=backends.SERIAL, rounds=None):
    """Two-pass NONE -> INTERMEDIATE -> MARKED dilation over face neighbours."""
    backends.validate_backend(backend)
    if forest.count_marks(level, RefineMark.INTERMEDIATE, leaf_only=False):
        raise InvalidParameterError(f"level {level} already carries intermediate marks")
    if rounds is None:
        rounds = propagation_rounds(d_spec, float(np.min(forest.block_length(level))))
    leaves = forest._leaves(level)
    if leaves.numel() == 0 or rounds == 0:
        return
    _lib.call("ow_propagate_marks", _lib.ctx(), C.byref(forest.view()), _lib.ptr(leaves), int(leaves.numel()),
              int(rounds), _lib.stream())


@dataclass
class StageTiming:
    stage: str
    level: int
    strategy: str
    bins_per_axis: int
    bin_fraction: int
    milliseconds: float

    CSV_HEADER = "stage,level,strategy,B,B_f,milliseconds"

    def csv_row(self):
        return (f"{self.stage},{self.level},{self.strategy},{self.bins_per_axis},"
                f"{self.bin_fraction},{self.milliseconds:.3f}")


def write_timings_csv(path, timings):
    with open(path, "w", encoding="utf-8") as f:
        f.write(StageTiming.CSV_HEADER + "\n")
        for t in timings:
            f.write(t.csv_row() + "\n")


@dataclass
class NearWallParams:
    d_spec: float
    n_levels: int = 3
    strategy: str = "binned"
    bins_per_axis: int = 8
    bin_fraction: int | None = None
    overlap_factor: int = 10
    spacing: float | None = None
    backend: str = backends.SERIAL

    def __post_init__(self):
        if self.strategy not in ("naive", "binned"):
            raise InvalidParameterError(f"unknown strategy {self.strategy!r}")
        if self.n_levels < 1:
            raise InvalidParameterError(f"n_levels must be >= 1, got {self.n_levels}")
        backends.validate_backend(self.backend)


@dataclass
class NearWallResult:
    forest: Forest
    timings: list = field(default_factory=list)
    marked_detected: list = field(default_factory=list)
    marked_refined: list = field(default_factory=list)
    bins: BinnedFaces | None = None
    grid: BinGrid | None = None
    cell_face_tests: list = field(default_factory=list)  # T per marking pass
    pairs_evaluated: list = field(default_factory=list)
    sphere_tests: list = field(default_factory=list)  # bounding-sphere prefilter tests per pass
    box_culls: list = field(default_factory=list)  # FP64 block-box culls per pass

    @property
    def total_marked(self):
        return sum(self.marked_refined)

    def total_ms(self, stage=None):
        return sum(t.milliseconds for t in self.timings if stage is None or t.stage == stage)


class _Clock:
    """Stage wall clock; every stage ends in a host readback, so the GPU work
    of the stage is complete when the clock stops (same semantics as the
    reference's perf_counter records, nearwall.py:452-490)."""

    def __init__(self, sync):
        self.sync = sync

    def __enter__(self):
        if self.sync:
            torch.cuda.current_stream().synchronize()
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *a):
        if self.sync:
            torch.cuda.current_stream().synchronize()
        self.ms = 1e3 * (time.perf_counter() - self.t0)


def _driver_setup(forest, n_faces, params, reuse_bins, shard):
    """Bin buffers and the ow_nearwall_params struct of one driver call."""
    binned = params.strategy == "binned"
    b = params.bins_per_axis if binned else 1
    bf = params.bin_fraction
    if binned and bf is None:
        bf = auto_bin_fraction(b ** forest.dim, n_faces)
    if params.n_levels - 1 > _lib.MAX_PASSES:
        raise InvalidParameterError(f"n_levels must be <= {_lib.MAX_PASSES + 1}, got {params.n_levels}")
    if params.d_spec <= 0:
        raise InvalidParameterError(f"near-wall distance must be positive, got {params.d_spec}")
    backends.validate_backend(params.backend)
    grid = bins_t = g = None
    cap = 0
    h = 0.0
    if binned:
        grid = BinGrid(forest.domain, params.bins_per_axis)
        if bf < 1:
            raise InvalidParameterError(f"bin_fraction must be >= 1, got {bf}")
        h = np.float32(params.spacing) if params.spacing is not None else np.float32(default_spacing(grid))
        if h <= 0:
            raise InvalidParameterError(f"spacing must be positive, got {h}")
        cap = max(1, params.overlap_factor * n_faces)
        dev = forest.device
        bins_t = (torch.empty(cap, dtype=torch.int32, device=dev), torch.empty(grid.n_bins, dtype=torch.int32, device=dev),
                  torch.empty(grid.n_bins, dtype=torch.int32, device=dev))
        g = grid.c_struct()
    p = _lib.NearWallParamsC()
    p.d_spec = float(np.float32(params.d_spec))
    p.n_levels = params.n_levels
    p.d_spec64 = float(params.d_spec)
    p.reach = 0.0  # set by the caller (or derived natively)
    p.binned = int(binned)
    p.reuse_bins = int(bool(reuse_bins))
    p.spacing = float(h)
    p.overlap_factor = int(params.overlap_factor)
    p.bin_fraction = int(bf or 1)
    keep = None
    if shard is not None and shard.world > 1 and hasattr(shard, "allgather_"):  # parallel.DeviceComm
        p.rank, p.world = shard.rank, shard.world
        p.comm = shard.handle.value
    elif shard is not None and shard.world > 1:
        p.rank, p.world = shard.rank, shard.world
        keep = _lib.EXCHANGE_FN(shard.exchange_callback(forest))
        p.exchange = keep
    else:
        p.rank, p.world = 0, 1
    return dict(binned=binned, b=b, bf=bf, grid=grid, g=g, bins_t=bins_t, cap=cap, p=p, keep=keep)


def _driver_done(forest, out):
    forest._sync_from_view()
    forest._version += 1
    forest._leaf_cache.clear()
    for level in range(out.n_passes):
        if out.n_split[level] > 0:
            forest._n_levels = max(forest._n_levels, level + 2)


def _driver_result(forest, params, st, out) -> NearWallResult:
    result = NearWallResult(forest=forest)
    binned, b, bf = st["binned"], st["b"], st["bf"]
    stages = ("bin_setup", "face_detection", "propagation", "refinement")
    for level in range(out.n_passes):
        for k, stage in enumerate(stages):
            if stage in ("bin_setup", "propagation") and not binned:
                continue
            result.timings.append(StageTiming(stage, level, params.strategy, b, bf if binned else 1,
                                              float(out.stage_ms[level][k])))
    n = out.n_passes
    result.marked_detected = list(out.marked_detected[:n])
    result.marked_refined = list(out.marked_refined[:n])
    result.cell_face_tests = list(out.tests[:n])
    result.pairs_evaluated = list(out.evaluated[:n])
    result.sphere_tests = list(out.sphere_tests[:n])
    result.box_culls = list(out.box_culls[:n])
    if binned:
        e = int(out.bin_entries)
        ids, counts, offsets = st["bins_t"]
        result.bins = BinnedFaces(st["grid"].n_bins, ids[:e], counts, offsets)
        result.grid = st["grid"]
    return result


def refine_near_wall(forest: Forest, geom: CoordListGeometry, params: NearWallParams, reuse_bins=True,
                     shard=None) -> NearWallResult:
    """Per level L in 0..n_levels-2: bins -> mark -> propagate -> refine.

    The level loop runs natively (``ow_refine_near_wall``): one host call per
    pass over the geometry, device-event stage timings.  The bin CSR depends
    only on (geometry, grid), so it is built once and reused for every level
    (``reuse_bins``); the reference rebuilds an identical structure per level.
    ``shard`` (a ``parallel.Shard``) splits each marking pass across ranks and
    all-gathers the marks through the driver's exchange callback (multi-GPU).
    """
    if geom.n_faces == 0:
        raise InvalidParameterError("cannot refine around empty geometry")
    bbox = bounding_box(geom)
    tol = 1e-6 * forest.domain.extent
    if np.any(bbox.min < forest.domain.min - tol) or np.any(bbox.max > forest.domain.max + tol):
        raise InvalidParameterError(
            f"geometry spans {bbox.min.tolist()}..{bbox.max.tolist()}, outside the forest domain")
    if params.n_levels - 1 == 0:
        return NearWallResult(forest=forest)
    _check_marking_inputs(forest, geom, params.d_spec)
    st = _driver_setup(forest, geom.n_faces, params, reuse_bins, shard)
    p = st["p"]
    p.reach = float(_cull_reach(params.d_spec, _coordinate_scale(forest, geom)))
    out = _lib.NearWallResultC()
    g, bins_t = st["g"], st["bins_t"]
    v = forest.view()
    try:
        _lib.call("ow_refine_near_wall", _lib.ctx(), C.byref(v), _lib.ptr(geom.coords), geom.n_faces, geom.key,
                  C.byref(g) if g is not None else None, C.byref(p),
                  _lib.ptr(bins_t[0]) if bins_t else None, st["cap"],
                  _lib.ptr(bins_t[1]) if bins_t else None, _lib.ptr(bins_t[2]) if bins_t else None,
                  C.byref(out), _lib.stream())
    finally:
        _driver_done(forest, out)
    return _driver_result(forest, params, st, out)


def _mark_level(forest, level, geom, d_spec, bins, grid, shard):
    if shard is None:
        return _mark(forest, level, geom, d_spec, bins, grid)
    return shard.mark_level(forest, level, geom, d_spec, bins, grid, _mark)


@dataclass
class CellFaceLinks:
    """Per-cell face links on the finest level (CUDA tensors; nearwall.py:494-519)."""

    level: int
    d_link: float
    capacity: int
    block_ids: torch.Tensor  # (n_cells,) int64
    cell_indices: torch.Tensor  # (n_cells,) int64
    offsets: torch.Tensor  # (n_cells + 1,) int64
    face_ids: torch.Tensor  # int32

    @property
    def n_linked_cells(self):
        return int(self.block_ids.numel())

    def links_for(self, block_id, cell_index):
        sel = torch.nonzero((self.block_ids == block_id) & (self.cell_indices == cell_index)).flatten()
        if sel.numel() == 0:
            return torch.zeros(0, dtype=torch.int32, device=self.face_ids.device)
        i = int(sel[0])
        return self.face_ids[int(self.offsets[i]):int(self.offsets[i + 1])]


def build_cell_face_links(forest: Forest, geom: CoordListGeometry, bins: BinnedFaces, grid: BinGrid, d_link=None,
                          capacity=16) -> CellFaceLinks:
    """Link finest-level leaf cells to the nearby faces of their bin (GPU)."""
    _check_marking_inputs(forest, geom, 1.0 if d_link is None else d_link)
    level = forest.n_levels - 1
    if d_link is None:
        cell_len = forest.block_length(level) / 4.0
        d_link = math.sqrt(forest.dim) * float(np.linalg.norm(cell_len))
    leaves = forest._leaves(level)
    if leaves.numel() == 0:
        raise InvalidParameterError(f"no leaf blocks at finest level {level}")
    reach = _cull_reach(d_link, _coordinate_scale(forest, geom))
    g = grid.c_struct()
    ncell, nlink = C.c_int64(0), C.c_int64(0)
    ctx, st = _lib.ctx(), _lib.stream()
    _lib.call("ow_cell_face_links_count", ctx, C.byref(forest.view()), _lib.ptr(leaves), int(leaves.numel()),
              _lib.ptr(geom.coords), geom.n_faces, geom.key, C.byref(g), _lib.ptr(bins.ids), _lib.ptr(bins.counts),
              _lib.ptr(bins.offsets), float(np.float32(d_link)), float(reach), int(capacity), C.byref(ncell),
              C.byref(nlink), st)
    dev = forest.device
    nc, nl = int(ncell.value), int(nlink.value)
    block_ids = torch.empty(nc, dtype=torch.int64, device=dev)
    cell_idx = torch.empty(nc, dtype=torch.int64, device=dev)
    offsets = torch.empty(nc + 1, dtype=torch.int64, device=dev)
    face_ids = torch.empty(nl, dtype=torch.int32, device=dev)
    _lib.call("ow_cell_face_links_emit", ctx, _lib.ptr(block_ids), _lib.ptr(cell_idx), _lib.ptr(offsets),
              _lib.ptr(face_ids), st)
    return CellFaceLinks(level=level, d_link=float(d_link), capacity=capacity, block_ids=block_ids,
                         cell_indices=cell_idx, offsets=offsets, face_ids=face_ids)
