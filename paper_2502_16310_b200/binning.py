"""Spatial binning of geometry faces over a regular grid — sm_100a fill_bins.

Mirrors octowall/binning.py (BinGrid, BinnedFaces, fill_bins, bin_of_point,
discretize_face, ...).  ``fill_bins`` runs on the GPU (csrc/ow_binning.cu):
a face is stored in every bin touched by one of its float32 discretisation
samples, ids ascending per bin, with the reference's capacity rule and error
messages.  ``bin_fraction`` is accepted and validated but, as in the
reference, cannot change the output (it only sized the reference's dense
per-batch indicator, which this implementation does not need).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, backends
from .errors import CapacityError, InvalidParameterError
from .geometry import Aabb, CoordListGeometry, bounding_box, validate_faces

F32 = np.float32
EMPTY = np.int32(-1)
DEFAULT_OVERLAP_FACTOR = 10
_SLOT_BUDGET = 2 ** 25
_DOMAIN_REL_TOL = 1e-6


@dataclass
class BinGrid:
    """Regular grid of bins_per_axis**dim bins covering the domain box."""

    domain: Aabb
    bins_per_axis: int

    def __post_init__(self):
        if self.bins_per_axis < 1:
            raise InvalidParameterError(f"bins_per_axis must be >= 1, got {self.bins_per_axis}")
        if np.any(self.domain.extent <= 0):
            raise InvalidParameterError("bin grid domain must have positive extent")
        self._min32 = self.domain.min.astype(np.float32)
        self._len32 = (self.domain.extent / self.bins_per_axis).astype(np.float32)

    @property
    def dim(self):
        return self.domain.dim

    @property
    def n_bins(self):
        return self.bins_per_axis ** self.dim

    @property
    def bin_length(self):
        return self.domain.extent / self.bins_per_axis

    def c_struct(self):
        g = _lib.Grid()
        g.dim = self.dim
        g.bins_per_axis = self.bins_per_axis
        for a in range(self.dim):
            g.dmin[a] = float(self.domain.min[a])
            g.dmax[a] = float(self.domain.max[a])
            g.min32[a] = float(self._min32[a])
            g.len32[a] = float(self._len32[a])
        return g


def linear_bin_indices(points, grid: BinGrid, what="point"):
    """Host helper (binning.py:63-85) for small point sets; x fastest, clamped."""
    p = np.asarray(points, dtype=np.float32)
    tol = _DOMAIN_REL_TOL * grid.domain.extent
    bad = np.any((p < grid.domain.min - tol) | (p > grid.domain.max + tol), axis=-1)
    if np.any(bad):
        raise InvalidParameterError(f"{what} outside binning domain: {p[bad][0].tolist()}")
    idx = np.clip(np.floor((p - grid._min32) / grid._len32).astype(np.int64), 0, grid.bins_per_axis - 1)
    lin = np.zeros(idx.shape[:-1], np.int64)
    for ax in range(grid.dim - 1, -1, -1):
        lin = lin * grid.bins_per_axis + idx[..., ax]
    return lin


def bin_of_point(p, grid: BinGrid):
    p = np.asarray(p, dtype=np.float32).reshape(1, grid.dim)
    lin = int(linear_bin_indices(p, grid)[0])
    tup, rem = [], lin
    for _ in range(grid.dim):
        tup.append(rem % grid.bins_per_axis)
        rem //= grid.bins_per_axis
    return tuple(tup), lin


def default_spacing(grid: BinGrid):
    """Half the smallest bin edge, float32 (binning.py:101-103)."""
    return float(F32(0.5) * grid._len32.min())


def _segment_samples(a, b, h):
    d = b - a
    sq = d[0] * d[0]
    for ax in range(1, len(d)):
        sq = sq + d[ax] * d[ax]
    n = int(np.ceil(np.sqrt(sq) / h))
    t = np.arange(n + 1, dtype=np.float32) / F32(max(n, 1))
    return a + t[:, None] * d


def discretize_face(face, spacing):
    """Sample points of one face (host utility; binning.py:106-127)."""
    f = np.asarray(face, dtype=np.float32)
    if f.ndim != 2 or f.shape[0] not in (2, 3) or f.shape[1] != f.shape[0]:
        raise InvalidParameterError(f"face must be (2,2) or (3,3), got {f.shape}")
    if spacing <= 0:
        raise InvalidParameterError(f"spacing must be positive, got {spacing}")
    h = F32(spacing)
    if f.shape[0] == 2:
        if np.array_equal(f[0], f[1]):
            raise InvalidParameterError("degenerate edge: identical endpoints")
        return _segment_samples(f[0], f[1], h)
    g = CoordListGeometry(3, f[:, :, None].copy())
    validate_faces(g)
    base = _segment_samples(f[0], f[1], h)
    return np.vstack([_segment_samples(p, f[2], h) for p in base])


@dataclass
class FaceBinIndicator:
    """Dense per-batch occupancy of the reference (binning.py:140-150), kept for API parity."""

    slots: np.ndarray
    first_bin: int
    batch_index: int

    @property
    def batch_bins(self):
        return self.slots.shape[1]


def compact_indicators(indicator: FaceBinIndicator):
    occ = indicator.slots != EMPTY
    counts = occ.sum(axis=0, dtype=np.int32)
    ids = np.nonzero(occ.T)[1].astype(np.int32)
    return counts, ids


class BinnedFaces:
    """Face ids grouped by bin (CUDA int32 tensors): ids, counts, offsets."""

    def __init__(self, n_bins, ids, counts, offsets):
        self.n_bins = int(n_bins)
        self.ids = ids
        self.counts = counts
        self.offsets = offsets

    def faces_in_bin(self, b):
        o, c = int(self.offsets[b]), int(self.counts[b])
        return self.ids[o:o + c]

    def numpy(self):
        return self.ids.cpu().numpy(), self.counts.cpu().numpy(), self.offsets.cpu().numpy()

    def __eq__(self, other):
        if not isinstance(other, BinnedFaces):
            return NotImplemented
        return (self.n_bins == other.n_bins and torch.equal(self.ids.cpu(), other.ids.cpu())
                and torch.equal(self.counts.cpu(), other.counts.cpu())
                and torch.equal(self.offsets.cpu(), other.offsets.cpu()))

    def dump_csv(self, path):
        counts, offsets = self.counts.cpu().numpy(), self.offsets.cpu().numpy()
        with open(path, "w", encoding="utf-8") as f:
            f.write("bin_id,count,offset\n")
            for b in range(self.n_bins):
                f.write(f"{b},{counts[b]},{offsets[b]}\n")


def auto_bin_fraction(n_bins, n_faces, slot_budget=_SLOT_BUDGET):
    if n_faces == 0:
        return 1
    return max(1, math.ceil(n_bins * max(1, n_faces) / slot_budget))


def batch_ranges(n_bins, bin_fraction):
    if bin_fraction < 1:
        raise InvalidParameterError(f"bin_fraction must be >= 1, got {bin_fraction}")
    bf = min(bin_fraction, n_bins)
    per = math.ceil(n_bins / bf)
    return [(s, min(s + per, n_bins)) for s in range(0, n_bins, per)]


def check_in_domain(geom: CoordListGeometry, domain: Aabb, what="face outside binning domain"):
    bbox = bounding_box(geom)
    tol = _DOMAIN_REL_TOL * domain.extent
    if np.any(bbox.min < domain.min - tol) or np.any(bbox.max > domain.max + tol):
        raise InvalidParameterError(f"{what}: geometry spans {bbox.min.tolist()}..{bbox.max.tolist()}")


def fill_bins(geom: CoordListGeometry, grid: BinGrid, bin_fraction=None, overlap_factor=DEFAULT_OVERLAP_FACTOR,
              spacing=None, backend=backends.SERIAL) -> BinnedFaces:
    """Assign every face to each bin touched by its discretisation (GPU)."""
    backends.validate_backend(backend)
    if geom.dim != grid.dim:
        raise InvalidParameterError(f"geometry is {geom.dim}D but bin grid is {grid.dim}D")
    if geom.n_faces == 0:
        raise InvalidParameterError("cannot bin empty geometry")
    validate_faces(geom)
    check_in_domain(geom, grid.domain)
    if bin_fraction is None:
        bin_fraction = auto_bin_fraction(grid.n_bins, geom.n_faces)
    batches = batch_ranges(grid.n_bins, bin_fraction)
    h = F32(spacing) if spacing is not None else F32(default_spacing(grid))
    if h <= 0:
        raise InvalidParameterError(f"spacing must be positive, got {h}")
    n_faces = geom.n_faces
    capacity = overlap_factor * n_faces
    dev = geom.coords.device
    counts = torch.empty(grid.n_bins, dtype=torch.int32, device=dev)
    g = grid.c_struct()
    ctx, st = _lib.ctx(), _lib.stream()
    entries, outside = C.c_int64(0), C.c_int64(-1)
    _lib.call("ow_fill_bins_count", ctx, C.byref(g), _lib.ptr(geom.coords), n_faces, float(h), _lib.ptr(counts),
              C.byref(entries), C.byref(outside), st)
    if outside.value >= 0:
        raise InvalidParameterError(f"face sample outside binning domain (face {outside.value})")
    e = int(entries.value)
    if e > capacity:
        cnt = counts.cpu().numpy().astype(np.int64)
        acc = 0
        for b0, b1 in batches:  # first batch whose running total overflows (binning.py:246-254)
            acc += int(cnt[b0:b1].sum())
            if acc > capacity:
                break
        raise CapacityError(
            f"bin assignment overflow: {acc} face-bin entries exceed capacity {capacity} "
            f"(= {overlap_factor} x {n_faces} faces); raise overlap_factor, or raise bin_fraction "
            f"to shrink the per-batch indicator")
    ids = torch.empty(e, dtype=torch.int32, device=dev)
    offsets = torch.empty(grid.n_bins, dtype=torch.int32, device=dev)
    _lib.call("ow_fill_bins_emit", ctx, C.byref(g), _lib.ptr(ids), _lib.ptr(counts), _lib.ptr(offsets), st)
    return BinnedFaces(grid.n_bins, ids, counts, offsets)
