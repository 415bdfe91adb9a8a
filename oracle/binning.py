"""Oracle: face -> bin assignment (test infrastructure only).

Restates octowall/binning.py:
  BinGrid single-precision constants    binning.py:34-60
  linear bin index (floor, clamp)       binning.py:63-85
  default spacing (half min bin edge)   binning.py:101-103
  segment / triangle discretisation     binning.py:106-137, 294-311
  fill_bins membership + CSR + capacity binning.py:200-266, 314-346
  batch ranges (capacity message)       binning.py:183-197

Membership is sample based: face f is in bin b iff one of f's float32
discretisation samples lands in b.  The dense per-batch indicator of the
reference is replaced by an equivalent sort-unique over (bin, face) keys,
which yields the same ascending-per-bin CSR (checked against goldens).
"""

from __future__ import annotations

import math

import numpy as np

from .errors import Capacity, InvalidParameter

F32 = np.float32
DOMAIN_REL_TOL = 1e-6
SLOT_BUDGET = 2 ** 25


class Grid:
    def __init__(self, dmin, dmax, bins_per_axis):
        self.dmin = np.asarray(dmin, np.float64)
        self.dmax = np.asarray(dmax, np.float64)
        self.B = int(bins_per_axis)
        if self.B < 1:
            raise InvalidParameter("bins_per_axis must be >= 1")
        self.extent = self.dmax - self.dmin
        self.min32 = self.dmin.astype(F32)
        self.len32 = (self.extent / self.B).astype(F32)
        self.dim = len(self.dmin)
        self.n_bins = self.B ** self.dim

    def default_spacing(self):
        return float(F32(0.5) * self.len32.min())

    def bin_of(self, pts, what="point"):
        """pts (..., D) float32 -> linear bin (x fastest), int64."""
        p = np.asarray(pts, F32)
        tol = DOMAIN_REL_TOL * self.extent
        bad = np.any((p < self.dmin - tol) | (p > self.dmax + tol), axis=-1)
        if np.any(bad):
            raise InvalidParameter(f"{what} outside binning domain")
        ix = np.floor((p - self.min32) / self.len32).astype(np.int64)
        np.clip(ix, 0, self.B - 1, out=ix)
        lin = ix[..., self.dim - 1].copy()
        for ax in range(self.dim - 2, -1, -1):
            lin = lin * self.B + ix[..., ax]
        return lin


def segment_samples(a, b, h):
    """Segments a->b ((D, n) float32 each): returns (segment index, points (m, D)).

    n_k = ceil(|b-a| / h); points a + (i / max(n_k,1)) * (b - a), i = 0..n_k.
    """
    d = b - a
    sq = d[0] * d[0]
    for ax in range(1, d.shape[0]):
        sq = sq + d[ax] * d[ax]
    nseg = np.ceil(np.sqrt(sq) / h).astype(np.int64)
    npts = nseg + 1
    seg = np.repeat(np.arange(d.shape[1]), npts)
    first = np.cumsum(npts) - npts
    i = (np.arange(seg.size, dtype=np.int64) - first[seg]).astype(F32)
    t = i / np.maximum(nseg, 1).astype(F32)[seg]
    pts = a[:, seg] + t * d[:, seg]
    return seg, pts.T


def face_samples(coords, h):
    """All discretisation samples: (face index, points (m, D))."""
    c = np.asarray(coords, F32)
    h = F32(h)
    if c.shape[0] == 2:
        return segment_samples(c[0], c[1], h)
    base_face, base = segment_samples(c[0], c[1], h)
    sub, pts = segment_samples(np.ascontiguousarray(base.T), c[2][:, base_face], h)
    return base_face[sub], pts


def batch_ranges(n_bins, bin_fraction):
    if bin_fraction < 1:
        raise InvalidParameter("bin_fraction must be >= 1")
    per = math.ceil(n_bins / min(bin_fraction, n_bins))
    return [(s, min(s + per, n_bins)) for s in range(0, n_bins, per)]


def auto_bin_fraction(n_bins, n_faces):
    return 1 if n_faces == 0 else max(1, math.ceil(n_bins * max(1, n_faces) / SLOT_BUDGET))


def fill_bins(coords, grid: Grid, spacing=None, overlap_factor=10, bin_fraction=None):
    """-> (ids int32[E], counts int32[n_bins], offsets int32[n_bins])."""
    from .geometry import bbox, first_degenerate

    c = np.asarray(coords, F32)
    nf = c.shape[2]
    if nf == 0:
        raise InvalidParameter("cannot bin empty geometry")
    bad = first_degenerate(c)
    if bad >= 0:
        raise InvalidParameter(f"degenerate face at {bad}")
    lo, hi = bbox(c)
    tol = DOMAIN_REL_TOL * grid.extent
    if np.any(lo < grid.dmin - tol) or np.any(hi > grid.dmax + tol):
        raise InvalidParameter("face outside binning domain")
    if bin_fraction is None:
        bin_fraction = auto_bin_fraction(grid.n_bins, nf)
    h = F32(spacing) if spacing is not None else F32(grid.default_spacing())
    if h <= 0:
        raise InvalidParameter("spacing must be positive")
    face, pts = face_samples(c, h)
    b = grid.bin_of(pts, what="face sample")
    key = np.unique(b * nf + face)
    bins, faces = key // nf, key % nf
    counts = np.bincount(bins, minlength=grid.n_bins).astype(np.int32)
    cap = overlap_factor * nf
    if key.size > cap:
        acc = 0
        for b0, b1 in batch_ranges(grid.n_bins, bin_fraction):
            acc += int(counts[b0:b1].sum())
            if acc > cap:
                break
        raise Capacity(f"bin assignment overflow: {acc} face-bin entries exceed capacity {cap}")
    offsets = np.zeros(grid.n_bins, np.int32)
    np.cumsum(counts[:-1], out=offsets[1:])
    return faces.astype(np.int32), counts, offsets
