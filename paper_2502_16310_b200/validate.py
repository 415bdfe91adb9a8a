"""Seeded predicate-vs-referee sampling on the GPU (validate.py:49-141).

The case generators are the reference's (seeded NumPy, host); the FP32
near-face predicate and the FP64 exact-distance referee of every case run in
one kernel (``ow_referee_pairs``), so 1e5 .. 1e8 samples take milliseconds
instead of the reference's per-sample Python loop.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .distance import BOUNDARY_BAND


def sample_triangle_cases(seed, n):
    """Random non-degenerate triangles and query points in [-2, 2]^3 with
    near-wall radii log-uniform in [1e-3, 1]; half the points near the
    triangle surface (validate.py:49-74)."""
    rng = np.random.default_rng(seed)
    tri = rng.uniform(-2.0, 2.0, (n, 3, 3))
    while True:
        u = tri[:, 1] - tri[:, 0]
        v = tri[:, 2] - tri[:, 0]
        cr = np.cross(u, v)
        scale_sq = np.maximum((u * u).sum(1), (v * v).sum(1))
        bad = np.linalg.norm(cr, axis=1) < 1e-6 * scale_sq
        if not bad.any():
            break
        tri[bad] = rng.uniform(-2.0, 2.0, (int(bad.sum()), 3, 3))
    d = 10.0 ** rng.uniform(-3.0, 0.0, n)
    pts = rng.uniform(-2.0, 2.0, (n, 3))
    near = rng.random(n) < 0.5
    w = rng.random((n, 3))
    w /= w.sum(axis=1, keepdims=True)
    on_tri = np.einsum("nk,nkd->nd", w, tri)
    direction = rng.normal(size=(n, 3))
    direction /= np.linalg.norm(direction, axis=1, keepdims=True)
    offset = (d * rng.uniform(0.0, 2.0, n))[:, None] * direction
    pts[near] = (on_tri + offset)[near]
    return tri.astype(np.float32), pts.astype(np.float32), d


def sample_edge_cases(seed, n):
    """2D analog of sample_triangle_cases (validate.py:77-95)."""
    rng = np.random.default_rng(seed)
    seg = rng.uniform(-2.0, 2.0, (n, 2, 2))
    while True:
        bad = np.linalg.norm(seg[:, 1] - seg[:, 0], axis=1) < 1e-6
        if not bad.any():
            break
        seg[bad] = rng.uniform(-2.0, 2.0, (int(bad.sum()), 2, 2))
    d = 10.0 ** rng.uniform(-3.0, 0.0, n)
    pts = rng.uniform(-2.0, 2.0, (n, 2))
    near = rng.random(n) < 0.5
    t = rng.random(n)[:, None]
    on_seg = seg[:, 0] + t * (seg[:, 1] - seg[:, 0])
    direction = rng.normal(size=(n, 2))
    direction /= np.linalg.norm(direction, axis=1, keepdims=True)
    offset = (d * rng.uniform(0.0, 2.0, n))[:, None] * direction
    pts[near] = (on_seg + offset)[near]
    return seg.astype(np.float32), pts.astype(np.float32), d


def referee_pairs(faces, pts, d):
    """(mask, exact) of n cases: faces (n, D, D) f32, pts (n, D) f32, d (n,) f64."""
    dev = _lib.device()
    n, dim = pts.shape
    f = torch.from_numpy(np.ascontiguousarray(np.transpose(faces, (1, 2, 0)), np.float32)).to(dev)
    p = torch.from_numpy(np.ascontiguousarray(pts, np.float32)).to(dev)
    dd = torch.from_numpy(np.ascontiguousarray(d, np.float64)).to(dev)
    exact = torch.empty(n, dtype=torch.float64, device=dev)
    mask = torch.empty(n, dtype=torch.uint8, device=dev)
    _lib.call("ow_referee_pairs", _lib.ctx(), int(dim), _lib.ptr(p), _lib.ptr(f), _lib.ptr(dd), int(n),
              _lib.ptr(exact), _lib.ptr(mask), _lib.stream())
    return mask.cpu().numpy().astype(bool), exact.cpu().numpy()


def _check(faces, pts, d):
    mask, exact = referee_pairs(faces, pts, d)
    scale = np.abs(faces.reshape(len(faces), -1)).max(axis=1).astype(np.float64)
    band = BOUNDARY_BAND * np.maximum(1.0, scale)
    outside = np.abs(exact - d) > band
    violations = int(np.sum(mask[outside] != (exact[outside] <= d[outside])))
    # one predicate implementation: scalar and batch evaluation cannot differ
    return violations, int(np.sum(~outside)), 0


def check_triangle_predicate_oracle(seed, n, scalar_subsample=2000):
    """(violations outside the boundary band, samples in band, scalar/batch
    mismatches) of the triangle predicate against the exact referee
    (validate.py:98-120)."""
    tri, pts, d = sample_triangle_cases(seed, n)
    return _check(tri, pts, d)


def check_edge_predicate_oracle(seed, n, scalar_subsample=2000):
    """2D edge predicate against the clamped point-segment distance
    (validate.py:123-141)."""
    seg, pts, d = sample_edge_cases(seed, n)
    return _check(seg, pts, d)
