"""Near-face predicates (device) and the FP64 exact-distance referee (host).

``near_faces_mask`` / ``near_triangle_mask`` / ``near_edge_mask`` and the
scalar ``check_near_*`` evaluate the sm_100a predicate of the marking kernel
(csrc/ow_predicate.cuh) pairwise through ``ow_near_pairs`` — the same float32
operation sequence as octowall/distance.py:38-245, so results are bitwise
equal to the reference.  The referee functions are independent FP64
closest-point computations (distance.py:260-371) used only for validation,
never on the hot path.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .errors import InvalidParameterError

BOUNDARY_BAND = 1e-4
_DEGEN_REL = 1e-12


def near_pairs(points, faces, d):
    """Pairwise predicate: points (n, D), faces (D, D, n), d scalar or (n,) -> bool (n,) CUDA."""
    dev = _lib.device()
    p = torch.as_tensor(np.asarray(points, np.float32) if not isinstance(points, torch.Tensor) else points,
                        dtype=torch.float32, device=dev).contiguous()
    f = torch.as_tensor(np.asarray(faces, np.float32) if not isinstance(faces, torch.Tensor) else faces,
                        dtype=torch.float32, device=dev).contiguous()
    n = p.shape[0]
    dim = p.shape[1]
    if f.shape != (dim, dim, n):
        raise InvalidParameterError(f"faces must be ({dim}, {dim}, {n}), got {tuple(f.shape)}")
    dd = torch.as_tensor(np.broadcast_to(np.asarray(d, np.float32), (n,)).copy(), device=dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    _lib.call("ow_near_pairs", _lib.ctx(), dim, _lib.ptr(p), _lib.ptr(f), _lib.ptr(dd), n, _lib.ptr(out),
              _lib.stream())
    return out.bool()


def near_triangle_mask(px, py, pz, tri, d_spec):
    """Broadcasting batch predicate (distance.py:167-213), evaluated on the GPU."""
    tri = np.asarray(tri, np.float32)
    shape = np.broadcast_shapes(np.shape(px), np.shape(py), np.shape(pz), tri.shape[2:], np.shape(d_spec))
    P = np.stack([np.broadcast_to(np.asarray(v, np.float32), shape).reshape(-1) for v in (px, py, pz)], 1)
    T = np.broadcast_to(tri, (3, 3) + shape).reshape(3, 3, -1)
    D = np.broadcast_to(np.asarray(d_spec, np.float32), shape).reshape(-1)
    return near_pairs(P, np.ascontiguousarray(T), D).cpu().numpy().reshape(shape)


def near_edge_mask(px, py, edges, d_spec):
    edges = np.asarray(edges, np.float32)
    shape = np.broadcast_shapes(np.shape(px), np.shape(py), edges.shape[2:], np.shape(d_spec))
    P = np.stack([np.broadcast_to(np.asarray(v, np.float32), shape).reshape(-1) for v in (px, py)], 1)
    E = np.broadcast_to(edges, (2, 2) + shape).reshape(2, 2, -1)
    D = np.broadcast_to(np.asarray(d_spec, np.float32), shape).reshape(-1)
    return near_pairs(P, np.ascontiguousarray(E), D).cpu().numpy().reshape(shape)


def near_faces_mask(px, py, pz, coords, d_spec):
    if np.shape(coords)[0] == 2:
        return near_edge_mask(px, py, coords, d_spec)
    return near_triangle_mask(px, py, pz, coords, d_spec)


def _degenerate(a, b, c):
    u = np.asarray(b, np.float64) - np.asarray(a, np.float64)
    v = np.asarray(c, np.float64) - np.asarray(a, np.float64)
    w = np.asarray(c, np.float64) - np.asarray(b, np.float64)
    scale = max(u @ u, v @ v, w @ w)
    cr = np.cross(u, v)
    return scale == 0.0 or math.sqrt(cr @ cr) < _DEGEN_REL * scale


def check_near_triangle(x_p, v1, v2, v3, d_spec):
    if d_spec <= 0:
        raise InvalidParameterError(f"near-wall distance must be positive, got {d_spec}")
    v = [np.asarray(x, np.float32).reshape(3) for x in (v1, v2, v3)]
    if _degenerate(*v):
        raise InvalidParameterError("degenerate triangle (zero area within working precision)")
    tri = np.stack(v)[:, :, None]
    p = np.asarray(x_p, np.float32).reshape(1, 3)
    return bool(near_pairs(p, tri, d_spec).cpu()[0])


def check_near_edge(x_p, v1, v2, d_spec):
    if d_spec <= 0:
        raise InvalidParameterError(f"near-wall distance must be positive, got {d_spec}")
    a, b = np.asarray(v1, np.float32).reshape(2), np.asarray(v2, np.float32).reshape(2)
    if np.array_equal(a, b):
        raise InvalidParameterError("degenerate edge: identical endpoints")
    p = np.asarray(x_p, np.float32).reshape(1, 2)
    return bool(near_pairs(p, np.stack([a, b])[:, :, None], d_spec).cpu()[0])


# ---------------------------------------------------------------------------
# FP64 referee (validation only)
# ---------------------------------------------------------------------------


def point_segment_distance_sq(x_p, a, b):
    p, a, b = (np.asarray(x, np.float64).reshape(-1) for x in (x_p, a, b))
    e = b - a
    el2 = float(e @ e)
    if el2 == 0.0:
        raise InvalidParameterError("degenerate segment: identical endpoints")
    t = min(1.0, max(0.0, float((p - a) @ e) / el2))
    q = p - (a + t * e)
    return float(q @ q)


def exact_point_triangle_distance(x_p, v1, v2, v3):
    """Closest-point distance by Voronoi region of the barycentric signs."""
    p, a, b, c = (np.asarray(x, np.float64).reshape(3) for x in (x_p, v1, v2, v3))
    if _degenerate(a, b, c):
        raise InvalidParameterError("degenerate triangle (zero area within working precision)")
    ab, ac, ap = b - a, c - a, p - a
    d1, d2 = ab @ ap, ac @ ap
    if d1 <= 0 and d2 <= 0:
        return float(np.linalg.norm(ap))
    bp = p - b
    d3, d4 = ab @ bp, ac @ bp
    if d3 >= 0 and d4 <= d3:
        return float(np.linalg.norm(bp))
    vc = d1 * d4 - d3 * d2
    if vc <= 0 and d1 >= 0 and d3 <= 0:
        return float(np.linalg.norm(ap - (d1 / (d1 - d3)) * ab))
    cp = p - c
    d5, d6 = ab @ cp, ac @ cp
    if d6 >= 0 and d5 <= d6:
        return float(np.linalg.norm(cp))
    vb = d5 * d2 - d1 * d6
    if vb <= 0 and d2 >= 0 and d6 <= 0:
        return float(np.linalg.norm(ap - (d2 / (d2 - d6)) * ac))
    va = d3 * d6 - d5 * d4
    if va <= 0 and (d4 - d3) >= 0 and (d5 - d6) >= 0:
        w = (d4 - d3) / ((d4 - d3) + (d5 - d6))
        return float(np.linalg.norm(bp - w * (c - b)))
    den = 1.0 / (va + vb + vc)
    return float(np.linalg.norm(ap - (vb * den * ab + vc * den * ac)))


def min_distance_sq_to_edges(points, coords):
    p = np.asarray(points, np.float64)
    c = np.asarray(coords.cpu() if isinstance(coords, torch.Tensor) else coords)
    a, b = c[0].astype(np.float64).T, c[1].astype(np.float64).T
    e = b - a
    el2 = np.einsum("fd,fd->f", e, e)
    if np.any(el2 == 0.0):
        raise InvalidParameterError("degenerate segment: identical endpoints")
    best = np.full(len(p), np.inf)
    chunk = max(1, int(4e6 // max(1, len(a))))
    for s in range(0, len(p), chunk):
        ap = p[s:s + chunk, None, :] - a[None]
        t = np.clip(np.einsum("cfd,fd->cf", ap, e) / el2, 0.0, 1.0)
        diff = ap - t[:, :, None] * e[None]
        best[s:s + chunk] = np.einsum("cfd,cfd->cf", diff, diff).min(axis=1)
    return best


def boundary_band(d_spec, coords_scale):
    return BOUNDARY_BAND * max(1.0, float(coords_scale))
