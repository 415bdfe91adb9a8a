"""Deterministic synthetic geometries for the benchmark configurations.

The reference ships no mesh files (no bunny STL under /root/reference), so the
configurations of SURVEY.md §8(d) are generated procedurally, in float64,
rounded once to float32, and serialised as binary STL (50-byte records) so the
import stage of the hot path is exercised exactly as with a user file.

    C1  text primitive  ``circle 0.5 0.5 0.25 12800``
    C2  icosphere, 5 midpoint subdivisions (20,480 triangles), r=0.3
    C3  bumpy lat-lon sphere (187 x 188 -> 69,936 triangles)
    C4  (2,3) torus-knot tube, 4000 x 125 quads (1,000,000 triangles)
    C5  icosphere, 9 subdivisions (5,242,880 triangles)
"""

from __future__ import annotations

import struct

import numpy as np

__all__ = [
    "icosphere_triangles",
    "bumpy_sphere_triangles",
    "torus_knot_triangles",
    "binary_stl_bytes",
    "write_binary_stl",
    "circle_text",
]


def _icosahedron():
    t = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array(
        [
            [-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
            [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
            [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1],
        ],
        dtype=np.float64,
    )
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array(
        [
            [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
            [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
            [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
            [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1],
        ],
        dtype=np.int64,
    )
    return v[f]  # (20, 3, 3) unit-sphere triangles, outward winding


def icosphere_triangles(subdivisions=5, center=(0.5, 0.5, 0.5), radius=0.3):
    """Triangle soup (F, 3, 3) float64 of a midpoint-subdivided icosahedron.

    Each triangle (a, b, c) becomes (a, ab, ca), (ab, b, bc), (ca, bc, c),
    (ab, bc, ca) with midpoints pushed back onto the unit sphere; F = 20*4^s.
    """
    tri = _icosahedron()
    for _ in range(int(subdivisions)):
        a, b, c = tri[:, 0], tri[:, 1], tri[:, 2]

        def mid(p, q):
            m = 0.5 * (p + q)
            return m / np.linalg.norm(m, axis=1, keepdims=True)

        ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
        tri = np.stack(
            [
                np.stack([a, ab, ca], 1),
                np.stack([ab, b, bc], 1),
                np.stack([ca, bc, c], 1),
                np.stack([ab, bc, ca], 1),
            ],
            axis=1,
        ).reshape(-1, 3, 3)
    return np.asarray(center, np.float64) + float(radius) * tri


def bumpy_sphere_triangles(n_lat=187, n_lon=188, center=(0.5, 0.5, 0.5), radius=0.3):
    """Bunny-scale closed surface: lat-lon sphere with an FP64 radial bump
    r = R (1 + 0.12 sin(3 theta) cos(2 phi) + 0.05 sin(5 phi)).
    Triangles: 2*n_lon (pole fans) + 2*(n_lat-2)*n_lon."""
    theta = np.pi * np.arange(1, n_lat) / n_lat
    phi = 2.0 * np.pi * np.arange(n_lon) / n_lon
    th, ph = np.meshgrid(theta, phi, indexing="ij")
    r = radius * (1.0 + 0.12 * np.sin(3 * th) * np.cos(2 * ph) + 0.05 * np.sin(5 * ph))
    ring = np.stack([r * np.sin(th) * np.cos(ph), r * np.sin(th) * np.sin(ph), r * np.cos(th)], -1)
    c = np.asarray(center, np.float64)
    ring = ring + c
    north = c + np.array([0.0, 0.0, radius])
    south = c - np.array([0.0, 0.0, radius])
    j = np.arange(n_lon)
    jn = (j + 1) % n_lon
    tris = [np.stack([np.broadcast_to(north, (n_lon, 3)), ring[0, j], ring[0, jn]], 1)]
    a, b = ring[:-1], ring[1:]
    t1 = np.stack([a[:, j], b[:, j], b[:, jn]], 2).reshape(-1, 3, 3)
    t2 = np.stack([a[:, j], b[:, jn], a[:, jn]], 2).reshape(-1, 3, 3)
    quads = np.stack([t1.reshape(n_lat - 2, n_lon, 3, 3), t2.reshape(n_lat - 2, n_lon, 3, 3)], 2)
    tris.append(quads.reshape(-1, 3, 3))
    tris.append(np.stack([np.broadcast_to(south, (n_lon, 3)), ring[-1, jn], ring[-1, j]], 1))
    return np.concatenate(tris, 0)


def torus_knot_triangles(n_u=4000, n_v=125, p=2, q=3, tube=0.035, lo=0.1, hi=0.9):
    """(p,q) torus-knot tube, 2*n_u*n_v triangles, fitted into [lo, hi]^3."""
    u = 2.0 * np.pi * np.arange(n_u) / n_u
    v = 2.0 * np.pi * np.arange(n_v) / n_v

    def curve(s):
        rr = 2.0 + np.cos(q * s)
        return np.stack([rr * np.cos(p * s), rr * np.sin(p * s), -np.sin(q * s)], -1)

    c = curve(u)
    dc = curve(u + 1e-4) - curve(u - 1e-4)
    tng = dc / np.linalg.norm(dc, axis=1, keepdims=True)
    ref = np.array([0.0, 0.0, 1.0])
    nrm = np.cross(tng, ref)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    bin_ = np.cross(tng, nrm)
    ring = (
        c[:, None, :]
        + (tube * 3.0) * (np.cos(v)[None, :, None] * nrm[:, None, :] + np.sin(v)[None, :, None] * bin_[:, None, :])
    )
    lo3, hi3 = ring.reshape(-1, 3).min(0), ring.reshape(-1, 3).max(0)
    scale = (hi - lo) / float((hi3 - lo3).max())
    ring = lo + (ring - lo3) * scale
    i = np.arange(n_u)
    inx = (i + 1) % n_u
    j = np.arange(n_v)
    jn = (j + 1) % n_v
    a = ring[i][:, j]
    b = ring[inx][:, j]
    c2 = ring[inx][:, jn]
    d = ring[i][:, jn]
    t1 = np.stack([a, b, c2], 2)
    t2 = np.stack([a, c2, d], 2)
    return np.stack([t1, t2], 2).reshape(-1, 3, 3)


def binary_stl_bytes(tris, header=b"octowall-b200 synthetic"):
    """Serialise (F, 3, 3) triangles into binary STL bytes (float32, LE)."""
    t = np.asarray(tris, dtype=np.float32).reshape(-1, 3, 3)
    n = len(t)
    rec = np.zeros((n, 50), dtype=np.uint8)
    e1 = t[:, 1].astype(np.float64) - t[:, 0]
    e2 = t[:, 2].astype(np.float64) - t[:, 0]
    nn = np.cross(e1, e2)
    ln = np.linalg.norm(nn, axis=1, keepdims=True)
    nn = np.where(ln > 0, nn / np.where(ln > 0, ln, 1.0), 0.0).astype(np.float32)
    fl = np.concatenate([nn[:, None, :], t], axis=1).reshape(n, 12).astype("<f4")
    rec[:, :48] = fl.view(np.uint8).reshape(n, 48)
    return header.ljust(80, b"\0")[:80] + struct.pack("<I", n) + rec.tobytes()


def write_binary_stl(path, tris, header=b"octowall-b200 synthetic"):
    data = binary_stl_bytes(tris, header)
    with open(path, "wb") as f:
        f.write(data)
    return len(data)


def circle_text(cx=0.5, cy=0.5, r=0.25, n=12800):
    return f"circle {cx} {cy} {r} {n}\n"
