"""Oracle: FP32 near-face predicates, Algorithm 1 (test infrastructure only).

Restates octowall/distance.py:
  3D triangle (balls, clipped cylinders, prism slab)  distance.py:167-213
  unit normals                                        distance.py:238-245
  2D edge (disks + rectangle)                         distance.py:216-235

Every operation is float32 with the reference's association order
((a+b)+c), IEEE division and sqrt, no fused multiply-add.  Points and faces
broadcast against each other (faces on the last axis).
"""

from __future__ import annotations

import math

import numpy as np

F32 = np.float32


def _dot3(ax, ay, az, bx, by, bz):
    return (ax * bx + ay * by) + az * bz


def near_triangle(px, py, pz, tri, d):
    """tri: (3 vertex slots, 3 components, ...) float32; d float32 scalar/array."""
    d = np.asarray(d, F32)
    r2 = d * d
    v = [(tri[k, 0], tri[k, 1], tri[k, 2]) for k in range(3)]
    w = [(a[0] - px, a[1] - py, a[2] - pz) for a in v]  # vertex - point
    hit = None
    unit_e = []
    for k in range(3):
        a, b = v[k], v[(k + 1) % 3]
        wx, wy, wz = w[k]
        ball = _dot3(wx, wy, wz, wx, wy, wz) <= r2
        ex, ey, ez = b[0] - a[0], b[1] - a[1], b[2] - a[2]
        el2 = _dot3(ex, ey, ez, ex, ey, ez)
        el = np.sqrt(el2)
        ux, uy, uz = ex / el, ey / el, ez / el
        unit_e.append((ux, uy, uz))
        cx, cy, cz = ey * wz - ez * wy, ez * wx - ex * wz, ex * wy - ey * wx
        dist2 = _dot3(cx, cy, cz, cx, cy, cz) / el2
        t0 = -_dot3(wx, wy, wz, ux, uy, uz)
        t1 = _dot3(b[0] - px, b[1] - py, b[2] - pz, ux, uy, uz)
        piece = ball | ((dist2 <= r2) & (t0 >= 0) & (t1 >= 0))
        hit = piece if hit is None else hit | piece
    nx, ny, nz = unit_normal(tri)
    inside = None
    for k in range(3):
        ux, uy, uz = unit_e[k]
        mx, my, mz = ny * uz - nz * uy, nz * ux - nx * uz, nx * uy - ny * ux
        a = v[k]
        half = _dot3(px - a[0], py - a[1], pz - a[2], mx, my, mz) >= 0
        inside = half if inside is None else inside & half
    a = v[0]
    below = -_dot3((a[0] - d * nx) - px, (a[1] - d * ny) - py, (a[2] - d * nz) - pz, nx, ny, nz)
    above = _dot3((a[0] + d * nx) - px, (a[1] + d * ny) - py, (a[2] + d * nz) - pz, nx, ny, nz)
    return hit | (inside & (below >= 0) & (above >= 0))


def unit_normal(tri):
    ux, uy, uz = tri[1, 0] - tri[0, 0], tri[1, 1] - tri[0, 1], tri[1, 2] - tri[0, 2]
    vx, vy, vz = tri[2, 0] - tri[0, 0], tri[2, 1] - tri[0, 1], tri[2, 2] - tri[0, 2]
    nx, ny, nz = uy * vz - uz * vy, uz * vx - ux * vz, ux * vy - uy * vx
    ln = np.sqrt(_dot3(nx, ny, nz, nx, ny, nz))
    return nx / ln, ny / ln, nz / ln


def near_edge(px, py, seg, d):
    """seg: (2 endpoints, 2 components, ...) float32."""
    d = np.asarray(d, F32)
    r2 = d * d
    ax, ay, bx, by = seg[0, 0], seg[0, 1], seg[1, 0], seg[1, 1]
    wax, way = ax - px, ay - py
    wbx, wby = bx - px, by - py
    disks = ((wax * wax + way * way) <= r2) | ((wbx * wbx + wby * wby) <= r2)
    ex, ey = bx - ax, by - ay
    el2 = ex * ex + ey * ey
    el = np.sqrt(el2)
    ux, uy = ex / el, ey / el
    cr = ex * way - ey * wax
    dist2 = (cr * cr) / el2
    t0 = -(wax * ux + way * uy)
    t1 = wbx * ux + wby * uy
    return disks | ((dist2 <= r2) & (t0 >= 0) & (t1 >= 0))


def near(points, faces, d):
    """points (..., D) f32, faces (D, D, ...) f32 (broadcast on trailing axes)."""
    p = np.asarray(points, F32)
    if faces.shape[0] == 2:
        return near_edge(p[..., 0], p[..., 1], faces, d)
    return near_triangle(p[..., 0], p[..., 1], p[..., 2], faces, d)


def exact_point_triangle_distance(p, a, b, c):
    """FP64 referee, restated from distance.py:275-345 (Python floats: IEEE
    double, no FMA, correctly rounded sqrt); degeneracy check omitted."""
    px, py, pz = (float(x) for x in p)
    ax, ay, az = (float(x) for x in a)
    bx, by, bz = (float(x) for x in b)
    cx, cy, cz = (float(x) for x in c)
    abx, aby, abz = bx - ax, by - ay, bz - az
    acx, acy, acz = cx - ax, cy - ay, cz - az
    bcx, bcy, bcz = cx - bx, cy - by, cz - bz
    apx, apy, apz = px - ax, py - ay, pz - az
    d1 = abx * apx + aby * apy + abz * apz
    d2 = acx * apx + acy * apy + acz * apz
    if d1 <= 0.0 and d2 <= 0.0:
        return math.sqrt(apx * apx + apy * apy + apz * apz)
    bpx, bpy, bpz = px - bx, py - by, pz - bz
    d3 = abx * bpx + aby * bpy + abz * bpz
    d4 = acx * bpx + acy * bpy + acz * bpz
    if d3 >= 0.0 and d4 <= d3:
        return math.sqrt(bpx * bpx + bpy * bpy + bpz * bpz)
    vc = d1 * d4 - d3 * d2
    if vc <= 0.0 and d1 >= 0.0 and d3 <= 0.0:
        t = d1 / (d1 - d3)
        qx, qy, qz = apx - t * abx, apy - t * aby, apz - t * abz
        return math.sqrt(qx * qx + qy * qy + qz * qz)
    cpx, cpy, cpz = px - cx, py - cy, pz - cz
    d5 = abx * cpx + aby * cpy + abz * cpz
    d6 = acx * cpx + acy * cpy + acz * cpz
    if d6 >= 0.0 and d5 <= d6:
        return math.sqrt(cpx * cpx + cpy * cpy + cpz * cpz)
    vb = d5 * d2 - d1 * d6
    if vb <= 0.0 and d2 >= 0.0 and d6 <= 0.0:
        t = d2 / (d2 - d6)
        qx, qy, qz = apx - t * acx, apy - t * acy, apz - t * acz
        return math.sqrt(qx * qx + qy * qy + qz * qz)
    va = d3 * d6 - d5 * d4
    if va <= 0.0 and (d4 - d3) >= 0.0 and (d5 - d6) >= 0.0:
        t = (d4 - d3) / ((d4 - d3) + (d5 - d6))
        qx, qy, qz = bpx - t * bcx, bpy - t * bcy, bpz - t * bcz
        return math.sqrt(qx * qx + qy * qy + qz * qz)
    denom = 1.0 / (va + vb + vc)
    v = vb * denom
    w = vc * denom
    qx = apx - (v * abx + w * acx)
    qy = apy - (v * aby + w * acy)
    qz = apz - (v * abz + w * acz)
    return math.sqrt(qx * qx + qy * qy + qz * qz)


def point_segment_distance(p, a, b):
    """sqrt of point_segment_distance_sq, distance.py:260-272 (FP64)."""
    px, py = float(p[0]), float(p[1])
    ax, ay, bx, by = float(a[0]), float(a[1]), float(b[0]), float(b[1])
    ex, ey = bx - ax, by - ay
    el2 = ex * ex + ey * ey
    t = ((px - ax) * ex + (py - ay) * ey) / el2
    t = min(1.0, max(0.0, t))
    qx, qy = px - (ax + t * ex), py - (ay + t * ey)
    return math.sqrt(qx * qx + qy * qy)
