"""Oracle: lattice boundary links and wall fractions q (test infrastructure).

NORTH-STAR EXTENSION — the reference has no lattice links, Moller-Trumbore
or q (SURVEY.md finding 6), so this oracle is "parity unpinned by the
reference": it is pinned only by analytic known-answer tests
(tests/test_oracle_lattice.py).  Cell selection and conventions follow the
reference where it has them: finest-level leaves in ascending block id and
x-fastest cell index (nearwall.py:537-553), FP32 arithmetic with a fixed
operation order (distance.py:9-14).

Definition ("Lattice links"):
  * link i of a cell with centre x (float32) and finest cell size h (per
    axis, float32 of the FP64 value) is the segment x -> x + c_i*h;
  * candidate faces: every face whose float32 AABB overlaps the link's
    float32 AABB [min(x, x+c_i*h), max(x, x+c_i*h)] (closed intervals);
  * the segment-face test is WATERTIGHT (Woop, Benthin & Wald, "Watertight
    Ray/Triangle Intersection", JCGT 2(1), 2013, restated for segments):
    per direction a fixed frame (kz = first axis of max |dv|, kx, ky the
    next two cyclically, swapped when dv[kz] < 0; shear Sx = dv[kx]/dv[kz],
    Sy = dv[ky]/dv[kz], Sz = 1/dv[kz] in float32), vertices translated to
    the link origin and sheared (A = v - x; Ax = A[kx] - Sx A[kz], ...),
    edge functions U = Cx By - Cy Bx, V = Ax Cy - Ay Cx, W = Bx Ay - By Ax
    (float32; recomputed in float64 from the same sheared float32 values
    when any of them is zero), miss when they have mixed signs or when
    det = (U + V) + W is zero; T = (U Az + V Bz) + W Cz with Az = Sz A[kz]
    ...; t = T / det; hit iff 0 <= t <= 1.  An edge function depends only on
    the edge's two (translated, sheared) vertices, so faces that share an
    edge or a vertex evaluate it identically (up to sign): a link crossing a
    closed surface cannot slip between two faces (tests/test_oracle_lattice.py
    checks it on a closed icosphere against an exact FP64 inside/outside
    referee).  2D is the same with one transverse axis: the edge's endpoints
    have transverse coordinates Ax, Bx; U = Bx, V = -Ax (no products);
  * q_i = min t over hits (float32), -1 when link i hits nothing;
  * flags bit i set iff link i hits.
Opposite directions d, -d share the frame up to exact negations (the swap
exchanges the edge functions' sign, Sz changes sign), so t(-d) = -t(d)
bitwise; the CUDA kernel tests each lattice line once for both directions.
"""

from __future__ import annotations

import numpy as np

F32 = np.float32

D2Q9 = [(0, 0), (1, 0), (0, 1), (-1, 0), (0, -1), (1, 1), (-1, 1), (-1, -1), (1, -1)]


def _d3q19():
    dirs = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    for a, b in ((0, 1), (0, 2), (1, 2)):
        for sa, sb in ((1, 1), (-1, -1), (1, -1), (-1, 1)):
            v = [0, 0, 0]
            v[a], v[b] = sa, sb
            dirs.append(tuple(v))
    return dirs


D3Q19 = _d3q19()
D3Q27 = D3Q19 + [
    (1 - 2 * ((k >> 2) & 1), 1 - 2 * ((k >> 1) & 1), 1 - 2 * (k & 1)) for k in range(8)
]
LATTICES = {"D2Q9": D2Q9, "D3Q19": D3Q19, "D3Q27": D3Q27}


def directions(name):
    return np.asarray(LATTICES[name], np.int64)


def ray_frame(dv):
    """(kz, kx, ky, Sx, Sy, Sz) of a direction vector dv (float32, nonzero)."""
    dv = np.asarray(dv, F32)
    dim = dv.size
    a = np.abs(dv)
    kz = int(np.flatnonzero(a == a.max())[0])  # first axis of max |dv|
    if dim == 2:
        kx = 1 - kz
        return kz, kx, None, F32(dv[kx] / dv[kz]), None, F32(F32(1.0) / dv[kz])
    kx, ky = (kz + 1) % 3, (kz + 2) % 3
    if dv[kz] < 0:
        kx, ky = ky, kx
    return kz, kx, ky, F32(dv[kx] / dv[kz]), F32(dv[ky] / dv[kz]), F32(F32(1.0) / dv[kz])


def wt_hits(x, dv, tri):
    """Watertight segment-triangle test of pairs. x (n, 3) f32 origins, dv (3,)
    f32 direction shared by the pairs, tri (3, 3, n) f32 [vertex, axis, pair].

    Returns (hit bool (n,), t f32 (n,))."""
    kz, kx, ky, sx, sy, sz = ray_frame(dv)
    x = np.asarray(x, F32)
    P = []
    for j in range(3):  # translated, sheared vertices (float32, fixed order)
        a = [tri[j][k] - x[:, k] for k in range(3)]
        P.append((a[kx] - sx * a[kz], a[ky] - sy * a[kz], sz * a[kz]))
    (ax, ay, az), (bx, by, bz), (cx, cy, cz) = P
    u = cx * by - cy * bx
    v = ax * cy - ay * cx
    w = bx * ay - by * ax
    z = (u == 0) | (v == 0) | (w == 0)
    if z.any():  # exact signs: float products are exact in float64
        def d(a):
            return a[z].astype(np.float64)

        u[z] = (d(cx) * d(by) - d(cy) * d(bx)).astype(F32)
        v[z] = (d(ax) * d(cy) - d(ay) * d(cx)).astype(F32)
        w[z] = (d(bx) * d(ay) - d(by) * d(ax)).astype(F32)
    mixed = ((u < 0) | (v < 0) | (w < 0)) & ((u > 0) | (v > 0) | (w > 0))
    det = (u + v) + w
    T = (u * az + v * bz) + w * cz
    with np.errstate(divide="ignore", invalid="ignore"):
        t = T / det
    hit = ~mixed & (det != 0) & (t >= 0) & (t <= 1)
    return hit, t


def wt_hits2(x, dv, seg):
    """2D watertight segment-segment test of pairs. x (n, 2) f32, dv (2,) f32,
    seg (2, 2, n) f32 [endpoint, axis, pair]."""
    kz, kx, _, sx, _, sz = ray_frame(dv)
    x = np.asarray(x, F32)
    a = [seg[0][k] - x[:, k] for k in range(2)]
    b = [seg[1][k] - x[:, k] for k in range(2)]
    ax, az = a[kx] - sx * a[kz], sz * a[kz]
    bx, bz = b[kx] - sx * b[kz], sz * b[kz]
    u, v = bx, -ax
    mixed = ((u < 0) | (v < 0)) & ((u > 0) | (v > 0))
    det = u + v
    T = u * az + v * bz
    with np.errstate(divide="ignore", invalid="ignore"):
        t = T / det
    hit = ~mixed & (det != 0) & (t >= 0) & (t <= 1)
    return hit, t


def mt_hits(x, dvec, tri):
    """Round-1 definition (Moller-Trumbore, not watertight), kept only so the
    tests can count the links it loses at shared edges. x, dvec: (n, 3) f32."""
    v0, v1, v2 = tri[0], tri[1], tri[2]
    e1 = v1 - v0
    e2 = v2 - v0
    dx, dy, dz = dvec[:, 0], dvec[:, 1], dvec[:, 2]
    px = dy * e2[2] - dz * e2[1]
    py = dz * e2[0] - dx * e2[2]
    pz = dx * e2[1] - dy * e2[0]
    det = (e1[0] * px + e1[1] * py) + e1[2] * pz
    tx, ty, tz = x[:, 0] - v0[0], x[:, 1] - v0[1], x[:, 2] - v0[2]
    qx = ty * e1[2] - tz * e1[1]
    qy = tz * e1[0] - tx * e1[2]
    qz = tx * e1[1] - ty * e1[0]
    with np.errstate(divide="ignore", invalid="ignore"):
        u = ((tx * px + ty * py) + tz * pz) / det
        v = ((dx * qx + dy * qy) + dz * qz) / det
        t = ((e2[0] * qx + e2[1] * qy) + e2[2] * qz) / det
    with np.errstate(invalid="ignore"):
        hit = (det != 0) & (u >= 0) & (v >= 0) & ((u + v) <= 1) & (t >= 0) & (t <= 1)
    return hit, t


def link_hits(x, dv, faces):
    """The definition's test for one direction: 3D triangles or 2D segments."""
    return wt_hits(x, dv, faces) if faces.shape[0] == 3 else wt_hits2(x, dv, faces)


def lattice_links(forest, coords, lattice="D3Q19"):
    """-> dict(cells (n,) i64 flat index leafpos*4^D+cell, flags u32 (n_cells,),
    boundary (nb,) i64, q f32 (nb, Q))."""
    coords = np.asarray(coords, F32)
    dirs = directions(lattice)
    dim = forest.dim
    if dirs.shape[1] != dim:
        raise ValueError("lattice dimension mismatch")
    level = forest.n_levels - 1
    leaves = forest.leaves_at(level)
    ncell = 4 ** dim
    h64 = forest.spacing([level])[0] / 4.0
    h = h64.astype(F32)
    cen = forest.cell_centers(leaves).reshape(-1, dim)
    flo = coords.min(axis=0).T  # (F, D) f32
    fhi = coords.max(axis=0).T
    nq = len(dirs)
    flags = np.zeros(len(cen), np.uint32)
    qall = np.full((len(cen), nq), F32(-1.0), F32)
    # conservative per-block candidate faces: box of the block grown by 2 cells
    blo, bhi = forest.boxes(leaves)
    grow = 2.0 * h64
    dvs = [(dirs[i].astype(F32) * h).astype(F32) for i in range(nq)]  # exact: c in {-1,0,1}
    ends = [(cen + dv).astype(F32) for dv in dvs]
    for b0 in range(0, len(leaves), 256):
        b1 = min(len(leaves), b0 + 256)
        bl = np.repeat(np.arange(b0, b1), coords.shape[2])
        ff = np.tile(np.arange(coords.shape[2]), b1 - b0)
        ok = np.all((flo[ff] <= bhi[bl] + grow) & (fhi[ff] >= blo[bl] - grow), axis=1)
        bl, ff = bl[ok], ff[ok]
        if bl.size == 0:
            continue
        cell0 = np.repeat(bl * ncell, ncell) + np.tile(np.arange(ncell), bl.size)
        fac0 = np.repeat(ff, ncell)
        for i in range(1, nq):
            llo, lhi = np.minimum(cen[cell0], ends[i][cell0]), np.maximum(cen[cell0], ends[i][cell0])
            ov = np.all((flo[fac0] <= lhi) & (fhi[fac0] >= llo), axis=1)
            cell, fac = cell0[ov], fac0[ov]
            if cell.size == 0:
                continue
            hit, t = link_hits(cen[cell], dvs[i], coords[:, :, fac])
            cell, t = cell[hit], t[hit] + F32(0.0)  # -0 -> +0
            if cell.size == 0:
                continue
            flags[cell] |= np.uint32(1 << i)
            best = np.full(len(cen), np.inf, F32)
            np.minimum.at(best, cell, t)
            u = np.unique(cell)
            qall[u, i] = np.where(qall[u, i] < 0, best[u], np.minimum(qall[u, i], best[u]))
    boundary = np.flatnonzero(flags)
    return {"level": level, "leaves": leaves, "flags": flags, "boundary": boundary.astype(np.int64),
            "q": qall[boundary]}
