"""Exact-arithmetic referees for lattice links (test infrastructure only).

The lattice-link definition (oracle/lattice.py) is a north-star extension with
no reference implementation, so besides the analytic known answers it is
checked against geometry computed independently in float64, in the style of
the reference's own predicate referee (validate.py:98-141, which compares the
float32 predicate against an FP64 distance with an error band):

* ``StarSurface``: inside / outside of a closed mesh that is star-shaped
  about a centre (the icospheres of C2 / C5, the bumpy sphere of C3): the
  FP64 crossing of the ray from the centre through the point with the mesh
  gives the radial signed distance; points closer than a band to the
  surface are excluded as ambiguous.
* ``segment_t64``: FP64 Moller-Trumbore on (segment, triangle) pairs with
  barycentric margins, for the wall-distance fraction q.

Nothing in the product imports this module.
"""

from __future__ import annotations

import numpy as np

F64 = np.float64


class StarSurface:
    """FP64 side test of a closed mesh that is star-shaped about `centre`
    (every ray from the centre crosses it once: the icospheres of C2 / C5,
    the bumpy sphere of C3).  coords (3, 3, F) float32."""

    def __init__(self, coords, centre=(0.5, 0.5, 0.5), k=24):
        from scipy.spatial import cKDTree

        self.tri = np.transpose(np.asarray(coords, F64), (2, 0, 1))  # (F, vertex, axis)
        self.c = np.asarray(centre, F64)
        cd = self.tri.mean(axis=1) - self.c
        self.tree = cKDTree(cd / np.linalg.norm(cd, axis=1, keepdims=True))
        self.k = k

    def signed(self, p):
        """|p - c| minus the distance from c to the surface along the ray
        through p (> 0 outside); NaN when no candidate face holds the ray."""
        p = np.asarray(p, F64).reshape(-1, 3)
        r = p - self.c
        rn = np.linalg.norm(r, axis=1)
        u = r / rn[:, None]
        _, nb = self.tree.query(u, self.k)
        tri = self.tri[nb]  # (n, k, 3, 3)
        e1 = tri[:, :, 1] - tri[:, :, 0]
        e2 = tri[:, :, 2] - tri[:, :, 0]
        d = np.broadcast_to(u[:, None, :], e1.shape)
        pv = np.cross(d, e2)
        det = np.einsum("nkj,nkj->nk", e1, pv)
        s = self.c - tri[:, :, 0]
        qv = np.cross(s, e1)
        with np.errstate(divide="ignore", invalid="ignore"):
            bu = np.einsum("nkj,nkj->nk", s, pv) / det
            bv = np.einsum("nkj,nkj->nk", d, qv) / det
            t = np.einsum("nkj,nkj->nk", e2, qv) / det
        ok = (det != 0) & (bu >= -1e-12) & (bv >= -1e-12) & (bu + bv <= 1 + 1e-12) & (t > 0)
        tt = np.where(ok, t, np.inf).min(axis=1)
        return np.where(np.isfinite(tt), rn - tt, np.nan)


def segment_t64(x, e, tri):
    """FP64 segment-triangle intersection of pairs: x, e (n, 3) segment ends,
    tri (n, 3, 3) [pair, vertex, axis].  Returns (u, v, t, det) with the
    barycentrics of the crossing point and t along x -> e."""
    x, e, tri = (np.asarray(a, F64) for a in (x, e, tri))
    d = e - x
    e1 = tri[:, 1] - tri[:, 0]
    e2 = tri[:, 2] - tri[:, 0]
    p = np.cross(d, e2)
    det = np.einsum("ij,ij->i", e1, p)
    s = x - tri[:, 0]
    qv = np.cross(s, e1)
    with np.errstate(divide="ignore", invalid="ignore"):
        u = np.einsum("ij,ij->i", s, p) / det
        v = np.einsum("ij,ij->i", d, qv) / det
        t = np.einsum("ij,ij->i", e2, qv) / det
    return u, v, t, det


def check_links(cen, dvs, flags, q, coords, surface=None, band=1e-6, tol=1e-5, chunk=8192):
    """Referee of lattice links for the given cells.

    cen (n, D=3) f32 cell centres; dvs (Q, 3) f32 link vectors; flags (n,)
    uint32 flag words and q (n, Q) f32 of these cells (as the product or the
    oracle computed them); coords (3, 3, F) f32; surface: a StarSurface of
    the same mesh for the closed-mesh invariants (None: q checks only).
    (A convex surface cannot meet a link with both ends inside; for a merely
    star-shaped one `inside_flagged` is informational.)

    Returns a dict of counts:
      crossing / crossing_missed: links whose ends lie on opposite sides of the
        closed surface (FP64, both ends farther than `band` from it) / those
        of them left unflagged (the watertightness invariant: must be 0);
      inside / inside_flagged: links with both ends inside by more than `band`
        / those flagged;
      flagged / q_checked / q_bad / q_ambiguous: flagged links, those whose
        FP64 crossing with a face holds with margin, those whose float32 q
        differs from the FP64 min t by more than `tol`, and flagged links with
        no FP64 crossing beyond the margins (grazing an edge or an end);
      unflagged_hit: unflagged links that the FP64 test crosses with margin
        (a miss of the float32 definition away from every edge: must be 0).
    """
    from scipy.spatial import cKDTree

    cen = np.asarray(cen, np.float32)
    flags = np.asarray(flags, np.uint32)
    n, nq = len(cen), len(dvs)
    tri = np.transpose(np.asarray(coords, F64), (2, 0, 1))
    cent = tri.mean(axis=1)
    rmax = float(np.max(np.linalg.norm(tri - cent[:, None, :], axis=2)))
    tree = cKDTree(cent)
    dv64 = np.asarray(dvs, F64)
    reach = float(np.max(np.linalg.norm(dv64, axis=1)))
    out = dict(crossing=0, crossing_missed=0, inside=0, inside_flagged=0, flagged=0, q_checked=0, q_bad=0,
               q_ambiguous=0, q_max_err=0.0, unflagged_hit=0)
    eps = 1e-9
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        x64 = cen[c0:c1].astype(F64)
        near = tree.query_ball_point(x64, reach + rmax)
        lens = np.fromiter((len(a) for a in near), np.int64, len(near))
        rep = np.repeat(np.arange(c1 - c0), lens)
        fac = np.concatenate([np.asarray(a, np.int64) for a in near]) if rep.size else np.zeros(0, np.int64)
        s0 = surface.signed(x64) if surface is not None else None
        for i in range(1, nq):
            fl = ((flags[c0:c1] >> np.uint32(i)) & 1).astype(bool)
            if surface is not None:
                s1 = surface.signed(x64 + dv64[i])
                cross = ((s0 < -band) & (s1 > band)) | ((s0 > band) & (s1 < -band))
                inside = (s0 < -band) & (s1 < -band)
                out["crossing"] += int(cross.sum())
                out["crossing_missed"] += int((cross & ~fl).sum())
                out["inside"] += int(inside.sum())
                out["inside_flagged"] += int((inside & fl).sum())
            out["flagged"] += int(fl.sum())
            if rep.size == 0:
                out["q_ambiguous"] += int(fl.sum())
                continue
            xs = x64[rep]
            u, v, t, det = segment_t64(xs, xs + dv64[i], tri[fac])
            with np.errstate(invalid="ignore"):
                ok = (det != 0) & (u >= eps) & (v >= eps) & (u + v <= 1 - eps) & (t >= eps) & (t <= 1 - eps)
                touch = (det != 0) & (u >= -eps) & (v >= -eps) & (u + v <= 1 + eps) & (t >= -eps) & (t <= 1 + eps)
            tmin = np.full(c1 - c0, np.inf)
            np.minimum.at(tmin, rep[touch], np.clip(t[touch], 0.0, 1.0))
            clear = np.zeros(c1 - c0, bool)
            clear[rep[ok]] = True
            out["unflagged_hit"] += int((clear & ~fl).sum())
            chk = fl & clear
            out["q_ambiguous"] += int((fl & ~clear).sum())
            if chk.any():
                err = np.abs(q[c0:c1][chk, i].astype(F64) - tmin[chk])
                out["q_checked"] += int(chk.sum())
                out["q_max_err"] = max(out["q_max_err"], float(err.max()))
                out["q_bad"] += int((err > tol).sum())
    return out
