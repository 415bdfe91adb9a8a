"""Oracle: near-wall marking, propagation, refinement driver, cell-face links.

Test infrastructure only.  Restates octowall/nearwall.py:
  coordinate scale / cull reach              nearwall.py:31-40
  face boxes + box-distance cull             nearwall.py:43-54, 64-133
  bounding-sphere prefilter                  nearwall.py:146-156, 162-214
  naive marking                              nearwall.py:217-242
  binned marking                             nearwall.py:253-311
  propagation rounds + two-pass dilation     nearwall.py:314-366
  per-level driver                           nearwall.py:430-491
  cell-face links (CSR, capacity order)      nearwall.py:522-594

A pair (cell c, face f) is evaluated iff f's FP64 box lies within ``reach``
of c's block box, c's FP32 distance to f's bounding-sphere centre passes the
sphere prefilter, and (binned) f is stored in the bin holding c's centre —
the same three filters the reference applies, evaluated here per pair and
vectorised in chunks instead of per block.
"""

from __future__ import annotations

import math

import numpy as np

from . import predicate
from .binning import Grid, fill_bins
from .errors import Capacity, InvalidParameter
from .forest import INTERMEDIATE, MARKED, NONE, Forest

F32 = np.float32
CHUNK = 1 << 21  # pairs per vectorised chunk


def coordinate_scale(forest: Forest, coords):
    s = max(float(np.abs(forest.dmin).max()), float(np.abs(forest.dmax).max()))
    if coords.shape[2]:
        s = max(s, float(np.abs(coords).max()))
    return s


def cull_reach(d, scale):
    return d + 1e-3 * max(1.0, scale, d)


def face_boxes(coords):
    c = np.asarray(coords, np.float64)
    return c.min(axis=0).T.copy(), c.max(axis=0).T.copy()


def face_spheres(lo, hi, reach):
    ctr = (0.5 * (lo + hi)).astype(F32)
    r = np.linalg.norm(0.5 * (hi - lo), axis=1) + reach
    return ctr, (r * r).astype(F32)


def box_gap_ok(blo, bhi, flo, fhi, reach):
    gap = np.maximum(0.0, np.maximum(flo - bhi, blo - fhi))
    return np.einsum("nd,nd->n", gap, gap) <= reach * reach


def _pairs_from_lists(owner_counts):
    """[3, 2] -> owner [0,0,0,1,1], rank [0,1,2,0,1]."""
    owner = np.repeat(np.arange(len(owner_counts)), owner_counts)
    start = np.cumsum(owner_counts) - owner_counts
    return owner, np.arange(owner.size) - start[owner]


class _Ctx:
    def __init__(self, forest, coords, d):
        self.coords = np.asarray(coords, F32)
        self.d = d
        self.reach = cull_reach(d, coordinate_scale(forest, self.coords))
        self.flo, self.fhi = face_boxes(self.coords)
        self.sc, self.sr2 = face_spheres(self.flo, self.fhi, self.reach)


def _check_inputs(forest, coords, d):
    from .geometry import first_degenerate

    if coords.shape[0] != forest.dim:
        raise InvalidParameter("dimension mismatch")
    if coords.shape[2] == 0:
        raise InvalidParameter("cannot mark near-wall blocks with empty geometry")
    if d <= 0:
        raise InvalidParameter("near-wall distance must be positive")
    if first_degenerate(coords) >= 0:
        raise InvalidParameter("degenerate face")


def _block_candidates(forest, blocks, ctx):
    """Per block, ascending faces passing the box cull: (owner, face)."""
    lo, hi = forest.boxes(blocks)
    nf = ctx.coords.shape[2]
    owners, faces = [], []
    step = max(1, CHUNK // max(nf, 1))
    for s in range(0, len(blocks), step):
        e = min(len(blocks), s + step)
        ob = np.repeat(np.arange(s, e), nf)
        ff = np.tile(np.arange(nf), e - s)
        ok = box_gap_ok(lo[ob], hi[ob], ctx.flo[ff], ctx.fhi[ff], ctx.reach)
        owners.append(ob[ok])
        faces.append(ff[ok])
    return np.concatenate(owners), np.concatenate(faces)


def _eval_pairs(ctx, pts, faces):
    """Sphere prefilter + exact predicate on (point, face) pairs."""
    dx = pts[:, 0] - ctx.sc[faces, 0]
    dy = pts[:, 1] - ctx.sc[faces, 1]
    dist = dx * dx + dy * dy
    if pts.shape[1] == 3:
        dz = pts[:, 2] - ctx.sc[faces, 2]
        dist = dist + dz * dz
    keep = dist <= ctx.sr2[faces]
    out = np.zeros(len(faces), bool)
    if np.any(keep):
        k = np.flatnonzero(keep)
        out[k] = predicate.near(pts[k], ctx.coords[:, :, faces[k]], ctx.d)
    return out


def cell_face_tests(forest: Forest, level, grid: Grid | None, counts, n_faces):
    """T = sum over leaf cells at ``level`` of |bin(centre)| (naive: n_faces)."""
    leaves = forest.leaves_at(level)
    ncell = 4 ** forest.dim
    if grid is None:
        return int(len(leaves) * ncell * n_faces)
    total = 0
    for s in range(0, len(leaves), 1 << 14):
        c = forest.cell_centers(leaves[s:s + (1 << 14)])
        total += int(np.asarray(counts, np.int64)[grid.bin_of(c)].sum())
    return total


def mark(forest: Forest, level, coords, d, bins=None, grid: Grid | None = None):
    """Naive (bins None) or binned marking of leaves at ``level``; returns #marked."""
    coords = np.asarray(coords, F32)
    _check_inputs(forest, coords, d)
    leaves = forest.leaves_at(level)
    todo = leaves[forest.marks[leaves] != MARKED]
    if len(todo) == 0:
        return 0
    ctx = _Ctx(forest, coords, d)
    ncell = 4 ** forest.dim
    hit = np.zeros(len(todo), bool)
    blk_step = max(1, CHUNK // (ncell * 64))
    for s in range(0, len(todo), blk_step):
        blocks = todo[s:s + blk_step]
        cen = forest.cell_centers(blocks)  # (nb, C, D)
        blo, bhi = forest.boxes(blocks)
        if bins is None:
            own, fac = _block_candidates(forest, blocks, ctx)
            # expand each (block, face) over the block's cells, chunk by chunk
            step = max(1, CHUNK // ncell)
            for c0 in range(0, len(own), step):
                pb = np.repeat(own[c0:c0 + step], ncell)
                pf = np.repeat(fac[c0:c0 + step], ncell)
                cell = np.tile(np.arange(ncell), len(pb) // ncell)
                res = _eval_pairs(ctx, cen[pb, cell], pf)
                hit[s + np.unique(pb[res])] = True
            continue
        else:
            ids, counts, offsets = bins
            cb = grid.bin_of(cen, what="cell center").reshape(-1)
            cnt = counts[cb].astype(np.int64)
            owner, rank = _pairs_from_lists(cnt)
            pf = ids[offsets[cb][owner] + rank].astype(np.int64)
            pb = owner // ncell
            cell = owner % ncell
            ok = box_gap_ok(blo[pb], bhi[pb], ctx.flo[pf], ctx.fhi[pf], ctx.reach)
            pb, pf, cell = pb[ok], pf[ok], cell[ok]
        for c0 in range(0, len(pb), CHUNK):
            sl = slice(c0, c0 + CHUNK)
            res = _eval_pairs(ctx, cen[pb[sl], cell[sl]], pf[sl])
            hit[s + np.unique(pb[sl][res])] = True
    forest.marks[todo[hit]] = MARKED
    return int(hit.sum())


def propagation_rounds(d, block_length):
    if d <= 0 or block_length <= 0:
        raise InvalidParameter("d_spec and block_length must be positive")
    return 1 + math.floor(d / block_length)


def propagate(forest: Forest, level, d, rounds=None):
    if np.any(forest.marks[forest.ids_at(level)] == INTERMEDIATE):
        raise InvalidParameter(f"level {level} already carries intermediate marks")
    if rounds is None:
        rounds = propagation_rounds(d, float(np.min(forest.spacing([level])[0])))
    leaves = forest.leaves_at(level)
    if len(leaves) == 0 or rounds == 0:
        return
    nbrs = forest.adjacent_leaves(leaves)
    owner = np.repeat(np.arange(len(leaves)), [len(x) for x in nbrs])
    flat = np.concatenate(nbrs) if nbrs else np.zeros(0, np.int64)
    for _ in range(rounds):
        got = np.zeros(len(leaves), bool)
        got[owner[forest.marks[flat] == MARKED]] = True
        grow = got & (forest.marks[leaves] == NONE)
        forest.marks[leaves[grow]] = INTERMEDIATE
        forest.marks[leaves[forest.marks[leaves] == INTERMEDIATE]] = MARKED


def refine_near_wall(forest: Forest, coords, d, n_levels=3, strategy="binned", bins_per_axis=8,
                     overlap_factor=10, spacing=None):
    """Returns dict(marked_detected, marked_refined, bins, cell_face_tests)."""
    coords = np.asarray(coords, F32)
    if coords.shape[2] == 0:
        raise InvalidParameter("cannot refine around empty geometry")
    lo, hi = coords.min(axis=(0, 2)).astype(np.float64), coords.max(axis=(0, 2)).astype(np.float64)
    tol = 1e-6 * forest.extent
    if np.any(lo < forest.dmin - tol) or np.any(hi > forest.dmax + tol):
        raise InvalidParameter("geometry outside the forest domain")
    out = {"marked_detected": [], "marked_refined": [], "bins": None, "cell_face_tests": []}
    binned = strategy == "binned"
    for level in range(n_levels - 1):
        if binned:
            grid = Grid(forest.dmin, forest.dmax, bins_per_axis)
            bins = fill_bins(coords, grid, spacing=spacing, overlap_factor=overlap_factor)
            out["bins"] = bins
            out["cell_face_tests"].append(cell_face_tests(forest, level, grid, bins[1], coords.shape[2]))
            out["marked_detected"].append(mark(forest, level, coords, d, bins, grid))
            propagate(forest, level, d)
        else:
            out["cell_face_tests"].append(cell_face_tests(forest, level, None, None, coords.shape[2]))
            out["marked_detected"].append(mark(forest, level, coords, d))
        leaves = forest.leaves_at(level)
        out["marked_refined"].append(int(np.sum(forest.marks[leaves] == MARKED)))
        forest.refine_marked(level)
    return out


def cell_face_links(forest: Forest, coords, bins, grid: Grid, d_link=None, capacity=16):
    """-> dict(level, d_link, block_ids, cell_indices, offsets, face_ids)."""
    coords = np.asarray(coords, F32)
    _check_inputs(forest, coords, 1.0 if d_link is None else d_link)
    level = forest.n_levels - 1
    if d_link is None:
        cell = forest.spacing([level])[0] / 4.0
        d_link = math.sqrt(forest.dim) * float(np.linalg.norm(cell))
    leaves = forest.leaves_at(level)
    if len(leaves) == 0:
        raise InvalidParameter(f"no leaf blocks at finest level {level}")
    ctx = _Ctx(forest, coords, d_link)
    ids, counts, offsets = bins
    ncell = 4 ** forest.dim
    cen = forest.cell_centers(leaves)
    blo, bhi = forest.boxes(leaves)
    cb = grid.bin_of(cen, what="cell center").reshape(-1)
    owner, rank = _pairs_from_lists(counts[cb].astype(np.int64))
    pf = ids[offsets[cb][owner] + rank].astype(np.int64)
    pb = owner // ncell
    ok = box_gap_ok(blo[pb], bhi[pb], ctx.flo[pf], ctx.fhi[pf], ctx.reach)
    owner, pf, pb = owner[ok], pf[ok], pb[ok]
    res = np.zeros(len(pf), bool)
    flat = cen.reshape(-1, forest.dim)
    for c0 in range(0, len(pf), CHUNK):
        sl = slice(c0, c0 + CHUNK)
        res[sl] = predicate.near(flat[owner[sl]], coords[:, :, pf[sl]], d_link)
    owner, pf = owner[res], pf[res]  # ascending cell, ascending face within cell
    hits = np.bincount(owner, minlength=len(flat))
    over = np.flatnonzero(hits > capacity)
    if over.size:
        key = (over // ncell) * (grid.n_bins * ncell) + cb[over] * ncell + over % ncell
        w = over[np.argmin(key)]
        raise Capacity(f"cell-face link overflow: block {int(leaves[w // ncell])} cell {int(w % ncell)} "
                       f"links {int(hits[w])} faces, capacity {capacity}")
    linked = np.flatnonzero(hits)
    return {
        "level": level,
        "d_link": float(d_link),
        "block_ids": leaves[linked // ncell].astype(np.int64),
        "cell_indices": (linked % ncell).astype(np.int64),
        "offsets": np.concatenate([[0], np.cumsum(hits[linked])]).astype(np.int64),
        "face_ids": pf.astype(np.int32),
    }
