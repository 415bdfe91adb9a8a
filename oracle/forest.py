"""Oracle: forest of quadtrees / octrees (test infrastructure only).

Restates octowall/forest.py:
  block storage, x-fastest root grid       forest.py:47-129, 405-409
  leaves per level                         forest.py:135-150
  block origin / length / cell centres     forest.py:152-205
  face neighbours across levels            forest.py:224-285
  split (deterministic child ids)          forest.py:300-329
  refine MARKED leaves + 2:1 rebalance     forest.py:331-370
  level signature                          forest.py:388-402

The reference finds blocks through a (level, coords) -> id dictionary; the
oracle instead descends from the root lattice by child bits (same answers,
checked against the reference's neighbour known answers and goldens).
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidParameter

NONE, MARKED, INTERMEDIATE = 0, 1, 2


class Forest:
    def __init__(self, dmin, dmax, root_dims, max_level=10):
        self.dmin = np.asarray(dmin, np.float64)
        self.dmax = np.asarray(dmax, np.float64)
        self.extent = self.dmax - self.dmin
        self.dim = len(self.dmin)
        self.root = np.asarray(root_dims, np.int64)
        self.max_level = max_level
        self.nc = 1 << self.dim
        r = int(np.prod(self.root))
        idx = np.arange(r)
        coords = np.empty((r, self.dim), np.int64)
        rem = idx
        for ax in range(self.dim):
            coords[:, ax] = rem % self.root[ax]
            rem = rem // self.root[ax]
        self.level = np.zeros(r, np.int16)
        self.coords = coords
        self.parent = np.full(r, -1, np.int32)
        self.first_child = np.full(r, -1, np.int32)
        self.marks = np.zeros(r, np.int8)

    @property
    def n(self):
        return len(self.level)

    @property
    def n_levels(self):
        return int(self.level.max()) + 1

    # --- queries ---------------------------------------------------------
    def leaves_at(self, level):
        return np.flatnonzero((self.level == level) & (self.first_child == -1))

    def ids_at(self, level):
        return np.flatnonzero(self.level == level)

    def blocks_per_level(self):
        return np.bincount(self.level, minlength=self.n_levels).tolist()

    def leaves_per_level(self):
        leaf = self.first_child == -1
        return np.bincount(self.level[leaf], minlength=self.n_levels).tolist()

    def spacing(self, levels):
        """Block edge per axis (n, D) float64: extent / (root * 2^L)."""
        lv = np.asarray(levels, np.int64)
        return self.extent[None, :] / (self.root[None, :] * (np.int64(1) << lv)[:, None])

    def origins(self, ids):
        ids = np.asarray(ids, np.int64)
        return self.dmin[None, :] + self.coords[ids] * self.spacing(self.level[ids])

    def boxes(self, ids):
        lo = self.origins(ids)
        return lo, lo + self.spacing(self.level[np.asarray(ids, np.int64)])

    def cell_centers(self, ids):
        """(n, 4^D, D) float32; cell index x fastest; FP64 then one rounding."""
        ids = np.asarray(ids, np.int64)
        o = self.origins(ids)
        q = self.spacing(self.level[ids])
        frac = (np.arange(4) + 0.5) / 4
        grid = np.stack(np.meshgrid(*([frac] * self.dim), indexing="ij"), -1)
        unit = grid.transpose(*range(self.dim - 1, -1, -1), self.dim).reshape(-1, self.dim)
        return (o[:, None, :] + unit[None, :, :] * q[:, None, :]).astype(np.float32)

    def locate(self, level, nc):
        """Deepest existing block on the path to lattice cell (level, nc).

        nc: (n, D) int64 at ``level``; returns block ids (n,).  The result is
        at ``level`` when that block exists, else the coarser leaf covering it.
        """
        level = np.broadcast_to(np.asarray(level, np.int64), (len(nc),))
        rc = nc >> level[:, None]
        node = rc[:, self.dim - 1].copy()
        for ax in range(self.dim - 2, -1, -1):
            node = node * self.root[ax] + rc[:, ax]
        depth = np.zeros(len(nc), np.int64)
        active = depth < level
        while np.any(active):
            fc = self.first_child[node]
            go = active & (fc != -1)
            if not np.any(go):
                break
            shift = (level - 1 - depth)[go]
            ci = np.zeros(int(go.sum()), np.int64)
            for ax in range(self.dim):
                ci |= ((nc[go, ax] >> shift) & 1) << ax
            node[go] = fc[go] + ci
            depth[go] += 1
            active = go & (depth < level)
        return node

    def _side_targets(self, ids):
        """For each id and side (ax-, ax+, ...): neighbour lattice cell + validity."""
        ids = np.asarray(ids, np.int64)
        lv = self.level[ids].astype(np.int64)
        dims = self.root[None, :] << lv[:, None]
        out = []
        for ax in range(self.dim):
            for step in (-1, 1):
                nc = self.coords[ids].copy()
                nc[:, ax] += step
                ok = (nc[:, ax] >= 0) & (nc[:, ax] < dims[:, ax])
                out.append((ax, step, np.where(ok[:, None], nc, 0), ok))
        return lv, out

    def adjacent_leaves(self, ids):
        """Sorted unique face-adjacent leaves of each id (list of arrays)."""
        ids = np.asarray(ids, np.int64)
        lv, sides = self._side_targets(ids)
        qid, leaf = [], []
        for ax, step, nc, ok in sides:
            sel = np.flatnonzero(ok)
            node = self.locate(lv[sel], nc[sel])
            want = 0 if step == 1 else 1  # children on the face toward us
            owner = sel
            while True:
                fc = self.first_child[node]
                is_leaf = fc == -1
                qid.append(owner[is_leaf])
                leaf.append(node[is_leaf])
                if np.all(is_leaf):
                    break
                par = node[~is_leaf]
                own = owner[~is_leaf]
                kids = [ci for ci in range(self.nc) if ((ci >> ax) & 1) == want]
                node = (self.first_child[par][:, None] + np.asarray(kids)[None, :]).reshape(-1)
                owner = np.repeat(own, len(kids))
        qid = np.concatenate(qid)
        leaf = np.concatenate(leaf)
        key = np.unique(qid * (self.n + 1) + leaf)
        q, l = key // (self.n + 1), key % (self.n + 1)
        bounds = np.searchsorted(q, np.arange(len(ids) + 1))
        return [l[bounds[i]:bounds[i + 1]] for i in range(len(ids))]

    def face_neighbors(self, bid):
        """Per-side tuples like forest.py:224-244 (for known-answer tests)."""
        lv, sides = self._side_targets([bid])
        res = []
        for ax, step, nc, ok in sides:
            if not ok[0]:
                res.append(())
                continue
            node = self.locate(lv, nc)
            want = 0 if step == 1 else 1
            stack, found = [int(node[0])], []
            while stack:
                b = stack.pop()
                fc = int(self.first_child[b])
                if fc == -1:
                    found.append(b)
                else:
                    stack.extend(fc + ci for ci in range(self.nc) if ((ci >> ax) & 1) == want)
            res.append(tuple(sorted(found)))
        return res

    # --- mutation ----------------------------------------------------------
    def _append_children(self, parents):
        parents = np.asarray(parents, np.int64)
        m = len(parents)
        if m == 0:
            return np.zeros(0, np.int64)
        if np.any(self.first_child[parents] != -1):
            raise InvalidParameter("cannot split an already refined block")
        if np.any(self.level[parents] >= self.max_level):
            raise InvalidParameter(f"refinement beyond max level {self.max_level}")
        base = self.n
        ci = np.arange(self.nc)
        bits = ((ci[:, None] >> np.arange(self.dim)[None, :]) & 1).astype(np.int64)
        kid_coords = (2 * self.coords[parents])[:, None, :] + bits[None, :, :]
        self.level = np.concatenate([self.level, np.repeat(self.level[parents] + 1, self.nc).astype(np.int16)])
        self.coords = np.concatenate([self.coords, kid_coords.reshape(-1, self.dim)])
        self.parent = np.concatenate([self.parent, np.repeat(parents, self.nc).astype(np.int32)])
        self.first_child = np.concatenate([self.first_child, np.full(m * self.nc, -1, np.int32)])
        self.marks = np.concatenate([self.marks, np.zeros(m * self.nc, np.int8)])
        self.first_child[parents] = base + self.nc * np.arange(m)
        self.marks[parents] = NONE
        return np.arange(base, self.n)

    def refine_marked(self, level):
        if np.any(self.marks[self.ids_at(level)] == INTERMEDIATE):
            raise InvalidParameter(f"level {level} still carries intermediate marks")
        leaves = self.leaves_at(level)
        marked = leaves[self.marks[leaves] == MARKED]
        frontier = self._append_children(marked)
        n_split = len(marked)
        while len(frontier):
            lv, sides = self._side_targets(frontier)
            viol = []
            for ax, step, nc, ok in sides:
                sel = np.flatnonzero(ok)
                node = self.locate(lv[sel], nc[sel])
                bad = (self.first_child[node] == -1) & (self.level[node] < lv[sel] - 1)
                viol.append(node[bad])
            viol = np.unique(np.concatenate(viol))
            frontier = self._append_children(viol)
            n_split += len(viol)
        return n_split

    def level_signature(self):
        sig = []
        for lv in range(self.n_levels):
            c = self.coords[self.leaves_at(lv)]
            sig.append(c[np.lexsort(c.T[::-1])])
        return sig
