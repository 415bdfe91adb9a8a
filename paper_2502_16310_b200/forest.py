"""Forest-of-octrees Cartesian grid resident in HBM.

Mirrors octowall/forest.py: dense monotone block ids, SoA block metadata,
x-fastest root grid, FP64 -> FP32 cell centres, deterministic splits and
2:1 face balance.  All block arrays are CUDA tensors (PyTorch owns the
memory); the hot operations — leaf listing, cell centres, refinement with
rebalancing, propagation — are libowb200 kernels.  The forest grows through
a callback the C library invokes when a split needs more capacity.

Layout (HBM, struct of arrays, `capacity` entries each):
    level int16 | coord[axis] int32 (lattice coords at the block's level)
    parent int32 | first_child int32 (-1 for leaves) | marks int8
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass
from enum import IntEnum

import numpy as np
import torch

from . import _lib
from .errors import InvalidParameterError
from .geometry import Aabb

CELLS_PER_AXIS = 4
DEFAULT_MAX_LEVEL = 10
MAX_LEVELS = 28


class RefineMark(IntEnum):
    NONE = 0
    MARKED = 1
    INTERMEDIATE = 2


@dataclass
class Block:
    id: int
    level: int
    origin: np.ndarray
    length: np.ndarray
    parent: int
    children: tuple
    mark: RefineMark

    @property
    def is_leaf(self):
        return not self.children


class Forest:
    def __init__(self, domain: Aabb, root_dims, max_level=DEFAULT_MAX_LEVEL, capacity=None, _init_root=True):
        root_dims = np.asarray(root_dims, dtype=np.int64).reshape(-1)
        if root_dims.shape[0] != domain.dim:
            raise InvalidParameterError(f"root_dims has {root_dims.shape[0]} axes but domain is {domain.dim}D")
        if np.any(root_dims < 1):
            raise InvalidParameterError(f"root_dims must be >= 1 per axis, got {root_dims.tolist()}")
        if np.any(domain.extent <= 0):
            raise InvalidParameterError("domain must have positive extent")
        if domain.dim not in (2, 3):
            raise InvalidParameterError(f"domain must be 2D or 3D, got {domain.dim}D")
        if max_level > MAX_LEVELS - 2:
            raise InvalidParameterError(f"max_level must be <= {MAX_LEVELS - 2}")
        self.dim = domain.dim
        self.domain = domain
        self.root_dims = tuple(int(v) for v in root_dims)
        self.max_level = max_level
        self.n_children = 2 ** self.dim
        self.cells_per_block = CELLS_PER_AXIS ** self.dim
        self.device = _lib.device()
        r = int(np.prod(root_dims))
        cap = max(int(capacity or 0), 4 * r, 1024)
        self._alloc(cap)
        self._n = 0
        self._n_levels = 1
        self._version = 0
        self._leaf_cache = {}
        self._view_struct = _lib.ForestView()
        # the callback holds the forest weakly: a bound method would form a
        # reference cycle that keeps every forest (and its HBM) alive until
        # the cyclic GC runs
        ref = weakref.ref(self)

        def grow(user, view_p, need):
            f = ref()
            return 1 if f is None else f._grow(user, view_p, need)

        self._grow_cb = _lib.GROW_FN(grow)
        # root blocks 0..R-1 (x-fastest lattice coords, level 0, no parent): one
        # kernel (ow_geometry_to_grid runs it itself: _init_root=False)
        if _init_root:
            v = self.view()
            _lib.call("ow_forest_init_root", _lib.ctx(), C.byref(v), _lib.stream())
            self._sync_from_view()

    # ------------------------------------------------------------------ storage
    def _alloc(self, cap):
        # entries past n_blocks are never read: the split kernel writes every
        # field of each block it appends, so the storage is left uninitialised
        dev = self.device
        self._cap = cap
        self._level_t = torch.empty(cap, dtype=torch.int16, device=dev)
        self._coord = [torch.empty(cap, dtype=torch.int32, device=dev) for _ in range(self.dim)]
        self._parent_t = torch.empty(cap, dtype=torch.int32, device=dev)
        self._first_child_t = torch.empty(cap, dtype=torch.int32, device=dev)
        self._marks = torch.empty(cap, dtype=torch.int8, device=dev)

    def _resize(self, new_cap, n):
        old = (self._level_t, self._coord, self._parent_t, self._first_child_t, self._marks)
        self._alloc(new_cap)
        self._level_t[:n] = old[0][:n]
        for ax in range(self.dim):
            self._coord[ax][:n] = old[1][ax][:n]
        self._parent_t[:n] = old[2][:n]
        self._first_child_t[:n] = old[3][:n]
        self._marks[:n] = old[4][:n]

    def reserve(self, n_blocks):
        """Make room for ``n_blocks`` blocks (geometric growth, one copy)."""
        if n_blocks > self._cap:
            self._resize(max(int(n_blocks), 2 * self._cap), self._n)

    def _grow(self, _user, view_p, need):
        try:
            # the C side may already have appended blocks during this refine
            # call: its view holds the live count, not self._n
            n = int(view_p.contents.n_blocks)
            self._n = n
            self._resize(max(int(need), 2 * self._cap), n)
            self._fill_view(view_p.contents)
            return 0
        except Exception:  # pragma: no cover - reported by the C side as a failed grow
            return 1

    def _fill_view(self, v):
        if not getattr(v, "_static_done", False):  # domain / root grid: once per (owned) struct
            v.dim = self.dim
            v.max_level = self.max_level
            for a in range(3):
                v.root[a] = self.root_dims[a] if a < self.dim else 1
                v.dmin[a] = float(self.domain.min[a]) if a < self.dim else 0.0
                v.dext[a] = float(self.domain.extent[a]) if a < self.dim else 1.0
            v._static_done = True
        v.max_level = self.max_level
        for a in range(3):
            v.d_coord[a] = self._coord[a].data_ptr() if a < self.dim else 0
        v.n_blocks = self._n
        v.capacity = self._cap
        v.d_level = self._level_t.data_ptr()
        v.d_parent = self._parent_t.data_ptr()
        v.d_first_child = self._first_child_t.data_ptr()
        v.d_marks = self._marks.data_ptr()
        v.grow = self._grow_cb
        v.grow_user = None

    def view(self):
        """ow_forest struct describing the current device arrays."""
        self._fill_view(self._view_struct)
        return self._view_struct

    def _reset_for_pass(self):
        """Empty forest over the same storage (ow_geometry_to_grid writes the roots)."""
        self._n = 0
        self._n_levels = 1
        self._version += 1
        self._leaf_cache.clear()

    def _sync_from_view(self):
        self._n = int(self._view_struct.n_blocks)

    # ------------------------------------------------------------------ basics
    @property
    def n_blocks(self):
        return self._n

    @property
    def n_levels(self):
        return self._n_levels

    @property
    def capacity(self):
        return self._cap

    @property
    def marks(self):
        """Refinement marks (int8 CUDA tensor view of the n_blocks live entries)."""
        return self._marks[: self._n]

    @marks.setter
    def marks(self, value):
        self._marks[: self._n] = torch.as_tensor(value, dtype=torch.int8, device=self.device)[: self._n]

    @property
    def level_tensor(self):
        return self._level_t[: self._n]

    @property
    def coords_tensor(self):
        return torch.stack([c[: self._n] for c in self._coord], 1)

    # host copies for reference-style inspection (forest.py keeps these in NumPy)
    @property
    def _level(self):
        return self._level_t[: self._n].cpu().numpy()

    @property
    def _coords(self):
        return self.coords_tensor.cpu().numpy().astype(np.int64)

    @property
    def _parent(self):
        return self._parent_t[: self._n].cpu().numpy()

    @property
    def _first_child(self):
        return self._first_child_t[: self._n].cpu().numpy()

    # ------------------------------------------------------------------ queries
    def level_counts(self):
        b = (C.c_int64 * MAX_LEVELS)()
        lv = (C.c_int64 * MAX_LEVELS)()
        _lib.call("ow_forest_level_counts", _lib.ctx(), C.byref(self.view()), b, lv, MAX_LEVELS, _lib.stream())
        n = self._n_levels
        return [int(b[i]) for i in range(n)], [int(lv[i]) for i in range(n)]

    def blocks_per_level(self):
        return self.level_counts()[0]

    def leaves_per_level(self):
        return self.level_counts()[1]

    def _leaves(self, level):
        """Ascending leaf ids at ``level`` as an int32 CUDA tensor (hot path).

        Cached until the block structure changes (refine_marked); marks do
        not change the leaf set."""
        key = (self._version, int(level))
        hit = self._leaf_cache.get(key)
        if hit is not None:
            return hit
        out = torch.empty(max(self._n, 1), dtype=torch.int32, device=self.device)
        n = C.c_int64(0)
        _lib.call("ow_forest_leaves", _lib.ctx(), C.byref(self.view()), int(level), _lib.ptr(out), C.byref(n),
                  _lib.stream())
        res = out[: n.value]
        if len(self._leaf_cache) > 8:
            self._leaf_cache.clear()
        self._leaf_cache[key] = res
        return res

    def leaf_blocks_at(self, level):
        if level < 0 or level >= self._n_levels:
            return torch.zeros(0, dtype=torch.int64, device=self.device)
        return self._leaves(level).to(torch.int64)

    def ids_at_level(self, level):
        return torch.nonzero(self.level_tensor == level).flatten()

    def all_leaf_ids(self):
        return torch.nonzero(self._first_child_t[: self._n] == -1).flatten()

    def is_leaf(self, bid):
        return int(self._first_child_t[int(bid)]) == -1

    def count_marks(self, level, mark, leaf_only=True):
        n = C.c_int64(0)
        _lib.call("ow_forest_count_marks", _lib.ctx(), C.byref(self.view()), int(level), int(bool(leaf_only)),
                  int(mark), C.byref(n), _lib.stream())
        return int(n.value)

    def block_length(self, level):
        return self.domain.extent / (np.asarray(self.root_dims) * (1 << level))

    def block_origins(self, ids):
        ids = np.asarray(torch.as_tensor(ids).cpu(), dtype=np.int64)
        lv = self._level[ids].astype(np.int64)
        denom = np.asarray(self.root_dims)[None, :] * (1 << lv)[:, None]
        return self.domain.min[None, :] + self._coords[ids] * (self.domain.extent[None, :] / denom)

    def block_aabbs(self, ids):
        ids = np.asarray(torch.as_tensor(ids).cpu(), dtype=np.int64)
        lo = self.block_origins(ids)
        lv = self._level[ids].astype(np.int64)
        ln = self.domain.extent[None, :] / (np.asarray(self.root_dims)[None, :] * (1 << lv)[:, None])
        return lo, lo + ln

    def block(self, bid):
        bid = int(bid)
        if bid < 0 or bid >= self._n:
            raise InvalidParameterError(f"no block with id {bid}")
        level = int(self._level_t[bid])
        fc = int(self._first_child_t[bid])
        return Block(id=bid, level=level, origin=self.block_origins([bid])[0], length=self.block_length(level),
                     parent=int(self._parent_t[bid]),
                     children=() if fc == -1 else tuple(range(fc, fc + self.n_children)),
                     mark=RefineMark(int(self._marks[bid])))

    def cell_centers_many(self, ids):
        """(n, 4^dim, dim) float32 CUDA tensor: FP64 from lattice coords, one rounding."""
        ids_t = torch.as_tensor(ids, device=self.device).to(torch.int32).contiguous()
        n = int(ids_t.numel())
        out = torch.empty((n, self.cells_per_block, self.dim), dtype=torch.float32, device=self.device)
        _lib.call("ow_forest_cell_centers", _lib.ctx(), C.byref(self.view()), _lib.ptr(ids_t), n, _lib.ptr(out),
                  _lib.stream())
        return out

    def cell_centers(self, bid):
        return self.cell_centers_many([int(bid)])[0]

    # --------------------------------------------------------- neighbours (host)
    def _host_arrays(self):
        return self._level, self._coords, self._first_child

    def _locate_host(self, lvl, nc, fc):
        node, stride = 0, 1
        for a in range(self.dim):
            node += (int(nc[a]) >> lvl) * stride
            stride *= self.root_dims[a]
        depth = 0
        while depth < lvl and fc[node] != -1:
            sh = lvl - 1 - depth
            ci = sum(((int(nc[a]) >> sh) & 1) << a for a in range(self.dim))
            node = int(fc[node]) + ci
            depth += 1
        return node

    def face_neighbors(self, bid):
        """Adjacent leaves per side (ax0-, ax0+, ...), forest.py:224-244."""
        level, coords, fc = self._host_arrays()
        bid = int(bid)
        lv = int(level[bid])
        out = []
        for ax in range(self.dim):
            for step in (-1, 1):
                nc = coords[bid].copy()
                nc[ax] += step
                if nc[ax] < 0 or nc[ax] >= self.root_dims[ax] << lv:
                    out.append(())
                    continue
                node = self._locate_host(lv, nc, fc)
                want = 0 if step == 1 else 1
                stack, found = [node], []
                while stack:
                    b = stack.pop()
                    if fc[b] == -1:
                        found.append(int(b))
                    else:
                        stack.extend(int(fc[b]) + ci for ci in range(self.n_children) if ((ci >> ax) & 1) == want)
                out.append(tuple(sorted(found)))
        return out

    def adjacent_leaf_ids(self, bid):
        ids = []
        for side in self.face_neighbors(bid):
            ids.extend(side)
        return sorted(set(ids))

    # ------------------------------------------------------------------ refinement
    def refine_marked(self, level):
        """Split MARKED leaves at ``level`` (ascending id) and restore 2:1 balance."""
        v = self.view()
        out = C.c_int64(0)
        try:
            _lib.call("ow_refine_marked", _lib.ctx(), C.byref(v), int(level), C.byref(out), _lib.stream())
        finally:
            self._sync_from_view()
            self._version += 1
            self._leaf_cache.clear()
        n = int(out.value)
        if n > 0:
            self._n_levels = max(self._n_levels, int(level) + 2)
        return n

    # ------------------------------------------------------------------ comparison
    def refines_at_least(self, other):
        if self.root_dims != other.root_dims or self.dim != other.dim:
            raise InvalidParameterError("forests with different root grids are not comparable")
        mine = set()
        lv, co = self._level, self._coords
        for i in range(self._n):
            mine.add((int(lv[i]), tuple(int(x) for x in co[i])))
        olv, oco, ofc = other._level, other._coords, other._first_child
        for i in np.flatnonzero(ofc == -1):
            if (int(olv[i]), tuple(int(x) for x in oco[i])) not in mine:
                return False
        return True

    def level_signature(self):
        lv, co, fc = self._level, self._coords, self._first_child
        sig = []
        for level in range(self._n_levels):
            c = co[(lv == level) & (fc == -1)]
            sig.append(c[np.lexsort(c.T[::-1])].copy())
        return sig


def init_root_grid(domain, root_dims, max_level=DEFAULT_MAX_LEVEL, capacity=None) -> Forest:
    if not isinstance(domain, Aabb):
        domain = Aabb(*domain)
    return Forest(domain, root_dims, max_level=max_level, capacity=capacity)
