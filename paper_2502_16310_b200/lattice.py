"""Lattice boundary links and wall fractions q (north-star extension).

The reference has no lattice-link concept (SURVEY.md finding 6); this module
defines one (DESIGN.md §Lattice links) in the reference's conventions: the
cells are the finest-level leaf cells (ascending block id, x-fastest cell
index, nearwall.py:537-553) and all arithmetic is float32 with a fixed
operation order.  For each cell centre x and lattice direction c_i (i >= 1)
the segment x -> x + c_i*h is tested against every face whose float32 AABB
overlaps the segment's AABB, with Moller-Trumbore (3D) or segment-segment
(2D) intersection; bit i of the cell's flag word records a hit and q_i is the
smallest hit parameter t in [0, 1].
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .binning import BinGrid
from .errors import InvalidParameterError
from .forest import Forest
from .geometry import CoordListGeometry, validate_faces

D2Q9 = [(0, 0), (1, 0), (0, 1), (-1, 0), (0, -1), (1, 1), (-1, 1), (-1, -1), (1, -1)]
D3Q19 = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)] + [
    tuple(v) for v in (
        (1, 1, 0), (-1, -1, 0), (1, -1, 0), (-1, 1, 0),
        (1, 0, 1), (-1, 0, -1), (1, 0, -1), (-1, 0, 1),
        (0, 1, 1), (0, -1, -1), (0, 1, -1), (0, -1, 1),
    )
]
D3Q27 = D3Q19 + [(1 - 2 * ((k >> 2) & 1), 1 - 2 * ((k >> 1) & 1), 1 - 2 * (k & 1)) for k in range(8)]
LATTICES = {"D2Q9": D2Q9, "D3Q19": D3Q19, "D3Q27": D3Q27}


def lattice_directions(name):
    if name not in LATTICES:
        raise InvalidParameterError(f"unknown lattice {name!r}; expected one of {tuple(LATTICES)}")
    return np.asarray(LATTICES[name], dtype=np.int8)


@dataclass
class LatticeLinks:
    """Boundary links of the finest level.

    flags   uint32 (n_leaves * 4^dim,) — bit i set iff link i of the cell hits
            (int32 storage of the same bits on the device)
    cells   int64 (n_boundary,) flat cell index leaf_position * 4^dim + cell
    q       float32 (n_boundary, Q) — min hit fraction t, -1 where no hit
    leaves  int64 (n_leaves,) ascending finest-level leaf ids
    """

    lattice: str
    level: int
    leaves: torch.Tensor
    flags: torch.Tensor
    cells: torch.Tensor
    q: torch.Tensor

    @property
    def n_boundary(self):
        return int(self.cells.numel())

    def n_links(self):
        f = self.flags.to(torch.int64) & 0xFFFFFFFF
        return int(sum(((f >> i) & 1).sum().item() for i in range(1, 27)))


def build_lattice_links(forest: Forest, geom: CoordListGeometry, grid: BinGrid | None = None,
                        lattice="D3Q19", shard=None) -> LatticeLinks:
    """Boundary links of the finest level.

    Candidate faces come from the forest itself (each face visits the finest
    blocks its box can reach), so ``grid`` is accepted for API stability,
    checked for dimension, and otherwise unused: it never changes the result."""
    dirs = lattice_directions(lattice)
    if grid is not None and grid.dim != forest.dim:
        raise InvalidParameterError(f"bin grid is {grid.dim}D but forest is {forest.dim}D")
    if dirs.shape[1] != forest.dim or geom.dim != forest.dim:
        raise InvalidParameterError(f"lattice {lattice} does not match a {forest.dim}D forest")
    if geom.n_faces == 0:
        raise InvalidParameterError("cannot build lattice links with empty geometry")
    validate_faces(geom)
    level = forest.n_levels - 1
    leaves = forest._leaves(level)
    n_leaves = int(leaves.numel())
    ncell = forest.cells_per_block
    dev = forest.device
    flags = torch.empty(n_leaves * ncell, dtype=torch.int32, device=dev)
    nb = C.c_int64(0)
    hd = np.ascontiguousarray(dirs.reshape(-1))
    ctx, st = _lib.ctx(), _lib.stream()
    lo, hi = 0, n_leaves
    sharded = shard is not None and shard.world > 1
    if sharded:  # this rank's contiguous slice of the finest leaves (parallel.partition)
        from .parallel import partition

        lo, hi = partition(n_leaves, shard.rank, shard.world)
    _lib.call("ow_lattice_links_count_range", ctx, C.byref(forest.view()), level, _lib.ptr(leaves), n_leaves, lo, hi,
              _lib.ptr(geom.coords), geom.n_faces, geom.key, None,
              hd.ctypes.data_as(C.c_void_p), len(dirs),
              _lib.ptr(flags), C.byref(nb), st)
    n_b = int(nb.value)
    cells = torch.empty(n_b, dtype=torch.int64, device=dev)
    q = torch.empty((n_b, len(dirs)), dtype=torch.float32, device=dev)
    _lib.call("ow_lattice_links_emit", ctx, _lib.ptr(cells), _lib.ptr(q), st)
    if sharded:
        flags, cells, q = shard.gather_links(flags, cells, q, lo, hi, ncell, n_leaves)
    return LatticeLinks(lattice=lattice, level=level, leaves=leaves.to(torch.int64), flags=flags, cells=cells, q=q)
