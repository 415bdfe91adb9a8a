"""Multi-GPU sharding of the geometry-to-grid pass: one process per GPU.

Octree blocks are independent units for marking, so each rank marks a
contiguous slice of the level's ascending leaf list and the per-leaf marks
are all-gathered.  The forest metadata and the bin CSR are replicated: every
rank builds them from the same inputs with the same deterministic kernels,
so propagation and refinement (tiny, latency-bound) run redundantly and
produce identical block ids on every rank without any further exchange
(SURVEY.md §8e).

Two exchange paths:

* ``DeviceComm`` (the fused ``GridPlan`` pass): a symmetric device buffer per
  rank mapped by every other rank through CUDA IPC; the native level loop
  computes work-balanced slices on the device and exchanges marks, marking
  statistics, lattice flag words and q rows with put / get kernels over peer
  memory (NVLink / NVSwitch) — no host round trip and no NCCL call inside the
  loop (csrc/ow_comm.cu).  torch.distributed (any backend) only carries the
  64-byte IPC handles once at setup.
* ``Shard`` (the per-function API): the marks of each level travel through
  torch.distributed collectives from the driver's exchange callback.
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist


def _wrap_int32(ptr, n, device):
    """Zero-copy int32 CUDA tensor over n elements of device memory at ptr."""
    if n == 0:
        return torch.zeros(0, dtype=torch.int32, device=device)

    class _Cuda:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<i4", "data": (int(ptr), False), "version": 2}

    return torch.as_tensor(_Cuda(), device=device)


def partition(n, rank, world, weights=None):
    """[lo, hi) slice of n ordered units for ``rank``; balanced by ``weights``
    (a 1-D cumulative-work tensor) when given, else by count."""
    if world <= 1:
        return 0, n
    if weights is None or n == 0:
        per = (n + world - 1) // world
        return min(n, rank * per), min(n, (rank + 1) * per)
    cum = torch.cumsum(weights.to(torch.float64), 0)
    total = float(cum[-1]) if n else 0.0
    cut = torch.tensor([total * r / world for r in range(world + 1)], dtype=torch.float64, device=cum.device)
    idx = torch.searchsorted(cum, cut, right=False).clamp_(0, n).tolist()
    idx[0], idx[-1] = 0, n
    return int(idx[rank]), int(idx[rank + 1])


def gather_slices(local, n, world, group=None, sizes=None):
    """All-gather variable-length contiguous slices (padded to the largest);
    returns the concatenation in rank order, length n.  ``sizes`` (every
    rank's slice length, when the caller knows them) skips the length
    exchange; otherwise the lengths travel in one all-gather and one host
    read.  NCCL gathers device memory directly; under gloo (CPU tests,
    several ranks on one device) the slices are staged through host memory."""
    if local.is_cuda and dist.get_backend(group) == "gloo":
        res, sizes = gather_slices(local.cpu(), n, world, group, sizes)
        return res.to(local.device), sizes
    dev = local.device
    if sizes is None:
        counts = torch.tensor([local.numel()], dtype=torch.int64, device=dev)
        all_counts = torch.empty(world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(all_counts, counts, group=group)
        sizes = all_counts.tolist()  # the one host read of the exchange
    assert sizes[dist.get_rank(group) if world > 1 else 0] == local.numel()
    m = max(max(sizes), 1)
    if local.numel() == m:
        buf = local.contiguous()
    else:
        buf = torch.zeros(m, dtype=local.dtype, device=dev)
        buf[: local.numel()] = local
    out = torch.empty(world * m, dtype=local.dtype, device=dev)
    dist.all_gather_into_tensor(out, buf, group=group)
    if all(sz == m for sz in sizes):
        res = out
    else:
        res = torch.cat([out[r * m: r * m + sizes[r]] for r in range(world)])
    assert n is None or res.numel() == n, (res.numel(), n)
    return res, sizes


class Shard:
    """Shard marking passes across the ranks of ``group`` (default world)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def gather_links(self, flags, cells, q, lo, hi, ncell, n_leaves):
        """All-gather the lattice results of every rank's leaf slice: flag words
        of leaves [lo, hi) and the slice's boundary rows (ascending, so the
        rank-order concatenation is the single-GPU order)."""
        nq = q.shape[1] if q.dim() == 2 else 0
        fsz = [(b - a) * ncell for a, b in (partition(n_leaves, r, self.world) for r in range(self.world))]
        allf, _ = gather_slices(flags[lo * ncell: hi * ncell].contiguous(), n_leaves * ncell, self.world,
                                self.group, sizes=fsz)
        allc, csz = gather_slices(cells, None, self.world, self.group)  # one length exchange for both
        allq, _ = gather_slices(q.reshape(-1), None, self.world, self.group, sizes=[c * nq for c in csz])
        return allf, allc, allq.view(-1, nq)

    def exchange_callback(self, forest):
        """ow_exchange_fn for the native driver: all-gather the marks of the
        level's leaves (each rank marked [lo, hi)) and sum the statistics."""

        def cb(_user, level, d_leaves, n, lo, hi, stats3):
            try:
                ptr = int(d_leaves or 0)
                leaves = _wrap_int32(ptr, n, forest.device)
                idx = leaves.to(torch.int64)
                mine = forest._marks.index_select(0, idx[lo:hi])
                per = (n + self.world - 1) // self.world  # the driver's slices (refine_driver)
                msz = [max(0, min(n, per * (r + 1)) - min(n, per * r)) for r in range(self.world)]
                allm, _ = gather_slices(mine, n, self.world, self.group, sizes=msz)
                forest._marks.index_copy_(0, idx, allm)
                sdev = "cpu" if dist.get_backend(self.group) == "gloo" else forest.device
                tot = torch.tensor([stats3[0], stats3[1], stats3[2]], dtype=torch.int64, device=sdev)
                dist.all_reduce(tot, group=self.group)
                for i, x in enumerate(tot.tolist()):
                    stats3[i] = int(x)
                return 0
            except Exception:  # pragma: no cover - surfaced by the C side as an exchange failure
                import traceback

                traceback.print_exc()
                return 1

        return cb

    def mark_level(self, forest, level, geom, d_spec, bins, grid, mark_fn):
        from .nearwall import MarkStats

        leaves = forest._leaves(level)
        n = int(leaves.numel())
        lo, hi = partition(n, self.rank, self.world)
        st = mark_fn(forest, level, geom, d_spec, bins, grid, leaves=leaves[lo:hi].contiguous())
        if self.world > 1:
            mine = forest.marks.index_select(0, leaves[lo:hi].to(torch.int64))
            msz = [b - a for a, b in (partition(n, r, self.world) for r in range(self.world))]
            allm, _ = gather_slices(mine, n, self.world, self.group, sizes=msz)
            forest.marks.index_copy_(0, leaves.to(torch.int64), allm)
            tot = torch.tensor([st.marked, st.tests, st.evaluated], dtype=torch.int64, device=allm.device)
            dist.all_reduce(tot, group=self.group)
            st = MarkStats(*(int(x) for x in tot.tolist()))
        return st


class DeviceComm:
    """Device-side exchange for the ranks of ``group`` on one node (collective
    constructor: every rank calls it).  ``area_bytes`` bounds the largest
    array one exchange carries (marks: one byte per leaf; lattice: four
    bytes per finest cell, four per (boundary row, direction))."""

    def __init__(self, area_bytes, group=None):
        from . import _lib

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.area_bytes = int(area_bytes)
        dev = _lib.device()
        self._p = C.c_void_p()
        handle = (C.c_uint8 * 64)()
        _lib.call("ow_comm_create", dev.index, self.rank, self.world, self.area_bytes, C.byref(self._p), handle)
        mine = bytes(handle)
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        buf = (C.c_uint8 * (64 * self.world)).from_buffer_copy(b"".join(allh))
        _lib.call("ow_comm_open", self._p, buf)
        dist.barrier(group=group)  # every rank has mapped every buffer before any put

    @property
    def handle(self):
        return self._p

    def status(self):
        """1 when an exchange gave up waiting for a peer (timeout), else 0."""
        from . import _lib

        v = C.c_int64(0)
        _lib.call("ow_comm_status", self._p, C.byref(v))
        return int(v.value)

    def allgather_(self, t, lo, hi):
        """In place: this rank's elements [lo, hi) of the 32-bit CUDA tensor t
        reach every rank (ranks' ranges partition t)."""
        from . import _lib

        assert t.is_cuda and t.element_size() == 4 and t.is_contiguous()
        _lib.call("ow_comm_allgather_u32", _lib.ctx(), self._p, _lib.ptr(t), int(lo), int(hi), t.numel(),
                  _lib.stream())
        return t

    def close(self):
        from . import _lib

        if self._p:
            _lib.lib().ow_comm_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass
