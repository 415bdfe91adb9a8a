"""One geometry-to-grid pass in one native call (``ow_geometry_to_grid``).

The reference runs import -> refine_near_wall as separate Python calls
(cli.py:87-113); each is available here with the reference's signature
(``import_stl``, ``refine_near_wall``, ``build_lattice_links``).  This module
adds the fused B200 path: binary STL records resident in HBM -> validated SoA
geometry -> root grid -> per-level {bins, marking, propagation, refinement}
-> lattice links + q on the finest level, driven from C++ with no Python
between the stages.  Every returned array is an ordinary CUDA tensor: output
buffers are allocated by PyTorch before the call (sized from the previous
pass of the same plan) or, when a size is first learnt on the device, through
an allocation callback.

``GridPlan`` holds everything that does not depend on the geometry (bin grid,
driver parameters, lattice directions, callbacks), so repeated passes — a
time series of geometries, a benchmark loop — pay only for the call itself.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvalidParameterError
from .forest import DEFAULT_MAX_LEVEL, Forest
from .geometry import Aabb, CoordListGeometry
from .geometry import _keys as _geom_keys
from .lattice import LatticeLinks, lattice_directions
from .nearwall import NearWallParams, NearWallResult, _driver_done, _driver_result, _driver_setup

_OUT_DTYPES = (torch.int64, torch.int32, torch.int64, torch.float32)  # OW_OUT_LEAVES, FLAGS, CELLS, Q


@dataclass
class GridPass:
    geometry: CoordListGeometry
    forest: Forest
    result: NearWallResult
    links: LatticeLinks | None
    host: dict | None = None  # pinned host copies of the results (run(host=True))
    reran: bool = False  # the device-resident level loop outgrew the capacity; rerun with host sync
    host_copied: int = 0  # native host copies made (bit 0 forest, bit 2 packed rows, bit 3 deferred)
    done: object = None  # torch.cuda.Event of deferred host copies (run(defer=True)); None: already ordered
    device_sized: int = 0  # 1: one device-sized pass (single readback); 2: it fell back to the synchronous pass

    def wait(self):
        """Block until the host copies of this pass are complete (the
        deferred copies' event, else the current stream)."""
        if self.done is not None:
            self.done.synchronize()
        else:
            torch.cuda.current_stream().synchronize()

    def host_q(self) -> np.ndarray:
        """Dense (boundary rows, Q) float32 q from the packed host copy (-1 where
        the link misses); valid once the stream is synchronised."""
        h = self.host
        return unpack_q(h["flags"].numpy().view(np.uint32), h["q_packed"].numpy(), self.links.q.shape[1])


class PendingGridPass:
    """A submitted pass (``GridPlan.run_async``); ``result()`` waits for it
    and returns its ``GridPass`` (the same object on every call; errors of
    the pass are raised there)."""

    def __init__(self, plan, state):
        self._plan = plan
        self._state = state
        self._ticket = 0
        self._gp = None
        self._err = None

    def result(self) -> GridPass:
        if self._gp is None and self._err is None:
            plan = self._plan
            if plan._pending is self:
                plan._pending = None
            try:
                self._gp = plan._finish(self._state, self._ticket)
            except Exception as e:
                self._err = e
            self._state = None
        if self._err is not None:
            raise self._err
        return self._gp


class _outside_message:
    """Re-raise the native 'outside the forest domain' error with the
    geometry's extent (the reference's message)."""

    def __init__(self, out, dim):
        self.out, self.dim = out, dim

    def __enter__(self):
        return self

    def __exit__(self, et, ev, tb):
        if et is InvalidParameterError and self.out.outside_domain:
            lo = np.array(self.out.faces.bbox_min[: self.dim], np.float32).astype(np.float64)
            hi = np.array(self.out.faces.bbox_max[: self.dim], np.float32).astype(np.float64)
            raise InvalidParameterError(
                f"geometry spans {lo.tolist()}..{hi.tolist()}, outside the forest domain") from None
        return False


def unpack_q(row_flags: np.ndarray, q_packed: np.ndarray, nq: int) -> np.ndarray:
    """Packed boundary rows -> dense q: row r's set bits of ``row_flags[r]``, in
    ascending direction order, take the next entries of ``q_packed``."""
    bits = ((row_flags[:, None] >> np.arange(nq, dtype=np.uint32)) & 1).astype(bool)
    q = np.full(bits.shape, -1.0, np.float32)
    q[bits] = q_packed[: int(bits.sum())]
    return q


class GridPlan:
    """Reusable setup of ``geometry_to_grid`` for one (domain, root grid,
    NearWallParams, lattice)."""

    def __init__(self, domain: Aabb, root_dims, params: NearWallParams, lattice: str | None = "D3Q19",
                 capacity=None, max_level=DEFAULT_MAX_LEVEL, reuse_outputs=False, comm=None, stage_times=True):
        """``reuse_outputs=True``: every pass writes into the same device
        arrays (forest, bins, links), so a pass's results are valid until the
        next ``run`` — for loops that consume each pass before the next
        (benchmarks, time series); all work is still recomputed.  The
        returned LatticeLinks object itself is reused while the output
        storage and sizes are unchanged (``gp_next.links is gp_prev.links``).

        ``comm`` (a ``parallel.DeviceComm``, one rank per GPU): the pass is
        sharded — work-balanced leaf slices per marking pass and equal
        finest-leaf slices for the lattice links, exchanged over peer memory
        inside the native call — and every rank returns the whole result.

        ``stage_times=False``: no CUDA events between the level loop's stages
        (an event between two kernels stops their programmatic overlap);
        ``NearWallResult.timings`` then read 0 ms.  Settable per pass."""
        self.domain = domain if isinstance(domain, Aabb) else Aabb(*domain)
        self.dim = self.domain.dim
        self.root_dims = tuple(int(v) for v in np.asarray(root_dims).reshape(-1))
        self.params = params
        self.lattice = lattice
        self.max_level = max_level
        r = int(np.prod(self.root_dims))
        self.capacity = int(capacity or 32 * r)
        self.dev = _lib.device()
        self.dirs = None
        if lattice:
            self.dirs = lattice_directions(lattice)
            if self.dirs.shape[1] != self.dim:
                raise InvalidParameterError(f"lattice {lattice} does not match a {self.dim}D domain")
        self._est = [0, 0, 0, 0]  # output bytes of the last pass (preallocation estimate)
        self._est_blocks = 0      # forest blocks / boundary rows of the last pass (host buffers)
        self._est_rows = 0
        self._est_links = 0
        self._outs = {}
        self._hbuf = None
        self._coords = None
        self._links = self._links_key = None
        self._gp = None  # the call's parameter struct, reused while nothing static changes
        self._gp_key = None
        self.reuse = bool(reuse_outputs)
        self.comm = comm if comm is not None and comm.world > 1 else None
        self.stage_times = bool(stage_times)
        self._forest = None
        self._setup = None  # (n_faces, _driver_setup result): the parts that depend on n_faces only
        self._gp0 = _lib.G2GParamsC()  # static fields of the call's parameter struct
        self._done = None  # torch.cuda.Event: the last pass's deferred host copies
        self._pending = None  # the plan's submitted, unfinished pass (run_async)
        self._dev_rows = self._dev_qp = None  # device staging of the packed rows (deferred passes)
        if self.dirs is not None:
            self._gp0.lattice_q = len(self.dirs)
            for i, v in enumerate(self.dirs.reshape(-1)):
                self._gp0.lattice_dirs[i] = int(v)

        def alloc(_user, what, nbytes, out_p):  # noqa: ARG001
            try:
                t = self._new_out(int(what), int(nbytes))
                out_p[0] = t.data_ptr() if t.numel() else None
                return 0
            except Exception:  # pragma: no cover - reported by the C side as a failed allocation
                return 1

        self._alloc_cb = _lib.ALLOC_FN(alloc)
        if self.dirs is not None:
            self._gp0.alloc = self._alloc_cb

    def __del__(self):
        # a submitted pass holds a ticket on the context: finish it (its
        # results are dropped with the plan)
        pend = getattr(self, "_pending", None)
        if pend is not None:
            try:
                pend.result()
            except Exception:  # pragma: no cover - nothing to report to at collection time
                pass

    def _new_out(self, what, nbytes):
        dt = _OUT_DTYPES[what]
        t = torch.empty(max(nbytes, 0) // (8 if dt in (torch.int64,) else 4), dtype=dt, device=self.dev)
        self._outs[what] = t
        return t

    def _pinned(self, dtype, n):
        return torch.empty(max(int(n), 1), dtype=dtype, pin_memory=True)

    def run(self, records: torch.Tensor | None = None, n_faces: int | None = None,
            geometry: CoordListGeometry | None = None, host: bool = False, defer: bool = False) -> GridPass:
        """One pass, returned complete: ``run_async(...).result()``."""
        return self.run_async(records, n_faces, geometry, host, defer).result()

    def run_async(self, records: torch.Tensor | None = None, n_faces: int | None = None,
                  geometry: CoordListGeometry | None = None, host: bool = False,
                  defer: bool = False) -> "PendingGridPass":
        """Binary STL records (device uint8, 50 bytes per face, after the
        84-byte header) — or an existing ``geometry`` — to a refined forest and
        its finest-level lattice links.

        ``host=True`` also returns pinned host copies of the results
        (``GridPass.host``: forest arrays, boundary cells (uint32 ids as int32
        views), their flag words and the packed q of the set bits): the forest
        arrays stream to the host on a side stream while the lattice work
        runs; the boundary rows travel packed ((8 + 4 popc) bytes per row
        instead of 8 + 4 Q) and ``GridPass.host_q()`` expands them to the
        dense (rows, Q) array.

        ``defer=True`` (with ``host=True``): every host copy of the pass runs
        on the library's copy stream and the current stream does not wait for
        them, so they overlap whatever is enqueued next (another plan's pass:
        alternate two plans to stream geometries); ``GridPass.wait()`` blocks
        until they are done.  The plan's next pass waits for them on the
        device before it rewrites its outputs.

        ``run_async`` submits the pass and returns a ``PendingGridPass``
        without waiting for the device (when the pass can run device-sized:
        from a plan's second pass on, without stage-timing events);
        ``.result()`` waits for it and returns the ``GridPass``.  Passes of
        other plans may be submitted in between, so a stream of geometries
        through two alternating plans keeps the GPU fed while the host
        finishes the previous pass.  A plan's pending pass is finished before
        its next one is submitted."""
        if self._pending is not None:
            self._pending.result()
        if geometry is None and records is None:
            raise InvalidParameterError("geometry_to_grid needs STL records or a geometry")
        dim = self.dim
        if geometry is not None:
            if geometry.dim != dim:
                raise InvalidParameterError(f"geometry is {geometry.dim}D but the domain is {dim}D")
            coords = geometry.coords
        else:
            if dim != 3:
                raise InvalidParameterError("binary STL records are 3D")
            c = self._coords if self.reuse else None  # (reuse_outputs: one geometry buffer per plan)
            if c is None or c.shape[2] != int(n_faces):
                c = torch.empty((3, 3, int(n_faces)), dtype=torch.float32, device=self.dev)
                if self.reuse:
                    self._coords = c
            coords = c
        nf = int(coords.shape[2])
        forest = self._forest
        if forest is not None and forest.capacity >= self.capacity:
            forest._reset_for_pass()
        else:
            forest = Forest(self.domain, self.root_dims, max_level=self.max_level, capacity=self.capacity,
                            _init_root=False)
            if self.reuse:
                self._forest = forest
        if self._setup is None or self._setup[0] != nf:
            self._setup = (nf, _driver_setup(forest, nf, self.params, True, self.comm))
        st = self._setup[1]
        if not self.reuse and st["bins_t"] is not None:  # fresh bin buffers for this pass's result
            st = dict(st)
            st["bins_t"] = tuple(torch.empty_like(t) for t in st["bins_t"])
        if self.reuse and self._gp is not None and self._gp_key is st:
            gp = self._gp  # steady state: same setup struct, output buffers checked below
        else:
            gp = _lib.G2GParamsC.from_buffer_copy(self._gp0)
            gp.nw = st["p"]
            if self.reuse:
                self._gp, self._gp_key = gp, st
        if not self.reuse:
            self._outs = {}
        if self.dirs is not None:
            for what in range(4):  # tensors sized from the last pass: no callback in steady state
                if self._est[what]:
                    t = self._outs.get(what)
                    if t is None or t.numel() * t.element_size() < self._est[what]:
                        t = self._new_out(what, self._est[what] + self._est[what] // 8 + 64)
                    gp.out_buf[what] = t.data_ptr()
                    gp.out_cap[what] = t.numel() * t.element_size()
        hbuf = None
        if not host and gp.host_level:  # a reused struct from a host=True pass: no host copies now
            gp.host_level = gp.host_cells = gp.host_q = gp.host_rows = gp.host_q_packed = None
            gp.host_block_cap = gp.host_row_cap = gp.host_link_cap = 0
        if host:
            # pinned host buffers owned by the plan and reused by every pass (a
            # pass's host results stay valid until the next host=True pass)
            nbk = max(self._est_blocks + self._est_blocks // 4 + 1024, 1024)
            nrow = max(self._est_rows + self._est_rows // 4 + 1024, 1024)
            nlink = max(self._est_links + self._est_links // 4 + 4096, 4096)
            hb = self._hbuf
            if (hb is None or hb["level"].numel() < nbk or hb["rows"].numel() < 2 * nrow
                    or hb["q_packed"].numel() < nlink):
                hb = dict(level=self._pinned(torch.int16, nbk), parent=self._pinned(torch.int32, nbk),
                          first_child=self._pinned(torch.int32, nbk), marks=self._pinned(torch.int8, nbk),
                          coords=[self._pinned(torch.int32, nbk) for _ in range(dim)],
                          rows=self._pinned(torch.int32, 2 * nrow), q_packed=self._pinned(torch.float32, nlink))
                self._hbuf = hb
            hbuf = dict(hb)
            nbk, nrow = hb["level"].numel(), hb["rows"].numel() // 2
            gp.host_level, gp.host_parent = hbuf["level"].data_ptr(), hbuf["parent"].data_ptr()
            gp.host_first_child, gp.host_marks = hbuf["first_child"].data_ptr(), hbuf["marks"].data_ptr()
            for a in range(dim):
                gp.host_coord[a] = hbuf["coords"][a].data_ptr()
            gp.host_block_cap = nbk
            gp.host_row_cap = nrow
            gp.host_rows, gp.host_q_packed = hbuf["rows"].data_ptr(), hbuf["q_packed"].data_ptr()
            gp.host_link_cap = hb["q_packed"].numel()
        if self._done is not None or (host and defer):
            if self._done is None:
                self._done = torch.cuda.Event()
                self._done.record()  # (creates the CUDA event; completes at once)
            gp.copy_done = self._done.cuda_event
        gp.dev_rows = gp.dev_q_packed = None
        gp.dev_row_cap = gp.dev_link_cap = 0
        if host and defer:
            nrow, nlink = gp.host_row_cap, gp.host_link_cap
            if self._dev_rows is None or self._dev_rows.numel() < 2 * nrow or self._dev_qp.numel() < nlink:
                self._dev_rows = torch.empty(2 * nrow, dtype=torch.int32, device=self.dev)
                self._dev_qp = torch.empty(nlink, dtype=torch.float32, device=self.dev)
            gp.dev_rows, gp.dev_q_packed = self._dev_rows.data_ptr(), self._dev_qp.data_ptr()
            gp.dev_row_cap, gp.dev_link_cap = nrow, nlink
        gp.no_stage_times = 0 if self.stage_times else 1
        out = _lib.G2GResultC()
        g, bins_t = st["g"], st["bins_t"]
        v = forest.view()
        args = (_lib.ptr(coords), nf, next(_geom_keys), C.byref(v), C.byref(g) if g is not None else None,
                C.byref(gp), _lib.ptr(bins_t[0]) if bins_t else None, st["cap"],
                _lib.ptr(bins_t[1]) if bins_t else None, _lib.ptr(bins_t[2]) if bins_t else None,
                C.byref(out), _lib.stream())
        ticket = C.c_int64(0)
        pending = PendingGridPass(self, (forest, v, out, st, gp, g, bins_t, coords, geometry, hbuf, host, args))
        with _outside_message(out, dim):
            try:
                _lib.call("ow_geometry_to_grid_submit", _lib.ctx(), _lib.ptr(records) if geometry is None else None,
                          *args, C.byref(ticket))
            except Exception:
                _driver_done(forest, out.nw)
                raise
        pending._ticket = int(ticket.value)
        if pending._ticket == 0 or self.stage_times:  # (stage events live in the context: finish now)
            pending.result()
        else:
            self._pending = pending
        return pending

    def _finish(self, state, ticket):
        forest, v, out, st, gp, g, bins_t, coords, geometry, hbuf, host, args = state
        dim = self.dim
        if ticket:
            with _outside_message(out, dim):
                try:
                    _lib.call("ow_geometry_to_grid_finish", _lib.ctx(), ticket, *args)
                finally:
                    _driver_done(forest, out.nw)
        else:
            _driver_done(forest, out.nw)
        geom = geometry if geometry is not None else CoordListGeometry._validated(dim, coords, out.faces)
        result = _driver_result(forest, self.params, st, out.nw)
        links = None
        if self.dirs is not None:
            nq, nl, nb = len(self.dirs), int(out.n_finest_leaves), int(out.n_boundary)
            ncell = 4 ** dim
            need = (8 * nl, 4 * nl * ncell, 8 * nb, 4 * nb * nq)
            self._est = list(need)
            self._est_rows = nb
            self._est_links = int(out.n_links)
            o = self._outs
            key = (o[0], o[1], o[2], o[3], nl, nb, int(out.finest_level))
            lk = self._links_key
            if self.reuse and lk is not None and all(a is b if isinstance(a, torch.Tensor) else a == b
                                                     for a, b in zip(key, lk)):
                links = self._links  # same storage and sizes as the last pass: the same views
            else:
                links = LatticeLinks(lattice=self.lattice, level=int(out.finest_level), leaves=o[0][:nl],
                                     flags=o[1][: nl * ncell], cells=o[2][:nb], q=o[3][: nb * nq].view(nb, nq))
                if self.reuse:
                    self._links, self._links_key = links, key
        self._est_blocks = forest.n_blocks
        # size the next pass's forest from this one: device refinement then never
        # overflows into the host fallback (which grows the arrays with syncs)
        self.capacity = max(self.capacity, forest.n_blocks + forest.n_blocks // 4)
        hres = None
        if host:
            hres = self._host_results(hbuf, int(out.host_copied), forest, links, int(out.n_links))
        done = self._done if int(out.host_copied) & 8 else None
        return GridPass(geom, forest, result, links, hres, bool(out.reran), int(out.host_copied), done,
                        int(out.device_sized))

    def _host_results(self, hbuf, copied, forest, links, n_links):
        """Pinned host copies (the C side streamed whatever fit; the rest is
        copied here).  Valid once the current stream is synchronised."""
        n = forest.n_blocks
        if not copied & 1:
            for name, t in (("level", forest._level_t), ("parent", forest._parent_t),
                            ("first_child", forest._first_child_t), ("marks", forest._marks)):
                hbuf[name] = self._pinned(t.dtype, n)
                hbuf[name][:n].copy_(t[:n], non_blocking=True)
            hbuf["coords"] = [self._pinned(torch.int32, n) for _ in range(self.dim)]
            for a in range(self.dim):
                hbuf["coords"][a][:n].copy_(forest._coord[a][:n], non_blocking=True)
        res = dict(level=hbuf["level"][:n], parent=hbuf["parent"][:n], first_child=hbuf["first_child"][:n],
                   marks=hbuf["marks"][:n], coords=[c[:n] for c in hbuf["coords"]])
        if links is not None:
            nb, nq = links.n_boundary, links.q.shape[1]
            if not copied & 4:  # the buffers did not fit (first pass of a plan): pack with torch
                hit = links.q >= 0
                rflags = (hit.to(torch.int64) << torch.arange(nq, device=hit.device)).sum(1).to(torch.int32)
                rows = torch.stack([links.cells.to(torch.int32), rflags], 1).reshape(-1)
                hbuf["rows"], hbuf["q_packed"] = self._pinned(torch.int32, 2 * nb), self._pinned(torch.float32, n_links)
                hbuf["rows"][: 2 * nb].copy_(rows, non_blocking=True)
                hbuf["q_packed"][:n_links].copy_(links.q[hit], non_blocking=True)
            rows = hbuf["rows"][: 2 * nb].view(nb, 2)  # (cell id as uint32, flag word) per row
            res["cells"], res["flags"] = rows[:, 0], rows[:, 1]
            res["q_packed"] = hbuf["q_packed"][:n_links]
        return res


def geometry_to_grid(records: torch.Tensor | None, n_faces: int | None, domain: Aabb, root_dims,
                     params: NearWallParams, lattice: str | None = "D3Q19", capacity=None,
                     geometry: CoordListGeometry | None = None, max_level=DEFAULT_MAX_LEVEL) -> GridPass:
    """One-shot ``GridPlan(...).run(...)``."""
    return GridPlan(domain, root_dims, params, lattice, capacity=capacity, max_level=max_level).run(
        records, n_faces, geometry)
