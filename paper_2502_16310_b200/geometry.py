"""Boundary geometry: primitives, text / STL import, coordinate lists on the GPU.

Mirrors octowall/geometry.py (same names, arguments, dtypes and errors).  The
coordinate-list form lives in HBM as a float32 (verts_per_face, dim, n_faces)
tensor — the reference's structure-of-arrays layout (geometry.py:94-124) —
and every per-face pass over it (binary-STL transpose, index gather,
degeneracy test, bounding box) is a sm_100a kernel in libowb200.so.  Text
primitives are parsed on the host and generated in float64 then rounded by
NumPy (bit-identical vertices); ASCII STL is parsed by the native host parser
(ow_parse_ascii_stl: parallel tokenising and conversion, the reference's
error messages and line numbers).
"""

from __future__ import annotations

import ctypes as C
import itertools
import threading
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import GeometryParseError, InvalidParameterError

_keys = itertools.count(1)


def _require(ok, message):
    """Raise InvalidParameterError(message) unless ok; ``message`` may be a
    callable so array formatting only happens on failure."""
    if not ok:
        raise InvalidParameterError(message() if callable(message) else message)


def as_point(p, dim):
    """float64 point of exactly ``dim`` finite components (geometry.py:16-25)."""
    a = np.asarray(p, dtype=np.float64).ravel()
    _require(a.size == dim, f"expected a {dim}-component point, got {a.size}")
    _require(bool(np.isfinite(a).all()), lambda: f"point has non-finite components: {a}")
    return a


@dataclass
class Aabb:
    """Axis-aligned box with float64 corners (geometry.py:28-55)."""

    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        lo, hi = (np.asarray(c, dtype=np.float64).ravel() for c in (self.min, self.max))
        _require(lo.shape == hi.shape, "aabb min/max dimension mismatch")
        _require(bool(np.isfinite(lo).all() and np.isfinite(hi).all()), "aabb has non-finite corners")
        _require(not bool((lo > hi).any()), lambda: f"aabb min {lo} exceeds max {hi}")
        self.min, self.max = lo, hi

    @property
    def dim(self):
        return int(self.min.size)

    @property
    def extent(self):
        return self.max - self.min

    def contains(self, p, tol=0.0):
        q = np.asarray(p, dtype=np.float64)
        return bool(((q >= self.min - tol) & (q <= self.max + tol)).all())


@dataclass
class IndexedGeometry:
    """Shared-vertex mesh on the host: vertices (V, dim) float32, faces
    (F, dim) int32 vertex indices (geometry.py:58-91)."""

    dim: int
    vertices: np.ndarray
    faces: np.ndarray

    def __post_init__(self):
        _require(self.dim in (2, 3), f"dim must be 2 or 3, got {self.dim}")
        v = np.asarray(self.vertices, dtype=np.float32).reshape(-1, self.dim)
        f = np.asarray(self.faces, dtype=np.int32).reshape(-1, self.dim)
        _require(bool(np.isfinite(v).all()), "geometry has non-finite vertex coordinates")
        if f.size:
            _require(0 <= int(f.min()) and int(f.max()) < len(v), "face index out of range")
            rep = f[:, 0] == f[:, 1]
            if self.dim == 3:
                rep |= (f[:, 0] == f[:, 2]) | (f[:, 1] == f[:, 2])
            _require(not bool(rep.any()), "face has repeated vertex indices")
        self.vertices, self.faces = v, f

    @property
    def n_faces(self):
        return len(self.faces)

    @classmethod
    def empty(cls, dim):
        return cls(dim, np.zeros((0, dim), np.float32), np.zeros((0, dim), np.int32))


class CoordListGeometry:
    """Per-face vertex coordinates, float32 (verts_per_face=dim, dim, n_faces) in HBM.

    ``coords`` is a CUDA tensor; NumPy input is uploaded.  ``coords_numpy()``
    returns a host copy.  Geometry is immutable once built (as in the
    reference), which lets the device caches key on ``key``.
    """

    def __init__(self, dim, coords):
        if dim not in (2, 3):
            raise InvalidParameterError(f"dim must be 2 or 3, got {dim}")
        self.dim = int(dim)
        if isinstance(coords, torch.Tensor):
            t = coords.to(device=_lib.device(), dtype=torch.float32).contiguous()
        else:
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(coords, dtype=np.float32))).to(_lib.device())
        if t.dim() != 3 or t.shape[0] != dim or t.shape[1] != dim:
            raise InvalidParameterError(
                f"coords must have shape (verts_per_face={dim}, dim={dim}, n_faces), got {tuple(t.shape)}")
        self.coords = t
        self.key = next(_keys)
        self._summary = None
        if self.summary().first_nonfinite >= 0:
            raise InvalidParameterError("geometry has non-finite coordinates")

    @classmethod
    def _validated(cls, dim, coords, summary):
        """Wrap device coords whose face summary the library already computed."""
        g = cls.__new__(cls)
        g.dim, g.coords, g.key, g._summary = int(dim), coords, next(_keys), summary
        return g

    @property
    def n_faces(self):
        return int(self.coords.shape[2])

    def face(self, k):
        return self.coords[:, :, k].cpu().numpy()

    def coords_numpy(self):
        return self.coords.cpu().numpy()

    def summary(self):
        """FaceSummary of one GPU pass: first degenerate / non-finite face, bbox, |max|."""
        if self._summary is None:
            s = _lib.FaceSummary()
            _lib.call("ow_face_check", _lib.ctx(), self.dim, _lib.ptr(self.coords), self.n_faces, C.byref(s),
                      _lib.stream())
            self._summary = s
        return self._summary

    def __repr__(self):
        return f"CoordListGeometry(dim={self.dim}, n_faces={self.n_faces}, device={self.coords.device})"


# ---------------------------------------------------------------------------
# primitives (host, float64 -> float32 like geometry.py:127-192)
# ---------------------------------------------------------------------------


def generate_circle(center, radius, n_edges):
    center = as_point(center, 2)
    if n_edges < 3:
        raise InvalidParameterError(f"a circle needs at least 3 edges, got {n_edges}")
    if radius <= 0:
        raise InvalidParameterError(f"circle radius must be positive, got {radius}")
    k = np.arange(n_edges)
    ang = 2.0 * np.pi * k / n_edges
    xy = np.empty((n_edges, 2))
    xy[:, 0] = center[0] + radius * np.cos(ang)
    xy[:, 1] = center[1] + radius * np.sin(ang)
    faces = np.stack([k, (k + 1) % n_edges], axis=1).astype(np.int32)
    return IndexedGeometry(2, xy.astype(np.float32), faces)


def generate_sphere(center, radius, n_lat, n_lon):
    """Lat-lon tessellation: pole fans + two triangles per quad, outward winding."""
    center = as_point(center, 3)
    if n_lat < 2:
        raise InvalidParameterError(f"sphere needs n_lat >= 2, got {n_lat}")
    if n_lon < 3:
        raise InvalidParameterError(f"sphere needs n_lon >= 3, got {n_lon}")
    if radius <= 0:
        raise InvalidParameterError(f"sphere radius must be positive, got {radius}")
    phi = 2.0 * np.pi * np.arange(n_lon) / n_lon
    rings = np.empty((n_lat - 1, n_lon, 3))
    for r in range(n_lat - 1):
        th = np.pi * (r + 1) / n_lat  # scalar libm path, as the reference evaluates it
        st = radius * np.sin(th)
        rings[r, :, 0] = center[0] + st * np.cos(phi)
        rings[r, :, 1] = center[1] + st * np.sin(phi)
        rings[r, :, 2] = center[2] + radius * np.full(n_lon, np.cos(th))
    verts = np.concatenate(
        [(center + np.array([0.0, 0.0, radius]))[None], rings.reshape(-1, 3),
         (center + np.array([0.0, 0.0, -radius]))[None]]).astype(np.float32)
    j = np.arange(n_lon)
    jn = (j + 1) % n_lon
    start = lambda k: 1 + (k - 1) * n_lon  # noqa: E731
    blocks = [np.stack([np.zeros(n_lon, np.int64), start(1) + j, start(1) + jn], 1)]
    for k in range(1, n_lat - 1):
        a, b = start(k), start(k + 1)
        quad = np.stack([np.stack([a + j, b + j, b + jn], 1), np.stack([a + j, b + jn, a + jn], 1)], 1)
        blocks.append(quad.reshape(-1, 3))
    south = len(verts) - 1
    last = start(n_lat - 1)
    blocks.append(np.stack([np.full(n_lon, south), last + jn, last + j], 1))
    return IndexedGeometry(3, verts, np.concatenate(blocks).astype(np.int32))


def append_geometry(parts):
    """One indexed mesh from several: vertices stacked, each part's face
    indices shifted by the vertices that precede it (geometry.py:195-208)."""
    parts = list(parts)
    if not parts:
        raise InvalidParameterError("nothing to append")
    dims = {p.dim for p in parts}
    if len(dims) != 1:
        raise InvalidParameterError("cannot append geometries of mixed dimension")
    if len(parts) == 1:
        return parts[0]
    shift = np.cumsum([0] + [len(p.vertices) for p in parts[:-1]])
    return IndexedGeometry(parts[0].dim, np.concatenate([p.vertices for p in parts]),
                           np.concatenate([p.faces + k for p, k in zip(parts, shift)]))


def _integer(token):
    """A float()-parsable token with an integral value (counts may be written 1e3)."""
    v = float(token)
    if not v.is_integer():
        raise ValueError(token)
    return int(v)


# primitive keyword -> (argument names, trailing integral counts, builder(reals, counts))
_PRIMITIVES = {
    "circle": (("cx", "cy", "r", "n_edges"), 1,
               lambda x, n: generate_circle(x[:2], x[2], n[0])),
    "sphere": (("cx", "cy", "cz", "r", "n_lat", "n_lon"), 2,
               lambda x, n: generate_sphere(x[:3], x[3], n[0], n[1])),
}


def _primitive_of(body, path, ln):
    kind, *args = body.split()
    kind = kind.lower()
    spec = _PRIMITIVES.get(kind)
    if spec is None:
        raise GeometryParseError(f"unknown primitive {kind!r}", path, ln)
    names, n_counts, build = spec
    if len(args) != len(names):
        raise GeometryParseError(f"{kind} takes {len(names)} values: {' '.join(names)}", path, ln)
    try:
        reals = [float(a) for a in args[: len(names) - n_counts]]
        counts = [_integer(a) for a in args[len(names) - n_counts:]]
        return build(reals, counts)
    except ValueError:
        raise GeometryParseError(f"cannot parse numbers in {body!r}", path, ln) from None
    except InvalidParameterError as e:
        raise GeometryParseError(str(e), path, ln) from None


def parse_text_primitives(text, path=None, dim=None):
    """Primitive description text -> IndexedGeometry (geometry.py:211-252):
    one primitive per line (``circle cx cy r n_edges`` in 2D, ``sphere cx cy
    cz r n_lat n_lon`` in 3D), ``#`` comments, parts concatenated; an empty
    description gives an empty geometry of dimension ``dim`` (default 2)."""
    bodies = ((ln, raw.partition("#")[0].strip()) for ln, raw in enumerate(text.splitlines(), start=1))
    parts = [_primitive_of(body, path, ln) for ln, body in bodies if body]
    if not parts:
        return IndexedGeometry.empty(2 if dim is None else dim)
    out = append_geometry(parts)
    if dim is not None and dim != out.dim:
        raise GeometryParseError(f"file holds {out.dim}D primitives but a {dim}D run was requested", path)
    return out


def import_text_primitives(path, dim=None):
    """Primitive file -> IndexedGeometry (geometry.py:211-252)."""
    try:
        with open(path, encoding="utf-8") as f:
            text = f.read()
    except OSError as e:
        raise GeometryParseError(str(e), path=path) from None
    return parse_text_primitives(text, path=path, dim=dim)


_staging = threading.local()


def _to_device(a: np.ndarray, slot: int, dev) -> torch.Tensor:
    """Host array -> device tensor through a reusable pinned staging buffer
    (per thread and slot), stream-ordered and without a host synchronisation
    (a pageable copy would wait for the device); the buffer is refilled only
    after its previous copy has completed."""
    bufs = getattr(_staging, "bufs", None)
    if bufs is None:
        bufs = _staging.bufs = {}
    a = np.ascontiguousarray(a)
    ent = bufs.get(slot)
    if ent is None or ent[0].numel() < a.nbytes:
        ent = (torch.empty(max(a.nbytes, 1 << 16), dtype=torch.uint8, pin_memory=True), torch.cuda.Event())
        bufs[slot] = ent
    else:
        ent[1].synchronize()
    buf, ev = ent
    host = buf[: a.nbytes].numpy()
    host[:] = a.reshape(-1).view(np.uint8)
    out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device=dev)
    out.view(-1).view(torch.uint8).copy_(buf[: a.nbytes], non_blocking=True)
    ev.record()
    return out


def index_to_coords(g: IndexedGeometry) -> CoordListGeometry:
    """Indexed mesh -> device coordinate list; pure gather on the GPU (the
    vertices and faces go host -> device stream-ordered, no host wait)."""
    dev = _lib.device()
    n = g.n_faces
    out = torch.empty((g.dim, g.dim, n), dtype=torch.float32, device=dev)
    if n:
        v = _to_device(g.vertices, 0, dev)
        fc = _to_device(g.faces, 1, dev)
        _lib.call("ow_index_to_coords", _lib.ctx(), g.dim, _lib.ptr(v), _lib.ptr(fc), n, _lib.ptr(out), _lib.stream())
    return CoordListGeometry(g.dim, out)


def validate_faces(g: CoordListGeometry):
    """Reject degenerate faces (FP64 test on the GPU, geometry.py:276-299)."""
    if g.n_faces == 0:
        return
    bad = g.summary().first_degenerate
    if bad >= 0:
        if g.dim == 2:
            raise InvalidParameterError(f"degenerate edge (identical endpoints) at face {bad}")
        raise InvalidParameterError(f"degenerate triangle (zero area) at face {bad}")


def bounding_box(g: CoordListGeometry) -> Aabb:
    if g.n_faces == 0:
        raise InvalidParameterError("bounding box of empty geometry")
    s = g.summary()
    return Aabb(np.array(s.bbox_min[: g.dim], np.float32).astype(np.float64),
                np.array(s.bbox_max[: g.dim], np.float32).astype(np.float64))


# ---------------------------------------------------------------------------
# STL
# ---------------------------------------------------------------------------
_HEADER = 80
_RECORD = 50


def _binary_size_consistent(data):
    if len(data) < _HEADER + 4:
        return False
    (n,) = struct.unpack_from("<I", data, _HEADER)
    return len(data) == _HEADER + 4 + n * _RECORD


def stl_records_to_coords(records: torch.Tensor, n_faces: int) -> CoordListGeometry:
    """Device bytes of 50-byte STL records -> CoordListGeometry (GPU transpose)."""
    out = torch.empty((3, 3, n_faces), dtype=torch.float32, device=records.device)
    if n_faces:
        _lib.call("ow_stl_binary_to_soa", _lib.ctx(), _lib.ptr(records), n_faces, _lib.ptr(out), _lib.stream())
    return CoordListGeometry(3, out)


def _binary_n(data, path):
    if len(data) < _HEADER + 4:
        raise GeometryParseError("binary STL shorter than header + facet count", path=path)
    (n,) = struct.unpack_from("<I", data, _HEADER)
    need = _HEADER + 4 + n * _RECORD
    if len(data) < need:
        raise GeometryParseError(f"binary STL truncated: {n} facets need {need} bytes, file has {len(data)}",
                                 path=path)
    return n


def _parse_binary(data, path):
    n = _binary_n(data, path)
    raw = torch.frombuffer(bytearray(data[_HEADER + 4:_HEADER + 4 + n * _RECORD]), dtype=torch.uint8) if n else \
        torch.zeros(0, dtype=torch.uint8)
    return stl_records_to_coords(raw.to(_lib.device(), non_blocking=False), n)


_STL_KEYWORDS = ("solid", "normal", "outer", "loop", "vertex", "endloop", "endfacet")  # err[4] of the C ABI


def _ascii_tokens(data, path):
    """Non-ASCII input: valid UTF-8 is re-spelled as an ASCII token stream
    with the same tokens per line (str.split / str.splitlines semantics); a
    token float() accepts becomes repr(float), any other non-ASCII token a
    placeholder.  Returns (ascii bytes, {offset: original token})."""
    try:
        text = data.decode("utf-8", errors="strict")
    except UnicodeDecodeError:
        raise GeometryParseError("not valid ASCII STL text", path=path) from None
    out, orig, off = [], {}, 0
    for line in text.splitlines():
        for tok in line.split():
            rep = tok
            if not tok.isascii():
                try:
                    rep = repr(float(tok))
                except ValueError:
                    rep = "?"
                orig[off] = tok
            out.append(rep + " ")
            off += len(rep) + 1
        out.append("\n")
        off += 1
    return "".join(out).encode("ascii"), orig


def _parse_ascii(data, path):
    """ASCII STL -> CoordListGeometry (geometry.py:349-412)."""
    return CoordListGeometry(3, np.ascontiguousarray(np.transpose(ascii_stl_triangles(data, path), (1, 2, 0))))


def ascii_stl_triangles(data, path=None):
    """ASCII STL bytes -> (n, 3, 3) float32 triangles on the host, through
    the native parser (ow_parse_ascii_stl), which also finds the error the
    reference reports (message and line, geometry.py:349-412)."""
    data = bytes(data)
    buf, orig = (data, {}) if data.isascii() else _ascii_tokens(data, path)
    cap = len(buf) // 64 + 1  # a facet takes more than 64 bytes of text
    tris = np.empty((cap, 3, 3), np.float32)
    n = C.c_int64(0)
    err = (C.c_int64 * 5)()
    st = _lib.lib().ow_parse_ascii_stl(buf, len(buf), tris.ctypes.data_as(C.c_void_p), cap, C.byref(n), err)
    if st == _lib.OW_OK:
        return tris[: n.value]
    if st != _lib.OW_ERR_PARSE:
        _lib.check(st)
    code, line, off, length, kw = (int(v) for v in err)
    tok = orig.get(off, buf[off:off + length].decode("ascii"))
    line = line if line > 0 else None
    if code == 1:
        msg = "unexpected end of file"
    elif code == 2:
        msg = f"expected {_STL_KEYWORDS[kw]!r}, got {tok!r}"
    elif code == 3:
        msg = f"expected a number, got {tok!r}"
    elif code == 4:
        msg = f"expected 'facet' or 'endsolid', got {tok!r}"
    elif code == 5:
        msg = f"unexpected {tok!r} after endsolid"
    else:
        raise GeometryParseError(f"ASCII STL parser failed (code {code})", path=path)
    raise GeometryParseError(msg, path, line)


def import_stl_bytes(data, path=None) -> CoordListGeometry:
    """ASCII / binary autodetect exactly like geometry.py:331-339."""
    if data.lstrip()[:5] == b"solid":
        try:
            return _parse_ascii(data, path)
        except GeometryParseError:
            if _binary_size_consistent(data):
                return _parse_binary(data, path)
            raise
    return _parse_binary(data, path)


def import_stl(path) -> CoordListGeometry:
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise GeometryParseError(str(e), path=path) from None
    return import_stl_bytes(data, path)
