"""Boundary geometry: primitives, text / STL import, coordinate lists on the GPU.

Mirrors octowall/geometry.py (same names, arguments, dtypes and errors).  The
coordinate-list form lives in HBM as a float32 (verts_per_face, dim, n_faces)
tensor — the reference's structure-of-arrays layout (geometry.py:94-124) —
and every per-face pass over it (binary-STL transpose, index gather,
degeneracy test, bounding box) is a sm_100a kernel in libowb200.so.  Text
primitives and ASCII STL are tokenised on the host (the reference does the
same in Python); their float64 -> float32 rounding is done by NumPy so the
vertices are bit-identical to the reference's.
"""

from __future__ import annotations

import ctypes as C
import itertools
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import GeometryParseError, InvalidParameterError

_keys = itertools.count(1)


def as_point(p, dim):
    a = np.asarray(p, dtype=np.float64).reshape(-1)
    if a.shape[0] != dim:
        raise InvalidParameterError(f"expected a {dim}-component point, got {a.shape[0]}")
    if not np.all(np.isfinite(a)):
        raise InvalidParameterError(f"point has non-finite components: {a}")
    return a


@dataclass
class Aabb:
    """Axis-aligned box, float64 (geometry.py:28-55)."""

    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        self.min = np.asarray(self.min, dtype=np.float64).reshape(-1)
        self.max = np.asarray(self.max, dtype=np.float64).reshape(-1)
        if self.min.shape != self.max.shape:
            raise InvalidParameterError("aabb min/max dimension mismatch")
        if not (np.all(np.isfinite(self.min)) and np.all(np.isfinite(self.max))):
            raise InvalidParameterError("aabb has non-finite corners")
        if np.any(self.min > self.max):
            raise InvalidParameterError(f"aabb min {self.min} exceeds max {self.max}")

    @property
    def dim(self):
        return self.min.shape[0]

    @property
    def extent(self):
        return self.max - self.min

    def contains(self, p, tol=0.0):
        p = np.asarray(p, dtype=np.float64)
        return bool(np.all(p >= self.min - tol) and np.all(p <= self.max + tol))


@dataclass
class IndexedGeometry:
    """Shared-vertex mesh (host): vertices (V, dim) float32, faces (F, dim) int32."""

    dim: int
    vertices: np.ndarray
    faces: np.ndarray

    def __post_init__(self):
        if self.dim not in (2, 3):
            raise InvalidParameterError(f"dim must be 2 or 3, got {self.dim}")
        self.vertices = np.asarray(self.vertices, dtype=np.float32).reshape(-1, self.dim)
        self.faces = np.asarray(self.faces, dtype=np.int32).reshape(-1, self.dim)
        if not np.all(np.isfinite(self.vertices)):
            raise InvalidParameterError("geometry has non-finite vertex coordinates")
        if self.faces.size:
            if self.faces.min() < 0 or self.faces.max() >= len(self.vertices):
                raise InvalidParameterError("face index out of range")
            for j in range(self.dim):
                for k in range(j + 1, self.dim):
                    if np.any(self.faces[:, j] == self.faces[:, k]):
                        raise InvalidParameterError("face has repeated vertex indices")

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
    parts = list(parts)
    if not parts:
        raise InvalidParameterError("nothing to append")
    dim = parts[0].dim
    if any(p.dim != dim for p in parts):
        raise InvalidParameterError("cannot append geometries of mixed dimension")
    verts, faces, off = [], [], 0
    for p in parts:
        verts.append(p.vertices)
        faces.append(p.faces + off)
        off += len(p.vertices)
    return IndexedGeometry(dim, np.vstack(verts), np.vstack(faces))


def _parse_count(s):
    v = float(s)
    if v != int(v):
        raise ValueError(s)
    return int(v)


def parse_text_primitives(text, path=None, dim=None):
    parts = []
    for ln, raw in enumerate(text.splitlines(), start=1):
        body = raw.split("#", 1)[0].strip()
        if not body:
            continue
        tok = body.split()
        kind, args = tok[0].lower(), tok[1:]
        try:
            if kind == "circle":
                if len(args) != 4:
                    raise GeometryParseError("circle takes 4 values: cx cy r n_edges", path, ln)
                cx, cy, r = (float(a) for a in args[:3])
                parts.append(generate_circle((cx, cy), r, _parse_count(args[3])))
            elif kind == "sphere":
                if len(args) != 6:
                    raise GeometryParseError("sphere takes 6 values: cx cy cz r n_lat n_lon", path, ln)
                cx, cy, cz, r = (float(a) for a in args[:4])
                parts.append(generate_sphere((cx, cy, cz), r, _parse_count(args[4]), _parse_count(args[5])))
            else:
                raise GeometryParseError(f"unknown primitive {kind!r}", path, ln)
        except ValueError:
            raise GeometryParseError(f"cannot parse numbers in {body!r}", path, ln) from None
        except InvalidParameterError as e:
            raise GeometryParseError(str(e), path, ln) from None
    if not parts:
        return IndexedGeometry.empty(dim if dim is not None else 2)
    out = append_geometry(parts)
    if dim is not None and out.dim != dim:
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


def index_to_coords(g: IndexedGeometry) -> CoordListGeometry:
    """Indexed mesh -> device coordinate list; pure gather on the GPU."""
    dev = _lib.device()
    n = g.n_faces
    out = torch.empty((g.dim, g.dim, n), dtype=torch.float32, device=dev)
    if n:
        v = torch.from_numpy(np.ascontiguousarray(g.vertices)).to(dev)
        fc = torch.from_numpy(np.ascontiguousarray(g.faces)).to(dev)
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


def _parse_ascii(data, path):
    """Native fast path first (ow_parse_ascii_stl); on anything it does not
    accept, the reference-faithful parser below reports the exact error."""
    cap = len(data) // 64 + 1  # a facet takes > 64 bytes of ASCII text
    tris = np.empty((cap, 3, 3), np.float32)
    n = C.c_int64(0)
    if _lib.lib().ow_parse_ascii_stl(bytes(data), len(data), tris.ctypes.data_as(C.c_void_p), cap, C.byref(n)) == 0:
        coords = np.ascontiguousarray(np.transpose(tris[: n.value], (1, 2, 0)))
        return CoordListGeometry(3, coords)
    return _parse_ascii_py(data, path)


def _parse_ascii_py(data, path):
    try:
        text = data.decode("utf-8", errors="strict")
    except UnicodeDecodeError:
        raise GeometryParseError("not valid ASCII STL text", path=path) from None
    toks, lines = [], []
    for ln, line in enumerate(text.splitlines(), start=1):
        for t in line.split():
            toks.append(t)
            lines.append(ln)
    pos = 0
    n_tok = len(toks)

    def take(expect=None):
        nonlocal pos
        if pos >= n_tok:
            raise GeometryParseError("unexpected end of file", path, lines[-1] if lines else None)
        t = toks[pos]
        pos += 1
        if expect is not None and t.lower() != expect:
            raise GeometryParseError(f"expected {expect!r}, got {t!r}", path, lines[pos - 1])
        return t

    def num():
        t = take()
        try:
            return float(t)
        except ValueError:
            raise GeometryParseError(f"expected a number, got {t!r}", path, lines[pos - 1]) from None

    take("solid")
    while pos < n_tok and toks[pos].lower() not in ("facet", "endsolid"):
        pos += 1
    vals = []
    while True:
        t = take()
        kw = t.lower()
        if kw == "endsolid":
            break
        if kw != "facet":
            raise GeometryParseError(f"expected 'facet' or 'endsolid', got {t!r}", path, lines[pos - 1])
        take("normal")
        num(), num(), num()
        take("outer")
        take("loop")
        for _ in range(3):
            take("vertex")
            vals.extend((num(), num(), num()))
        take("endloop")
        take("endfacet")
    while pos < n_tok:
        if toks[pos].lower() in ("facet", "solid", "vertex", "endsolid"):
            raise GeometryParseError(f"unexpected {toks[pos]!r} after endsolid", path, lines[pos])
        pos += 1
    tris = np.asarray(vals, dtype=np.float64).astype(np.float32).reshape(-1, 3, 3)
    coords = np.ascontiguousarray(np.transpose(tris, (1, 2, 0)))
    return CoordListGeometry(3, coords)


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
