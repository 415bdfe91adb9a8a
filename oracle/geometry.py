"""Oracle: geometry import and validation (test infrastructure only).

Restates octowall/geometry.py:
  circle primitive            geometry.py:127-138
  lat-lon sphere primitive    geometry.py:141-192
  primitive text format       geometry.py:211-259
  index -> coordinate list    geometry.py:262-273
  degenerate-face test        geometry.py:276-299
  bounding box                geometry.py:302-308
  STL autodetect / parsers    geometry.py:319-436
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import InvalidParameter, ParseError


def circle(cx, cy, r, n):
    """(vertices (n,2) f32, faces (n,2) i32) — angles 2*pi*k/n, f64 -> f32."""
    if n < 3 or r <= 0:
        raise InvalidParameter("bad circle")
    k = np.arange(n)
    ang = 2.0 * np.pi * k / n
    v = np.empty((n, 2), np.float64)
    v[:, 0] = cx + r * np.cos(ang)
    v[:, 1] = cy + r * np.sin(ang)
    f = np.stack([k, (k + 1) % n], 1).astype(np.int32)
    return v.astype(np.float32), f


def latlon_sphere(cx, cy, cz, r, n_lat, n_lon):
    """Pole fans + two triangles per interior quad (outward winding)."""
    if n_lat < 2 or n_lon < 3 or r <= 0:
        raise InvalidParameter("bad sphere")
    c = np.array([cx, cy, cz], np.float64)
    rows = [c + np.array([0.0, 0.0, r])]
    phi = 2.0 * np.pi * np.arange(n_lon) / n_lon
    for k in range(1, n_lat):
        th = np.pi * k / n_lat
        st, ct = np.sin(th), np.cos(th)
        ring = np.empty((n_lon, 3))
        ring[:, 0] = c[0] + r * st * np.cos(phi)
        ring[:, 1] = c[1] + r * st * np.sin(phi)
        ring[:, 2] = c[2] + r * np.full(n_lon, ct)
        rows.append(ring)
    rows.append(c + np.array([0.0, 0.0, -r]))
    verts = np.vstack([np.atleast_2d(x) for x in rows]).astype(np.float32)
    south = len(verts) - 1
    j = np.arange(n_lon)
    jn = (j + 1) % n_lon
    faces = [np.stack([np.zeros(n_lon, int), 1 + j, 1 + jn], 1)]
    for k in range(1, n_lat - 1):
        a0, b0 = 1 + (k - 1) * n_lon, 1 + k * n_lon
        quad = np.empty((n_lon, 2, 3), int)
        quad[:, 0] = np.stack([a0 + j, b0 + j, b0 + jn], 1)
        quad[:, 1] = np.stack([a0 + j, b0 + jn, a0 + jn], 1)
        faces.append(quad.reshape(-1, 3))
    last = 1 + (n_lat - 2) * n_lon
    faces.append(np.stack([np.full(n_lon, south), last + jn, last + j], 1))
    return verts, np.vstack(faces).astype(np.int32)


def parse_primitives(text, dim=None):
    """``circle cx cy r n`` / ``sphere cx cy cz r nlat nlon`` lines; '#' comments."""
    verts, faces, off, gdim = [], [], 0, None
    for ln, raw in enumerate(text.splitlines(), 1):
        body = raw.split("#", 1)[0].split()
        if not body:
            continue
        kind, args = body[0].lower(), body[1:]
        try:
            if kind == "circle" and len(args) == 4:
                n = float(args[3])
                if n != int(n):
                    raise ValueError
                v, f = circle(float(args[0]), float(args[1]), float(args[2]), int(n))
                d = 2
            elif kind == "sphere" and len(args) == 6:
                nl, nn = float(args[4]), float(args[5])
                if nl != int(nl) or nn != int(nn):
                    raise ValueError
                v, f = latlon_sphere(*(float(a) for a in args[:4]), int(nl), int(nn))
                d = 3
            else:
                raise ParseError(f"line {ln}: bad primitive")
        except ValueError:
            raise ParseError(f"line {ln}: cannot parse numbers") from None
        except InvalidParameter as e:
            raise ParseError(f"line {ln}: {e}") from None
        if gdim is not None and gdim != d:
            raise InvalidParameter("mixed dimension")
        gdim = d
        verts.append(v)
        faces.append(f + off)
        off += len(v)
    if gdim is None:
        d = dim if dim is not None else 2
        return np.zeros((0, d), np.float32), np.zeros((0, d), np.int32)
    if dim is not None and dim != gdim:
        raise ParseError("dimension mismatch")
    return np.vstack(verts), np.vstack(faces)


def index_to_coords(vertices, faces):
    """coords[j, c, k] = vertices[faces[k, j], c]  (pure gather)."""
    vertices = np.asarray(vertices, np.float32)
    faces = np.asarray(faces, np.int64)
    return np.ascontiguousarray(vertices[faces].transpose(1, 2, 0))


def first_degenerate(coords):
    """Index of the first degenerate face, or -1 (FP64 test)."""
    c = np.asarray(coords, np.float64)
    if c.shape[2] == 0:
        return -1
    if c.shape[0] == 2:
        e = c[1] - c[0]
        bad = (e[0] * e[0] + e[1] * e[1]) == 0.0
    else:
        u, v, w = c[1] - c[0], c[2] - c[0], c[2] - c[1]

        def sq(x):
            return (x[0] * x[0] + x[1] * x[1]) + x[2] * x[2]

        s = np.maximum(np.maximum(sq(u), sq(v)), sq(w))
        cx = u[1] * v[2] - u[2] * v[1]
        cy = u[2] * v[0] - u[0] * v[2]
        cz = u[0] * v[1] - u[1] * v[0]
        area = np.sqrt((cx * cx + cy * cy) + cz * cz)
        bad = (s == 0.0) | (area < 1e-12 * s)
    idx = np.flatnonzero(bad)
    return int(idx[0]) if idx.size else -1


def bbox(coords):
    c = np.asarray(coords, np.float32)
    return c.min(axis=(0, 2)).astype(np.float64), c.max(axis=(0, 2)).astype(np.float64)


def stl_binary(data):
    if len(data) < 84:
        raise ParseError("binary STL shorter than header + facet count")
    (n,) = struct.unpack_from("<I", data, 80)
    if len(data) < 84 + 50 * n:
        raise ParseError("binary STL truncated")
    rec = np.frombuffer(data, np.uint8, count=50 * n, offset=84).reshape(n, 50)
    fl = rec[:, 12:48].copy().view("<f4").reshape(n, 3, 3)  # vertex slots only
    return np.ascontiguousarray(fl.transpose(1, 2, 0).astype(np.float32))


def stl_ascii(data):
    toks = data.decode("utf-8").split()
    pos = 0

    def nxt():
        nonlocal pos
        if pos >= len(toks):
            raise ParseError("unexpected end of file")
        pos += 1
        return toks[pos - 1]

    def expect(word):
        t = nxt()
        if t.lower() != word:
            raise ParseError(f"expected {word!r}, got {t!r}")

    def num():
        t = nxt()
        try:
            return float(t)
        except ValueError:
            raise ParseError(f"expected a number, got {t!r}") from None

    expect("solid")
    while pos < len(toks) and toks[pos].lower() not in ("facet", "endsolid"):
        pos += 1
    tris = []
    while True:
        t = nxt().lower()
        if t == "endsolid":
            break
        if t != "facet":
            raise ParseError("expected 'facet' or 'endsolid'")
        expect("normal")
        num(), num(), num()
        expect("outer")
        expect("loop")
        tri = []
        for _ in range(3):
            expect("vertex")
            tri.append((num(), num(), num()))
        expect("endloop")
        expect("endfacet")
        tris.append(tri)
    for t in toks[pos:]:
        if t.lower() in ("facet", "solid", "vertex", "endsolid"):
            raise ParseError(f"unexpected {t!r} after endsolid")
    a = np.asarray(tris, np.float64).astype(np.float32).reshape(-1, 3, 3)
    return np.ascontiguousarray(a.transpose(1, 2, 0))


def stl(data):
    """Autodetect like geometry.py:331-339."""
    if data.lstrip()[:5] == b"solid":
        try:
            return stl_ascii(data)
        except (ParseError, UnicodeDecodeError):
            if len(data) >= 84:
                (n,) = struct.unpack_from("<I", data, 80)
                if len(data) == 84 + 50 * n:
                    return stl_binary(data)
            raise ParseError("bad ASCII STL") from None
    return stl_binary(data)
