"""The native ASCII STL parser (ow_parse_ascii_stl + the UTF-8 shim in
geometry.py) against the real reference parser's results on 36 cases
(tests/golden/stl_ascii_cases.json, made by tests/golden/make_stl_golden.py
from octowall.geometry._parse_ascii_stl): the same float32 triangles on
every input the reference accepts, and the same GeometryParseError message
and line on every input it rejects.  Host code only (no GPU)."""

import base64
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "stl_ascii_cases.json")))


@pytest.fixture(scope="module")
def geometry():
    from paper_2502_16310_b200 import _build, geometry

    _build.build()
    return geometry


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_ascii_stl_matches_reference(geometry, case):
    from paper_2502_16310_b200.errors import GeometryParseError

    data = base64.b64decode(case["data"])
    if "error" in case:
        with pytest.raises(GeometryParseError) as ei:
            geometry.ascii_stl_triangles(data, "case.stl")
        assert str(ei.value) == case["error"]
        return
    tris = geometry.ascii_stl_triangles(data, "case.stl")
    coords = np.ascontiguousarray(np.transpose(tris, (1, 2, 0)))
    if "invalid" in case:  # parsed; the reference's geometry constructor then rejects it
        assert not np.all(np.isfinite(coords))
        return
    want = np.frombuffer(base64.b64decode(case["coords"]), np.float32).reshape(case["shape"])
    np.testing.assert_array_equal(coords.view(np.uint32), want.view(np.uint32))


def test_ascii_stl_large_parallel(geometry):
    """A multi-megabyte file (parallel tokeniser) parses to the values the
    NumPy float64 -> float32 path gives, and an error deep inside it is
    located at the reference's line."""
    from paper_2502_16310_b200.errors import GeometryParseError

    rng = np.random.default_rng(4)
    tris = rng.uniform(-1, 1, (40000, 3, 3))
    body = "".join("facet normal 0 0 1\n outer loop\n" + "".join(f"  vertex {float(a)!r} {float(b)!r} {float(c)!r}\n" for a, b, c in t)
                   + " endloop\nendfacet\n" for t in tris)
    data = ("solid big\n" + body + "endsolid big\n").encode()
    assert len(data) > (1 << 20)
    got = geometry.ascii_stl_triangles(data)
    np.testing.assert_array_equal(got, tris.astype(np.float32))
    lines = data.split(b"\n")
    k = 7 * 30000 + 3  # a vertex line of facet 30000
    lines[k] = lines[k].replace(b"vertex", b"vertexx")
    with pytest.raises(GeometryParseError, match=f"line {k + 1}: expected 'vertex', got 'vertexx'"):
        geometry.ascii_stl_triangles(b"\n".join(lines))
