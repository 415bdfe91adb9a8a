"""Golden ASCII STL cases from the real reference parser (build container only).

Runs octowall.geometry._parse_ascii_stl (/root/reference/pkg/src) on
well-formed and malformed ASCII STL texts and records, per case, either the
parsed triangles (float32, base64) or the exact GeometryParseError message and
line.  Output: tests/golden/stl_ascii_cases.json, checked against the native
parser by tests/test_stl_ascii.py.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_stl_golden.py
"""

import base64
import json
import os

import numpy as np

from octowall import geometry as rg
from octowall.errors import GeometryParseError, InvalidParameterError

HERE = os.path.dirname(os.path.abspath(__file__))


def facet(v, n="0 0 1", sep="\n"):
    lines = [f"facet normal {n}", "outer loop"] + [f"vertex {a} {b} {c}" for a, b, c in v] + ["endloop", "endfacet"]
    return sep.join(lines)


def cases():
    t1 = [("0", "0", "0"), ("1", "0", "0"), ("0", "1", "0")]
    t2 = [("0.1", "-2.5e-3", "1_0"), ("+.5", "3.", "-0"), ("1E2", "1_000.000_1", "-1e-40")]
    good = "solid x\n" + facet(t1) + "\n" + facet(t2) + "\nendsolid x\n"
    yield "good", good
    yield "good_crlf", good.replace("\n", "\r\n")
    yield "good_mixed_breaks", "solid a b c\r" + facet(t1, sep="\x0b") + "\x0c" + facet(t1, sep="\x1c") + "\nendsolid"
    yield "good_case", good.upper()
    yield "nonfinite", "solid x\n" + facet([("0", "0", "0"), ("inf", "0", "0"), ("0", "nan", "0")]) + "\nendsolid\n"
    yield "nonfinite_normal_ok", "solid x\n" + facet(t1, n="Infinity -INF NaN") + "\nendsolid\n"
    yield "good_unicode_name", "solid café   x\n" + facet(t1) + "\nendsolid café\n"
    yield "good_unicode_digits", "solid x\n" + facet([("１", "0", "0"), ("0", "١", "0"), ("0", "0", "1")]) + "\nendsolid\n"
    yield "good_no_facets", "solid\nendsolid\n"
    yield "good_tabs", good.replace(" ", "\t\t")
    yield "good_trailing_name", good + "x y z\n"
    yield "empty", ""
    yield "only_solid", "solid"
    yield "no_solid", "facet normal 0 0 1\n"
    yield "bad_normal_kw", "solid x\nfacet norm 0 0 1\n"
    yield "bad_number_normal", "solid x\n" + facet(t1, n="0 zero 1") + "\nendsolid\n"
    yield "bad_number_vertex", "solid x\n" + facet([("0", "0", "0"), ("1", "0x1", "0"), ("0", "1", "0")]) + "\nendsolid\n"
    yield "bad_underscore", "solid x\n" + facet([("0", "0", "0"), ("1__0", "0", "0"), ("0", "1", "0")]) + "\nendsolid\n"
    yield "bad_trailing_underscore", "solid x\n" + facet([("0", "0", "0"), ("1_", "0", "0"), ("0", "1", "0")]) + "\nendsolid\n"
    yield "bad_outer", "solid x\nfacet normal 0 0 1\nouter lop\n"
    yield "bad_vertex_kw", "solid x\nfacet normal 0 0 1 outer loop vertx 0 0 0\n"
    yield "bad_endloop", "solid x\n" + facet(t1).replace("endloop", "endlop") + "\nendsolid\n"
    yield "bad_endfacet", "solid x\n" + facet(t1).replace("endfacet", "end") + "\nendsolid\n"
    yield "bad_facet_kw", "solid x\n" + facet(t1) + "\nfoo\nendsolid\n"
    yield "truncated_mid_facet", "solid x\n" + facet(t1)[:40]
    yield "truncated_no_endsolid", "solid x\n" + facet(t1) + "\n"
    yield "four_vertices", "solid x\nfacet normal 0 0 1\nouter loop\nvertex 0 0 0\nvertex 1 0 0\nvertex 0 1 0\nvertex 1 1 0\nendloop\nendfacet\nendsolid\n"
    yield "keyword_after_end", good + "facet\n"
    yield "solid_after_end", good + "name solid\n"
    yield "quote_token", "solid x\n" + facet([("0", "0", "0"), ("1'", "0", "0"), ("0", "1", "0")]) + "\nendsolid\n"
    yield "unicode_bad_token", "solid x\n" + facet([("0", "0", "0"), ("é", "0", "0"), ("0", "1", "0")]) + "\nendsolid\n"
    yield "unicode_bad_keyword", "solid x\nfacet nörmal 0 0 1\n"
    yield "error_line_after_crlf", "solid x\r\n\r\n" + facet(t1, sep="\r\n").replace("outer", "inner") + "\r\nendsolid\r\n"
    yield "error_line_after_vt", "solid x\x0b\x0b\x1d" + facet(t1, sep="\x1e").replace("vertex 0 1 0", "vertex 0 1") + "\nendsolid\n"
    yield "control_char_token", "solid x\n" + facet([("0", "0", "0"), ("1\x01", "0", "0"), ("0", "1", "0")]) + "\nendsolid\n"


def main():
    out = []
    for name, text in cases():
        data = text.encode("utf-8")
        rec = {"name": name, "data": base64.b64encode(data).decode()}
        try:
            g = rg._parse_ascii_stl(data, "case.stl")
            c = np.ascontiguousarray(np.asarray(g.coords, np.float32))
            rec["coords"] = base64.b64encode(c.tobytes()).decode()
            rec["shape"] = list(c.shape)
        except GeometryParseError as e:
            rec["error"] = str(e)
        except InvalidParameterError as e:
            rec["invalid"] = str(e)
        out.append(rec)
    rec = {"name": "invalid_utf8", "data": base64.b64encode(b"solid \xff\xfe\n").decode()}
    try:
        rg._parse_ascii_stl(b"solid \xff\xfe\n", "case.stl")
    except GeometryParseError as e:
        rec["error"] = str(e)
    out.append(rec)
    with open(os.path.join(HERE, "stl_ascii_cases.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print(len(out), "cases")


if __name__ == "__main__":
    main()
