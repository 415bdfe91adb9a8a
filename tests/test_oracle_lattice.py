"""Known-answer tests pinning the lattice-link oracle (north-star extension).

The reference has no lattice links, so oracle/lattice.py is pinned only by
analytic cases: an axis-aligned wall at a known offset (q exact), links
parallel to a wall (no hit), a link ending exactly on a wall (q = 1), a 2D
square, and the direction tables.
"""

import numpy as np

from oracle import forest as of
from oracle import lattice as ol

F32 = np.float32


def _wall_z(z, lo=0.0, hi=1.0):
    """Two triangles spanning z = const over [lo, hi]^2."""
    tri = np.array([[[lo, lo, z], [hi, lo, z], [hi, hi, z]], [[lo, lo, z], [hi, hi, z], [lo, hi, z]]], F32)
    return np.ascontiguousarray(np.transpose(tri, (1, 2, 0)))


def test_direction_tables():
    assert len(ol.D2Q9) == 9 and len(ol.D3Q19) == 19 and len(ol.D3Q27) == 27
    for name, dirs in ol.LATTICES.items():
        d = np.asarray(dirs)
        assert np.all(d[0] == 0)
        assert len({tuple(v) for v in d}) == len(d)  # distinct
        assert np.all(np.abs(d) <= 1)
    d19 = np.asarray(ol.D3Q19)
    assert np.all(np.abs(d19).sum(1)[1:] <= 2)
    assert ol.D3Q27[19] == (1, 1, 1) and ol.D3Q27[26] == (-1, -1, -1)


def test_axis_aligned_wall_q_is_analytic():
    # 1 root block, 64 cells of h = 0.25; cell centres at 0.125 + 0.25 k
    f = of.Forest((0, 0, 0), (1, 1, 1), (1, 1, 1))
    z = F32(0.2)  # between the first two cell-centre planes (0.125, 0.375)
    coords = _wall_z(z)
    out = ol.lattice_links(f, coords, "D3Q19")
    flags, q, cells = out["flags"], out["q"], out["boundary"]
    dirs = ol.directions("D3Q19")
    h = F32(0.25)
    for row, cell in enumerate(cells):
        ix, iy, iz = cell & 3, (cell >> 2) & 3, (cell >> 4) & 3
        if ix in (0, 3) or iy in (0, 3):
            continue  # diagonal links of rim cells cross outside the wall's extent
        x_z = F32(0.125) + F32(0.25) * F32(iz)
        for i in range(1, 19):
            hit = bool((flags[cell] >> i) & 1)
            cz = dirs[i][2]
            crosses = cz != 0 and min(x_z, x_z + cz * h) <= z <= max(x_z, x_z + cz * h)
            assert hit == crosses, (cell, i)
            if hit:
                assert abs(float(q[row, i]) - abs(float(z - x_z)) / 0.25) < 1e-6
            else:
                assert q[row, i] == -1.0
    # every cell of the two layers next to the wall links across it, no other cell
    assert len(cells) == 32


def test_parallel_links_never_hit():
    f = of.Forest((0, 0, 0), (1, 1, 1), (1, 1, 1))
    out = ol.lattice_links(f, _wall_z(F32(0.125)), "D3Q19")  # wall through the first centre plane
    dirs = ol.directions("D3Q19")
    for cell in out["boundary"]:
        for i in range(1, 19):
            if dirs[i][2] == 0 and (out["flags"][cell] >> i) & 1:
                # in-plane links of the cells lying on the wall touch it at t = 0
                assert ((cell >> 4) & 3) == 0
    # cells on the wall: links leaving the plane hit at t = 0 exactly
    row = list(out["boundary"]).index(0)
    assert out["q"][row, 5] == 0.0 and out["q"][row, 6] == 0.0


def test_link_ending_on_wall_has_q_one():
    f = of.Forest((0, 0, 0), (1, 1, 1), (1, 1, 1))
    out = ol.lattice_links(f, _wall_z(F32(0.375)), "D3Q19")
    cell = 0  # centre z = 0.125; +z link ends at 0.375 exactly
    row = list(out["boundary"]).index(cell)
    assert (out["flags"][cell] >> 5) & 1 and out["q"][row, 5] == 1.0


def test_square_2d():
    f = of.Forest((0, 0), (1, 1), (1, 1))
    sq = np.array([[[0.3, 0.3], [0.7, 0.3]], [[0.7, 0.3], [0.7, 0.7]], [[0.7, 0.7], [0.3, 0.7]],
                   [[0.3, 0.7], [0.3, 0.3]]], F32)
    coords = np.ascontiguousarray(np.transpose(sq, (1, 2, 0)))
    out = ol.lattice_links(f, coords, "D2Q9")
    dirs = ol.directions("D2Q9")
    # cell (1,1) centre (0.375, 0.375): -x link crosses x = 0.3 at t = 0.075/0.25
    cell = 1 + 4 * 1
    row = list(out["boundary"]).index(cell)
    assert abs(out["q"][row, 3] - F32(0.3)) < 1e-6 and tuple(dirs[3]) == (-1, 0)
    assert abs(out["q"][row, 4] - F32(0.3)) < 1e-6
    assert out["q"][row, 1] == -1.0  # +x stays inside the square
    # corner cell (0,0) centre (0.125, 0.125): diagonal (1,1) reaches (0.375, 0.375) through the corner region
    c0 = list(out["boundary"]).index(0)
    assert abs(out["q"][c0, 5] - F32(0.7)) < 1e-6


def test_packed_rows_round_trip_the_oracle_output():
    """The packed host form (flag word per boundary row + q of the set bits,
    rows in order, directions ascending) that GridPlan.run(host=True)
    transfers is lossless: pipeline.unpack_q restores the oracle's dense rows,
    and the set bits are exactly the q >= 0 entries."""
    from paper_2502_16310_b200.pipeline import unpack_q

    f = of.Forest((0, 0, 0), (1, 1, 1), (2, 2, 2))
    rng = np.random.default_rng(5)
    v0 = rng.uniform(0.1, 0.9, (40, 3)).astype(F32)
    tri = np.stack([v0, v0 + rng.uniform(-0.2, 0.2, (40, 3)).astype(F32),
                    v0 + rng.uniform(-0.2, 0.2, (40, 3)).astype(F32)], 1)
    coords = np.ascontiguousarray(np.transpose(tri, (1, 2, 0)))
    out = ol.lattice_links(f, coords, "D3Q27")
    q, cells = out["q"], out["boundary"]
    assert len(cells) > 0
    row_flags = out["flags"][cells].astype(np.uint32)
    bits = ((row_flags[:, None] >> np.arange(27, dtype=np.uint32)) & 1).astype(bool)
    np.testing.assert_array_equal(bits, q >= 0)
    q_packed = q[bits]  # row-major: rows in order, directions ascending
    np.testing.assert_array_equal(unpack_q(row_flags, q_packed, 27), q)


def _edge_crossings(n, seed):
    """Links aimed at points of the shared edge (a, b) of two triangles
    (a, b, c1), (b, a, c2) lying on opposite sides of the plane spanned by
    the link line and the edge: the line crosses the two-face fan through the
    edge.  Faces nearly parallel to the link (|sin| < 1e-3, where float32 t is
    meaningless) are dropped."""
    rng = np.random.default_rng(seed)
    a, b, c1, c2 = (rng.uniform(0.2, 0.8, (n, 3)).astype(F32) for _ in range(4))
    s = rng.uniform(0.05, 0.95, n).astype(F32)
    p = (a + s[:, None] * (b - a)).astype(F32)
    h = F32(1 / 64)
    dirs = ol.directions("D3Q27")
    for i in range(1, 27):
        dv = (dirs[i].astype(F32) * h).astype(F32)
        tt = rng.uniform(0.05, 0.95, n).astype(F32)
        x = (p - tt[:, None] * dv).astype(F32)
        d64 = dv.astype(np.float64) / np.linalg.norm(dv)
        nrm = np.cross(d64, (b - a).astype(np.float64))
        s1 = np.einsum("ij,ij->i", nrm, (c1 - a).astype(np.float64))
        s2 = np.einsum("ij,ij->i", nrm, (c2 - a).astype(np.float64))
        ok = s1 * s2 < 0
        for c in (c1, c2):  # well-conditioned: the face is not nearly parallel to the link
            fn = np.cross((b - a).astype(np.float64), (c - a).astype(np.float64))
            fn /= np.linalg.norm(fn, axis=1, keepdims=True)
            ok &= np.abs(fn @ d64) > 1e-3
        t1 = np.stack([a, b, c1]).transpose(0, 2, 1)
        t2 = np.stack([b, a, c2]).transpose(0, 2, 1)
        yield x[ok], dv, t1[:, :, ok], t2[:, :, ok]


def test_watertight_through_shared_edges():
    """A link crossing a two-triangle fan through (within rounding of) the
    shared edge hits at least one of the two faces: the edge functions of
    the shared edge are computed from the same translated, sheared vertices
    in both faces.  The round-1 Moller-Trumbore test loses a measurable
    fraction of exactly these links (printed; the reason the definition
    changed)."""
    total = wt_lost = mt_lost = 0
    for x, dv, t1, t2 in _edge_crossings(40000, 11):
        h1, _ = ol.wt_hits(x, dv, t1)
        h2, _ = ol.wt_hits(x, dv, t2)
        dvec = np.broadcast_to(dv, x.shape)
        m1, _ = ol.mt_hits(x, dvec, t1)
        m2, _ = ol.mt_hits(x, dvec, t2)
        total += x.shape[0]
        wt_lost += int((~h1 & ~h2).sum())
        mt_lost += int((~m1 & ~m2).sum())
    print(f"edge crossings {total}: watertight lost {wt_lost}, Moller-Trumbore lost {mt_lost}")
    assert total > 100000
    assert wt_lost == 0
    assert mt_lost > 0


def test_watertight_2d_through_shared_vertices():
    """2D: a link through (within rounding of) the shared vertex of two
    edges whose far ends lie on opposite sides of the link line hits one."""
    rng = np.random.default_rng(3)
    n = 50000
    h = F32(1 / 64)
    lost = total = 0
    for i in range(1, 9):
        dv = (ol.directions("D2Q9")[i].astype(F32) * h).astype(F32)
        p, c1, c2 = (rng.uniform(0.2, 0.8, (n, 2)).astype(F32) for _ in range(3))
        tt = rng.uniform(0.05, 0.95, n).astype(F32)
        x = (p - tt[:, None] * dv).astype(F32)
        cr = lambda c: dv[0] * (c[:, 1] - p[:, 1]).astype(np.float64) - dv[1] * (c[:, 0] - p[:, 0])  # noqa: E731
        ok = cr(c1) * cr(c2) < 0
        e1 = np.stack([c1, p]).transpose(0, 2, 1)[:, :, ok]
        e2 = np.stack([p, c2]).transpose(0, 2, 1)[:, :, ok]
        h1, _ = ol.wt_hits2(x[ok], dv, e1)
        h2, _ = ol.wt_hits2(x[ok], dv, e2)
        total += int(ok.sum())
        lost += int((~h1 & ~h2).sum())
    assert total > 100000 and lost == 0


def test_opposite_directions_share_the_line_test():
    """t(-d) = -t(d) bitwise and the same edge decision: the identity the
    CUDA kernel uses to test each lattice line once for both directions."""
    rng = np.random.default_rng(8)
    n = 20000
    tri = rng.uniform(0.3, 0.7, (3, 3, n)).astype(F32)
    x = rng.uniform(0.3, 0.7, (n, 3)).astype(F32)
    dirs = ol.directions("D3Q27")
    h = np.array([1 / 64, 1 / 64, 1 / 64], F32)
    for i in range(1, 27):
        dv = (dirs[i].astype(F32) * h).astype(F32)
        _, ta = ol.wt_hits(x, dv, tri)
        _, tb = ol.wt_hits(x, (-dv).astype(F32), tri)
        fin = np.isfinite(ta)
        np.testing.assert_array_equal(np.isfinite(tb), fin)
        np.testing.assert_array_equal((-ta[fin]).view(np.uint32), tb[fin].view(np.uint32))


def test_closed_icosphere_referee():
    """Closed-mesh invariants against an FP64 referee (oracle/referee.py) on a
    1 280-triangle icosphere over 8^3 root blocks (32 768 cells, D3Q19): every
    link whose ends lie on opposite sides of the surface (beyond a 1e-6 band)
    is flagged, no link with both ends inside is flagged (convex surface), and
    q equals the FP64 crossing parameter within 1e-5."""
    from oracle import referee as rf
    from paper_2502_16310_b200 import shapes

    tri = shapes.icosphere_triangles(3).astype(F32)
    coords = np.ascontiguousarray(np.transpose(tri, (1, 2, 0)))
    f = of.Forest((0, 0, 0), (1, 1, 1), (8, 8, 8))
    out = ol.lattice_links(f, coords, "D3Q19")
    cen = f.cell_centers(out["leaves"]).reshape(-1, 3)
    h = (f.spacing([0])[0] / 4).astype(F32)
    dvs = (ol.directions("D3Q19").astype(F32) * h).astype(F32)
    r = np.linalg.norm(cen.astype(np.float64) - 0.5, axis=1)
    sel = np.flatnonzero(np.abs(r - 0.3) < 3 * float(h.max()))
    q = np.full((len(cen), 19), -1.0, F32)
    q[out["boundary"]] = out["q"]
    res = rf.check_links(cen[sel], dvs, out["flags"][sel], q[sel], coords, rf.StarSurface(coords))
    assert res["crossing"] > 10000 and res["crossing_missed"] == 0
    assert res["inside"] > 10000 and res["inside_flagged"] == 0
    assert res["q_checked"] > 10000 and res["q_bad"] == 0 and res["q_max_err"] < 1e-6
    assert res["unflagged_hit"] == 0
