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
