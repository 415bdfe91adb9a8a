"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

Every fixture in tests/golden/ was produced by running the real reference
(tests/golden/make_golden.py).  The oracle must reproduce them bit for bit;
only then is it trusted as the checker for the CUDA path.
"""

import numpy as np
import pytest

import golden_util as gu
from oracle import binning as ob
from oracle import forest as of
from oracle import geometry as og
from oracle import nearwall as on
from oracle import predicate as op
from oracle.errors import Capacity, InvalidParameter


@pytest.mark.parametrize("path", gu.files("bins_"), ids=gu.ids(gu.files("bins_")))
def test_fill_bins_matches_reference(path):
    g = gu.load(path)
    coords = gu.geometry(g)
    dim = coords.shape[0]
    grid = ob.Grid(*gu.unit_domain(dim), int(g["bins_per_axis"]))
    h = None if np.isnan(g["spacing"]) else float(g["spacing"])
    ids, counts, offsets = ob.fill_bins(coords, grid, spacing=h, overlap_factor=10 ** 6)
    np.testing.assert_array_equal(counts, g["counts"])
    np.testing.assert_array_equal(offsets, g["offsets"])
    np.testing.assert_array_equal(ids, g["ids"])


def test_predicate_triangle_matches_reference():
    g = gu.load(gu.files("pred_tri")[0])
    coords = np.transpose(g["tri"], (1, 2, 0)).copy()
    mask = op.near(g["pts"], coords, g["d"])
    np.testing.assert_array_equal(mask, g["mask"])


def test_predicate_edge_matches_reference():
    g = gu.load(gu.files("pred_edge")[0])
    coords = np.transpose(g["seg"], (1, 2, 0)).copy()
    mask = op.near(g["pts"], coords, g["d"])
    np.testing.assert_array_equal(mask, g["mask"])


@pytest.mark.parametrize("path", gu.files("mark_"), ids=gu.ids(gu.files("mark_")))
def test_marking_matches_reference(path):
    g = gu.load(path)
    coords = gu.geometry(g)
    dim = coords.shape[0]
    f = of.Forest(*gu.unit_domain(dim), (int(g["root"]),) * dim)
    b = int(g["bins_per_axis"])
    if b < 0:
        n = on.mark(f, 0, coords, float(g["d_spec"]))
    else:
        grid = ob.Grid(*gu.unit_domain(dim), b)
        n = on.mark(f, 0, coords, float(g["d_spec"]), ob.fill_bins(coords, grid), grid)
    assert n == int(g["n_marked"])
    np.testing.assert_array_equal(f.marks, g["marks"])


def _pipe_files(big):
    out = []
    for p in gu.files("pipe_"):
        heavy = "12800" in p or "icosphere5" in p
        if heavy == big:
            out.append(p)
    return out


def _check_pipeline(path):
    g = gu.load(path)
    coords = gu.geometry(g)
    dim = coords.shape[0]
    f = of.Forest(*gu.unit_domain(dim), (int(g["root"]),) * dim)
    res = on.refine_near_wall(f, coords, float(g["d_spec"]), n_levels=int(g["n_levels"]),
                              strategy=str(g["strategy"]), bins_per_axis=int(g["bins_per_axis"]))
    assert res["marked_detected"] == g["marked_detected"].tolist()
    assert res["marked_refined"] == g["marked_refined"].tolist()
    assert f.n == int(g["n_blocks"])
    np.testing.assert_array_equal(f.level, g["level"])
    np.testing.assert_array_equal(f.coords, g["coords"])
    np.testing.assert_array_equal(f.parent, g["parent"])
    np.testing.assert_array_equal(f.first_child, g["first_child"])
    np.testing.assert_array_equal(f.marks, g["marks"])
    assert f.blocks_per_level() == g["blocks_per_level"].tolist()
    assert f.leaves_per_level() == g["leaves_per_level"].tolist()
    if "bin_ids" in g:
        np.testing.assert_array_equal(res["bins"][0], g["bin_ids"])
        np.testing.assert_array_equal(res["bins"][1], g["bin_counts"])


@pytest.mark.parametrize("path", _pipe_files(False), ids=gu.ids(_pipe_files(False)))
def test_pipeline_matches_reference(path):
    _check_pipeline(path)


@pytest.mark.slow
@pytest.mark.parametrize("path", _pipe_files(True), ids=gu.ids(_pipe_files(True)))
def test_pipeline_matches_reference_large(path):
    _check_pipeline(path)


def _forest_from(g, prefix, dim, root):
    f = of.Forest(*gu.unit_domain(dim), (root,) * dim)
    return f


def test_forest_units_match_reference():
    g = gu.load(gu.files("forest_units")[0])
    # propagation with scattered seeds on 8x8
    f = of.Forest(*gu.unit_domain(2), (8, 8))
    f.marks[[3, 17, 44]] = of.MARKED
    on.propagate(f, 0, 0.3)
    np.testing.assert_array_equal(f.marks, g["prop8_marks"])
    # 3D mixed-level propagation
    f = of.Forest(*gu.unit_domain(3), (4, 4, 4))
    f.marks[[5, 21, 42]] = of.MARKED
    f.refine_marked(0)
    lv1 = f.leaves_at(1)
    f.marks[lv1[::5]] = of.MARKED
    f.marks[[0, 63]] = of.MARKED
    on.propagate(f, 0, 0.3, rounds=2)
    np.testing.assert_array_equal(f.marks, g["prop3d_marks"])
    np.testing.assert_array_equal(f.coords, g["prop3d_coords"])
    # random refinements
    for dim, seed, rounds, root in ((2, 1, 3, 4), (2, 3, 4, 4), (3, 5, 3, 3), (3, 8, 4, 2)):
        rng = np.random.default_rng(seed)
        f = of.Forest(*gu.unit_domain(dim), (root,) * dim)
        splits = []
        for lv in range(rounds):
            leaves = f.leaves_at(lv)
            if len(leaves) == 0:
                break
            pick = leaves[rng.random(len(leaves)) < 0.4]
            f.marks[pick] = of.MARKED
            splits.append(f.refine_marked(lv))
        p = f"rand{dim}d_s{seed}_"
        assert splits == g[p + "splits"].tolist()
        np.testing.assert_array_equal(f.level, g[p + "level"])
        np.testing.assert_array_equal(f.coords, g[p + "coords"])
        np.testing.assert_array_equal(f.parent, g[p + "parent"])
        np.testing.assert_array_equal(f.first_child, g[p + "first_child"])


def _rebuild_forest(g, coords):
    dim = coords.shape[0]
    f = of.Forest(*gu.unit_domain(dim), (int(g["root"]),) * dim)
    lv = int(g["n_levels"])
    if lv > 1:
        on.refine_near_wall(f, coords, float(g["d_spec"]), n_levels=lv, bins_per_axis=int(g["bins_refine"]))
    np.testing.assert_array_equal(f.coords, g["coords"])
    return f


@pytest.mark.parametrize("path", gu.files("links_"), ids=gu.ids(gu.files("links_")))
def test_cell_face_links_match_reference(path):
    g = gu.load(path)
    coords = gu.geometry(g)
    f = _rebuild_forest(g, coords)
    grid = ob.Grid(*gu.unit_domain(coords.shape[0]), int(g["bins_per_axis"]))
    bins = ob.fill_bins(coords, grid)
    dl = None if np.isnan(g["d_link_arg"]) else float(g["d_link_arg"])
    err = str(g["error"])
    if err:
        with pytest.raises(Capacity) as ei:
            on.cell_face_links(f, coords, bins, grid, d_link=dl, capacity=int(g["capacity"]))
        assert str(ei.value) == err
        return
    out = on.cell_face_links(f, coords, bins, grid, d_link=dl, capacity=int(g["capacity"]))
    assert out["d_link"] == float(g["d_link"])
    for k in ("block_ids", "cell_indices", "offsets", "face_ids"):
        np.testing.assert_array_equal(out[k], g[k])


# --- restated reference known-answer tests (forest / propagation / bins) ----


def test_known_neighbors():
    f = of.Forest(*gu.unit_domain(2), (4, 4))
    assert f.face_neighbors(5) == [(4,), (6,), (1,), (9,)]  # test_forest.py:187-190
    assert f.face_neighbors(0) == [(), (1,), (), (4,)]
    f.marks[5] = of.MARKED
    assert f.refine_marked(0) == 1
    assert f.first_child[5] == 16 and f.blocks_per_level() == [16, 4]
    assert f.face_neighbors(6)[0] == (17, 19)  # test_forest.py:197-204
    assert f.face_neighbors(17)[1] == (6,)


def test_known_propagation():
    f = of.Forest(*gu.unit_domain(2), (4, 4))
    f.marks[5] = of.MARKED
    on.propagate(f, 0, 0.1, rounds=1)
    assert set(np.flatnonzero(f.marks == of.MARKED)) == {5, 4, 6, 1, 9}
    assert on.propagation_rounds(0.05, 1 / 16) == 1
    assert on.propagation_rounds(0.1, 1 / 64) == 7
    f = of.Forest(*gu.unit_domain(2), (4, 4))
    f.marks[5] = of.MARKED
    f.refine_marked(0)
    child = f.leaves_at(1)[1]
    f.marks[child] = of.MARKED
    on.propagate(f, 0, 0.1, rounds=1)
    assert f.marks[6] == of.MARKED  # test_nearwall.py:164-171


def test_known_bins_and_errors():
    c = np.zeros((2, 2, 1), np.float32)
    c[0, :, 0], c[1, :, 0] = (0.25, 0.25), (0.75, 0.25)
    ids, counts, _ = ob.fill_bins(c, ob.Grid((0, 0), (1, 1), 2), spacing=0.5)
    assert counts.tolist() == [1, 1, 0, 0] and ids.tolist() == [0, 0]
    c[0, :, 0], c[1, :, 0] = (0.01, 0.5), (0.99, 0.5)
    with pytest.raises(Capacity):
        ob.fill_bins(c, ob.Grid((0, 0), (1, 1), 16), overlap_factor=10)
    c[0, :, 0], c[1, :, 0] = (0.5, 0.5), (1.5, 0.5)
    with pytest.raises(InvalidParameter):
        ob.fill_bins(c, ob.Grid((0, 0), (1, 1), 2))
    c[0, :, 0], c[1, :, 0] = (0.5, 0.5), (0.5, 0.5)
    with pytest.raises(InvalidParameter):
        ob.fill_bins(c, ob.Grid((0, 0), (1, 1), 2))


def test_max_level_and_intermediate():
    f = of.Forest(*gu.unit_domain(2), (1, 1), max_level=1)
    f.marks[0] = of.MARKED
    f.refine_marked(0)
    f.marks[f.leaves_at(1)] = of.MARKED
    with pytest.raises(InvalidParameter, match="max level"):
        f.refine_marked(1)
    f = of.Forest(*gu.unit_domain(2), (4, 4))
    f.marks[3] = of.INTERMEDIATE
    with pytest.raises(InvalidParameter, match="intermediate"):
        f.refine_marked(0)


def test_cell_centers_pattern():
    f = of.Forest(*gu.unit_domain(2), (1, 1))
    c = f.cell_centers([0])[0]
    m = np.array([0.125, 0.375, 0.625, 0.875], np.float32)
    np.testing.assert_array_equal(c[:4, 0], m)
    np.testing.assert_array_equal(c[:4, 1], np.full(4, 0.125, np.float32))
    np.testing.assert_array_equal(c[::4, 1], m)


def test_primitives_and_stl_roundtrip():
    from paper_2502_16310_b200 import shapes

    tris = shapes.icosphere_triangles(2)
    coords = og.stl(shapes.binary_stl_bytes(tris))
    np.testing.assert_array_equal(coords, np.transpose(tris.astype(np.float32), (1, 2, 0)))
    v, fcs = og.parse_primitives("circle 0.5 0.5 0.25 16\n# c\n")
    assert v.shape == (16, 2) and fcs.shape == (16, 2)
    v, fcs = og.parse_primitives("sphere 0.5 0.5 0.5 0.3 15 18")
    assert fcs.shape[0] == 2 * 18 + 2 * 13 * 18


def test_forest_invariant_checker_on_oracle_forests():
    """The full-size invariant checker (tests/forest_invariants.py) accepts
    the oracle's own refined forests (2D and 3D) and rejects a forest with a
    2:1 violation and one with a broken child link."""
    import pytest

    from forest_invariants import check_forest_invariants
    from oracle import forest as of
    from oracle import nearwall as on
    from paper_2502_16310_b200 import shapes

    tri = shapes.icosphere_triangles(2).astype(np.float32)
    coords = np.ascontiguousarray(np.transpose(tri, (1, 2, 0)))
    for dim, (dmin, dmax, root, geo, d) in {
        3: ((0, 0, 0), (1, 1, 1), (4, 4, 4), coords, 0.08),
        2: ((0, 0), (1, 1), (8, 8), None, 0.1),
    }.items():
        if geo is None:
            from oracle import geometry as og

            v, fcs = og.circle(0.5, 0.5, 0.25, 256)
            geo = og.index_to_coords(v, fcs)
        f = of.Forest(dmin, dmax, root)
        on.refine_near_wall(f, geo, d, n_levels=3, bins_per_axis=4)
        args = (f.level.astype(np.int64), f.coords.astype(np.int64), f.parent.astype(np.int64),
                f.first_child.astype(np.int64), np.asarray(root, np.int64))
        check_forest_invariants(*args)
    # a leaf at level 2 next to a level-0 leaf: split one child of a root block twice
    f = of.Forest((0, 0), (1, 1), (4, 4))
    f.marks[5] = 1
    f.refine_marked(0)
    kid = int(f.first_child[5])
    f.marks[kid] = 1
    f._append_children(np.array([kid]))
    with pytest.raises(AssertionError):
        check_forest_invariants(f.level.astype(np.int64), f.coords.astype(np.int64), f.parent.astype(np.int64),
                                f.first_child.astype(np.int64), np.asarray((4, 4), np.int64))
