"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden fixtures and the CPU oracle, bit-exact for every integer / boolean
output (bins, marks, forest arrays, links, flags) and float32-exact for q."""

import os

import numpy as np
import pytest
import torch

import golden_util as gu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ow():
    import paper_2502_16310_b200 as m
    from paper_2502_16310_b200 import _build

    _build.build()
    return m


def domain(ow, dim):
    return ow.Aabb(np.zeros(dim), np.ones(dim))


def geom_of(ow, g):
    c = gu.geometry(g)
    return ow.CoordListGeometry(c.shape[0], c)


# --------------------------------------------------------------------------- predicate
def test_predicate_triangle_bitexact(ow):
    g = gu.load(gu.files("pred_tri")[0])
    faces = np.ascontiguousarray(np.transpose(g["tri"], (1, 2, 0)))
    from paper_2502_16310_b200.distance import near_pairs

    got = near_pairs(g["pts"], faces, g["d"].astype(np.float32)).cpu().numpy()
    np.testing.assert_array_equal(got, g["mask"])


def test_predicate_edge_bitexact(ow):
    g = gu.load(gu.files("pred_edge")[0])
    faces = np.ascontiguousarray(np.transpose(g["seg"], (1, 2, 0)))
    from paper_2502_16310_b200.distance import near_pairs

    got = near_pairs(g["pts"], faces, g["d"].astype(np.float32)).cpu().numpy()
    np.testing.assert_array_equal(got, g["mask"])


# --------------------------------------------------------------------------- bins
@pytest.mark.parametrize("path", gu.files("bins_"), ids=gu.ids(gu.files("bins_")))
def test_fill_bins_bitexact(ow, path):
    g = gu.load(path)
    geom = geom_of(ow, g)
    grid = ow.BinGrid(domain(ow, geom.dim), int(g["bins_per_axis"]))
    h = None if np.isnan(g["spacing"]) else float(g["spacing"])
    bins = ow.fill_bins(geom, grid, spacing=h, overlap_factor=10 ** 6)
    ids, counts, offsets = bins.numpy()
    np.testing.assert_array_equal(counts, g["counts"])
    np.testing.assert_array_equal(offsets, g["offsets"])
    np.testing.assert_array_equal(ids, g["ids"])


# --------------------------------------------------------------------------- marking
@pytest.mark.parametrize("path", gu.files("mark_"), ids=gu.ids(gu.files("mark_")))
def test_marking_bitexact(ow, path):
    g = gu.load(path)
    geom = geom_of(ow, g)
    dim = geom.dim
    f = ow.init_root_grid(domain(ow, dim), (int(g["root"]),) * dim)
    b = int(g["bins_per_axis"])
    if b < 0:
        n = ow.mark_near_wall_naive(f, 0, geom, float(g["d_spec"]))
    else:
        grid = ow.BinGrid(domain(ow, dim), b)
        n = ow.mark_near_wall_binned(f, 0, geom, ow.fill_bins(geom, grid), grid, float(g["d_spec"]))
    assert n == int(g["n_marked"])
    np.testing.assert_array_equal(f.marks.cpu().numpy(), g["marks"])


# --------------------------------------------------------------------------- pipelines
@pytest.mark.parametrize("path", gu.files("pipe_"), ids=gu.ids(gu.files("pipe_")))
def test_refine_near_wall_bitexact(ow, path):
    g = gu.load(path)
    geom = geom_of(ow, g)
    dim = geom.dim
    f = ow.init_root_grid(domain(ow, dim), (int(g["root"]),) * dim)
    params = ow.NearWallParams(d_spec=float(g["d_spec"]), n_levels=int(g["n_levels"]),
                               strategy=str(g["strategy"]), bins_per_axis=int(g["bins_per_axis"]))
    res = ow.refine_near_wall(f, geom, params)
    assert res.marked_detected == g["marked_detected"].tolist()
    assert res.marked_refined == g["marked_refined"].tolist()
    assert [t.stage for t in res.timings] == g["stages"].tolist()
    assert f.n_blocks == int(g["n_blocks"])
    np.testing.assert_array_equal(f._level, g["level"])
    np.testing.assert_array_equal(f._coords, g["coords"])
    np.testing.assert_array_equal(f._parent, g["parent"])
    np.testing.assert_array_equal(f._first_child, g["first_child"])
    np.testing.assert_array_equal(f.marks.cpu().numpy(), g["marks"])
    assert f.blocks_per_level() == g["blocks_per_level"].tolist()
    assert f.leaves_per_level() == g["leaves_per_level"].tolist()
    if "bin_ids" in g:
        ids, counts, offsets = res.bins.numpy()
        np.testing.assert_array_equal(ids, g["bin_ids"])
        np.testing.assert_array_equal(counts, g["bin_counts"])


# --------------------------------------------------------------------------- forest units
def test_forest_units_bitexact(ow):
    g = gu.load(gu.files("forest_units")[0])
    f = ow.init_root_grid(domain(ow, 2), (8, 8))
    f.marks[[3, 17, 44]] = int(ow.RefineMark.MARKED)
    ow.propagate_marks(f, 0, d_spec=0.3)
    np.testing.assert_array_equal(f.marks.cpu().numpy(), g["prop8_marks"])

    f = ow.init_root_grid(domain(ow, 3), (4, 4, 4))
    f.marks[[5, 21, 42]] = int(ow.RefineMark.MARKED)
    f.refine_marked(0)
    lv1 = f.leaf_blocks_at(1)
    f.marks[lv1[::5]] = int(ow.RefineMark.MARKED)
    f.marks[[0, 63]] = int(ow.RefineMark.MARKED)
    ow.propagate_marks(f, 0, d_spec=0.3, rounds=2)
    np.testing.assert_array_equal(f.marks.cpu().numpy(), g["prop3d_marks"])
    np.testing.assert_array_equal(f._coords, g["prop3d_coords"])

    for dim, seed, rounds, root in ((2, 1, 3, 4), (2, 3, 4, 4), (3, 5, 3, 3), (3, 8, 4, 2)):
        rng = np.random.default_rng(seed)
        f = ow.init_root_grid(domain(ow, dim), (root,) * dim)
        splits = []
        for lv in range(rounds):
            leaves = f.leaf_blocks_at(lv).cpu().numpy()
            if len(leaves) == 0:
                break
            pick = leaves[rng.random(len(leaves)) < 0.4]
            f.marks[torch.as_tensor(pick, device=f.device)] = int(ow.RefineMark.MARKED)
            splits.append(f.refine_marked(lv))
        p = f"rand{dim}d_s{seed}_"
        assert splits == g[p + "splits"].tolist()
        np.testing.assert_array_equal(f._level, g[p + "level"])
        np.testing.assert_array_equal(f._coords, g[p + "coords"])
        np.testing.assert_array_equal(f._parent, g[p + "parent"])
        np.testing.assert_array_equal(f._first_child, g[p + "first_child"])


def test_forest_growth_callback(ow):
    """Capacity growth through the C callback keeps ids/coords intact."""
    f = ow.Forest(domain(ow, 3), (2, 2, 2), capacity=8)
    assert f.capacity >= 8
    for lv in range(4):
        leaves = f.leaf_blocks_at(lv)
        f.marks[leaves] = int(ow.RefineMark.MARKED)
        f.refine_marked(lv)
    assert f.blocks_per_level() == [8, 64, 512, 4096, 32768]
    assert f.capacity >= f.n_blocks


# --------------------------------------------------------------------------- links
@pytest.mark.parametrize("path", gu.files("links_"), ids=gu.ids(gu.files("links_")))
def test_cell_face_links_bitexact(ow, path):
    g = gu.load(path)
    geom = geom_of(ow, g)
    dim = geom.dim
    f = ow.init_root_grid(domain(ow, dim), (int(g["root"]),) * dim)
    if int(g["n_levels"]) > 1:
        ow.refine_near_wall(f, geom, ow.NearWallParams(d_spec=float(g["d_spec"]), n_levels=int(g["n_levels"]),
                                                       bins_per_axis=int(g["bins_refine"])))
    np.testing.assert_array_equal(f._coords, g["coords"])
    grid = ow.BinGrid(domain(ow, dim), int(g["bins_per_axis"]))
    bins = ow.fill_bins(geom, grid)
    dl = None if np.isnan(g["d_link_arg"]) else float(g["d_link_arg"])
    err = str(g["error"])
    if err:
        with pytest.raises(ow.CapacityError) as ei:
            ow.build_cell_face_links(f, geom, bins, grid, d_link=dl, capacity=int(g["capacity"]))
        assert str(ei.value) == err
        return
    links = ow.build_cell_face_links(f, geom, bins, grid, d_link=dl, capacity=int(g["capacity"]))
    assert links.d_link == float(g["d_link"])
    np.testing.assert_array_equal(links.block_ids.cpu().numpy(), g["block_ids"])
    np.testing.assert_array_equal(links.cell_indices.cpu().numpy(), g["cell_indices"])
    np.testing.assert_array_equal(links.offsets.cpu().numpy(), g["offsets"])
    np.testing.assert_array_equal(links.face_ids.cpu().numpy(), g["face_ids"])


# --------------------------------------------------------------------------- STL import
def test_stl_binary_and_ascii_import(ow, tmp_path):
    from paper_2502_16310_b200 import shapes
    from oracle import geometry as og

    tris = shapes.icosphere_triangles(3)
    data = shapes.binary_stl_bytes(tris)
    got = ow.import_stl_bytes(data).coords_numpy()
    np.testing.assert_array_equal(got, og.stl(data))
    # ASCII round trip of the unit cube (test_acceptance.py criterion 10)
    cube = np.array([[[0, 0, 0], [0, 1, 0], [1, 1, 0]], [[0, 0, 0], [1, 1, 0], [1, 0, 0]]], np.float64)
    lines = ["solid c"]
    for t in cube:
        lines += ["facet normal 0 0 1", "outer loop"] + [f"vertex {p[0]} {p[1]} {p[2]}" for p in t]
        lines += ["endloop", "endfacet"]
    lines.append("endsolid c")
    a = ow.import_stl_bytes("\n".join(lines).encode())
    np.testing.assert_array_equal(a.coords_numpy(), np.transpose(cube.astype(np.float32), (1, 2, 0)))
    with pytest.raises(ow.GeometryParseError):
        ow.import_stl_bytes(data[:-25])


def test_index_to_coords_gather(ow):
    from oracle import geometry as og

    ig = ow.generate_sphere((0.5, 0.5, 0.5), 0.3, 15, 18)
    v, fc = og.latlon_sphere(0.5, 0.5, 0.5, 0.3, 15, 18)
    np.testing.assert_array_equal(ig.vertices, v)
    np.testing.assert_array_equal(ow.index_to_coords(ig).coords_numpy(), og.index_to_coords(v, fc))


# --------------------------------------------------------------------------- errors
def test_error_behaviour(ow):
    c = np.zeros((2, 2, 1), np.float32)
    c[0, :, 0], c[1, :, 0] = (0.01, 0.5), (0.99, 0.5)
    g = ow.CoordListGeometry(2, c)
    with pytest.raises(ow.CapacityError, match="overlap_factor"):
        ow.fill_bins(g, ow.BinGrid(domain(ow, 2), 16), overlap_factor=10)
    c[0, :, 0], c[1, :, 0] = (0.5, 0.5), (1.5, 0.5)
    with pytest.raises(ow.InvalidParameterError, match="outside"):
        ow.fill_bins(ow.CoordListGeometry(2, c), ow.BinGrid(domain(ow, 2), 2))
    c[0, :, 0], c[1, :, 0] = (0.5, 0.5), (0.5, 0.5)
    with pytest.raises(ow.InvalidParameterError, match="degenerate"):
        ow.fill_bins(ow.CoordListGeometry(2, c), ow.BinGrid(domain(ow, 2), 2))
    f = ow.init_root_grid(domain(ow, 2), (1, 1), max_level=1)
    f.marks[0] = int(ow.RefineMark.MARKED)
    f.refine_marked(0)
    f.marks[f.leaf_blocks_at(1)] = int(ow.RefineMark.MARKED)
    with pytest.raises(ow.InvalidParameterError, match="max level"):
        f.refine_marked(1)
    f = ow.init_root_grid(domain(ow, 2), (4, 4))
    f.marks[3] = int(ow.RefineMark.INTERMEDIATE)
    with pytest.raises(ow.InvalidParameterError, match="intermediate"):
        f.refine_marked(0)
    with pytest.raises(ow.InvalidParameterError):
        ow.propagate_marks(f, 0, d_spec=0.1)


def test_known_answers(ow):
    f = ow.init_root_grid(domain(ow, 2), (4, 4))
    assert f.face_neighbors(5) == [(4,), (6,), (1,), (9,)]
    f.marks[5] = int(ow.RefineMark.MARKED)
    assert f.refine_marked(0) == 1
    assert list(f.block(5).children) == [16, 17, 18, 19]
    assert f.face_neighbors(6)[0] == (17, 19)
    assert f.face_neighbors(17)[1] == (6,)
    c = f.cell_centers(0).cpu().numpy()
    np.testing.assert_array_equal(c[:4, 0], np.array([0.03125, 0.09375, 0.15625, 0.21875], np.float32))
    assert ow.check_near_triangle((0.5, 0.25, 0.05), (0, 0, 0), (1, 0, 0), (0, 1, 0), 0.1)
    assert not ow.check_near_triangle((2, 2, 2), (0, 0, 0), (1, 0, 0), (0, 1, 0), 0.1)
    assert ow.check_near_edge((0.5, 0.05), (0, 0), (1, 0), 0.1)


# --------------------------------------------------------------------------- oracle-vs-GPU at other sizes
@pytest.mark.parametrize("dim,seed,n_faces,root,d,B", [
    (2, 101, 300, 8, 0.05, 4), (2, 102, 500, 16, 0.02, 16), (3, 103, 300, 6, 0.07, 3), (3, 104, 800, 8, 0.04, 8),
])
def test_pipeline_random_soups_vs_oracle(ow, dim, seed, n_faces, root, d, B):
    from oracle import forest as of
    from oracle import nearwall as on

    rng = np.random.default_rng(seed)
    anchors = rng.uniform(0.1, 0.9, (n_faces, dim))
    coords = np.empty((dim, dim, n_faces), np.float32)
    for j in range(dim):
        coords[j] = (anchors + (rng.uniform(-0.04, 0.04, (n_faces, dim)) if j else 0.0)).T.astype(np.float32)
    from oracle.geometry import first_degenerate

    while first_degenerate(coords) >= 0:
        coords[:, :, first_degenerate(coords)] += np.float32(1e-3)
    fo = of.Forest(np.zeros(dim), np.ones(dim), (root,) * dim)
    ro = on.refine_near_wall(fo, coords, d, n_levels=3, bins_per_axis=B)
    geom = ow.CoordListGeometry(dim, coords)
    fg = ow.init_root_grid(domain(ow, dim), (root,) * dim)
    rg = ow.refine_near_wall(fg, geom, ow.NearWallParams(d_spec=d, n_levels=3, bins_per_axis=B))
    assert rg.marked_detected == ro["marked_detected"]
    assert rg.cell_face_tests == ro["cell_face_tests"]
    np.testing.assert_array_equal(fg._coords, fo.coords)
    np.testing.assert_array_equal(fg._first_child, fo.first_child)


# --------------------------------------------------------------------------- lattice links vs oracle
@pytest.fixture(params=[(-1, 4), (-1, 8), (0, 4), (6, 8)], ids=["inline-fpw4", "inline-fpw8", "mt-all", "split6"])
def inline_units(request):
    """Shapes of the lattice sweep (results must not depend on them): every
    row tested inside the face pass with 4 or 8 faces per warp, every row
    through k_lat_mt, rows of > 6 cells through k_lat_mt."""
    from paper_2502_16310_b200 import _lib

    _lib.call("ow_lattice_tune", _lib.ctx(), *request.param)
    yield request.param
    _lib.call("ow_lattice_tune", _lib.ctx(), -1, -1)


@pytest.mark.parametrize("case", ["circle", "icosphere", "soup3d", "soup2d"])
def test_lattice_links_vs_oracle(ow, case, inline_units):
    from oracle import forest as of
    from oracle import lattice as ol
    from oracle import nearwall as on
    from paper_2502_16310_b200 import shapes

    if case == "circle":
        ig = ow.generate_circle((0.5, 0.5), 0.25, 200)
        coords = ow.index_to_coords(ig).coords_numpy()
        dim, root, d, lat = 2, 8, 0.1, "D2Q9"
    elif case == "icosphere":
        coords = np.ascontiguousarray(np.transpose(shapes.icosphere_triangles(3).astype(np.float32), (1, 2, 0)))
        dim, root, d, lat = 3, 4, 0.08, "D3Q19"
    elif case in ("soup3d", "soup2d"):
        # random small faces, some snapped onto cell-centre planes and block seams
        dim = 3 if case == "soup3d" else 2
        rng = np.random.default_rng(7 + dim)
        n = 400 if dim == 3 else 300
        anchors = rng.uniform(0.05, 0.95, (n, dim))
        snap = rng.random((n, dim)) < 0.3
        anchors[snap] = np.round(anchors[snap] * 128) / 128
        coords = np.zeros((dim, dim, n), np.float32)
        for j in range(dim):
            coords[j] = (anchors + (rng.uniform(-0.03, 0.03, (n, dim)) if j else 0.0)).T.astype(np.float32)
        from oracle.geometry import first_degenerate

        while first_degenerate(coords) >= 0:
            coords[:, :, first_degenerate(coords)] += np.float32(1e-3)
        root, d, lat = 4, 0.06, "D3Q27" if dim == 3 else "D2Q9"
    else:
        from golden.make_golden import cube_triangles  # noqa: F401  (recipe only; reference not imported)
        raise pytest.skip("covered by icosphere/circle")
    fo = of.Forest(np.zeros(dim), np.ones(dim), (root,) * dim)
    on.refine_near_wall(fo, coords, d, n_levels=3, bins_per_axis=4)
    ref = ol.lattice_links(fo, coords, lat)
    geom = ow.CoordListGeometry(dim, coords)
    fg = ow.init_root_grid(domain(ow, dim), (root,) * dim)
    ow.refine_near_wall(fg, geom, ow.NearWallParams(d_spec=d, n_levels=3, bins_per_axis=4))
    # the candidate grid only prunes work: explicit coarse bins and the auto grid agree
    for grid in (ow.BinGrid(domain(ow, dim), 4), None, ow.BinGrid(domain(ow, dim), 1)):
        ll = ow.build_lattice_links(fg, geom, grid, lat)
        np.testing.assert_array_equal(ll.leaves.cpu().numpy(), ref["leaves"])
        np.testing.assert_array_equal(ll.flags.cpu().numpy().view(np.uint32), ref["flags"])
        np.testing.assert_array_equal(ll.cells.cpu().numpy(), ref["boundary"])
        np.testing.assert_array_equal(ll.q.cpu().numpy(), ref["q"])
        assert ll.n_boundary > 0


@pytest.mark.parametrize("sub,root,lat", [(3, 8, "D3Q19"), (4, 8, "D3Q27"), (5, 16, "D3Q19")])
def test_lattice_face_pass_shapes_agree(ow, sub, root, lat):
    """The face pass shaped by the face extent (default) and with 4 or 16
    faces per warp counts the same candidate blocks, rows and link-face tests
    and produces identical flags, boundary rows and q."""
    from paper_2502_16310_b200 import _lib, shapes

    coords = np.ascontiguousarray(np.transpose(shapes.icosphere_triangles(sub).astype(np.float32), (1, 2, 0)))
    geom = ow.CoordListGeometry(3, coords)
    fg = ow.init_root_grid(domain(ow, 3), (root,) * 3)
    ow.refine_near_wall(fg, geom, ow.NearWallParams(d_spec=0.05, n_levels=3, bins_per_axis=8))
    out = []
    for fpw in (-1, 1, 2, 4, 16):
        _lib.call("ow_lattice_tune", _lib.ctx(), -1, fpw)
        try:
            ll = ow.build_lattice_links(fg, geom, None, lat)
            out.append(([t.cpu().numpy() for t in (ll.leaves, ll.flags, ll.cells, ll.q)], _lib.lattice_stats()))
        finally:
            _lib.call("ow_lattice_tune", _lib.ctx(), -1, -1)
    for arrs, stats in out[1:]:
        assert stats == out[0][1]
        for a, b in zip(arrs, out[0][0]):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("case", ["wall_between", "wall_on_centres", "wall_at_link_end", "square2d"])
def test_lattice_known_answers_on_gpu(ow, case):
    from oracle import forest as of
    from oracle import lattice as ol

    from test_oracle_lattice import _wall_z

    if case == "square2d":
        sq = np.array([[[0.3, 0.3], [0.7, 0.3]], [[0.7, 0.3], [0.7, 0.7]], [[0.7, 0.7], [0.3, 0.7]],
                       [[0.3, 0.7], [0.3, 0.3]]], np.float32)
        coords, dim, lat = np.ascontiguousarray(np.transpose(sq, (1, 2, 0))), 2, "D2Q9"
    else:
        z = {"wall_between": 0.2, "wall_on_centres": 0.125, "wall_at_link_end": 0.375}[case]
        coords, dim, lat = _wall_z(np.float32(z)), 3, "D3Q27"
    fo = of.Forest(np.zeros(dim), np.ones(dim), (1,) * dim)
    ref = ol.lattice_links(fo, coords, lat)
    fg = ow.init_root_grid(domain(ow, dim), (1,) * dim)
    ll = ow.build_lattice_links(fg, ow.CoordListGeometry(dim, coords), None, lat)
    np.testing.assert_array_equal(ll.flags.cpu().numpy().view(np.uint32), ref["flags"])
    np.testing.assert_array_equal(ll.cells.cpu().numpy(), ref["boundary"])
    np.testing.assert_array_equal(ll.q.cpu().numpy(), ref["q"])


# --------------------------------------------------------------------------- sharded driver (2 ranks, 1 GPU)
def _shard_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2502_16310_b200 as ow
        from paper_2502_16310_b200 import parallel, shapes

        torch.cuda.set_device(0)
        coords = np.ascontiguousarray(np.transpose(shapes.icosphere_triangles(3).astype(np.float32), (1, 2, 0)))
        geom = ow.CoordListGeometry(3, coords)
        f = ow.init_root_grid(ow.Aabb(np.zeros(3), np.ones(3)), (8, 8, 8))
        sh = parallel.Shard()
        res = ow.refine_near_wall(f, geom, ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8), shard=sh)
        ll = ow.build_lattice_links(f, geom, None, "D3Q19", shard=sh)
        q.put((rank, f._coords, f._first_child, res.marked_detected, res.cell_face_tests,
               ll.flags.cpu().numpy(), ll.cells.cpu().numpy(), ll.q.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_sharded_native_driver_matches_single_rank(ow):
    """Two ranks (gloo, one GPU) each mark half of every level through the
    native driver's exchange hook; the gathered forest equals one rank's."""
    import socket

    import torch.multiprocessing as mp

    from paper_2502_16310_b200 import shapes

    coords = np.ascontiguousarray(np.transpose(shapes.icosphere_triangles(3).astype(np.float32), (1, 2, 0)))
    geom = ow.CoordListGeometry(3, coords)
    f = ow.init_root_grid(ow.Aabb(np.zeros(3), np.ones(3)), (8, 8, 8))
    ref = ow.refine_near_wall(f, geom, ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8))
    lref = ow.build_lattice_links(f, geom, None, "D3Q19")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=500) for _ in procs]
    for p in procs:
        p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    for _, co, fc, md, t, fl, ce, qq in outs:
        np.testing.assert_array_equal(co, f._coords)
        np.testing.assert_array_equal(fc, f._first_child)
        assert md == ref.marked_detected and t == ref.cell_face_tests
        np.testing.assert_array_equal(fl, lref.flags.cpu().numpy())
        np.testing.assert_array_equal(ce, lref.cells.cpu().numpy())
        np.testing.assert_array_equal(qq, lref.q.cpu().numpy())


def _comm_worker(rank, world, port, q, sub, root, lattice, levels):
    import os

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2502_16310_b200 as ow
        from paper_2502_16310_b200 import parallel, pipeline, shapes

        torch.cuda.set_device(0)
        data = shapes.binary_stl_bytes(shapes.icosphere_triangles(sub))
        n = int.from_bytes(data[80:84], "little")
        rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
        comm = parallel.DeviceComm(64 << 20)
        plan = pipeline.GridPlan(ow.Aabb(np.zeros(3), np.ones(3)), (root,) * 3,
                                 ow.NearWallParams(d_spec=0.06, n_levels=levels, bins_per_axis=8), lattice,
                                 comm=comm, reuse_outputs=True)
        outs = []
        for _ in range(2):  # a second pass reuses the plan (epochs continue)
            gp = plan.run(rec, n, host=True)
            torch.cuda.synchronize()
            f, ll = gp.forest, gp.links
            outs.append((f._coords.copy(), f._first_child.copy(), f.marks.cpu().numpy(), gp.result.marked_detected,
                         gp.result.cell_face_tests, ll.flags.cpu().numpy(), ll.cells.cpu().numpy(),
                         ll.q.cpu().numpy(), gp.host_q(), bool(gp.reran)))
        q.put((rank, comm.status(), outs))
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("sub,root,lattice,levels", [(3, 8, "D3Q19", 3), (4, 8, "D3Q27", 4)])
def test_device_comm_fused_pass_matches_single_rank(ow, sub, root, lattice, levels):
    """Two ranks sharing one GPU run the fused GridPlan pass with a
    DeviceComm: work-balanced marking slices and equal lattice slices,
    exchanged by put / get kernels over CUDA-IPC-mapped memory with no host
    round trip in the level loop.  Every rank's forest, marks, statistics,
    lattice flags, boundary rows, q and packed host rows equal the
    single-rank pass, twice in a row (the exchange epochs continue)."""
    import socket

    import torch.multiprocessing as mp

    from paper_2502_16310_b200 import pipeline, shapes

    data = shapes.binary_stl_bytes(shapes.icosphere_triangles(sub))
    n = int.from_bytes(data[80:84], "little")
    rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
    ref = pipeline.GridPlan(ow.Aabb(np.zeros(3), np.ones(3)), (root,) * 3,
                            ow.NearWallParams(d_spec=0.06, n_levels=levels, bins_per_axis=8), lattice).run(
        rec, n, host=True)
    torch.cuda.synchronize()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_comm_worker, args=(r, 2, port, q, sub, root, lattice, levels)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=800) for _ in procs]
    for p in procs:
        p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    f, ll = ref.forest, ref.links
    for rank, status, outs in res:
        assert status == 0, f"rank {rank}: an exchange timed out"
        for k, (co, fc, mk, md, t, fl, ce, qq, hq, reran) in enumerate(outs):
            np.testing.assert_array_equal(co, f._coords)
            np.testing.assert_array_equal(fc, f._first_child)
            np.testing.assert_array_equal(mk, f.marks.cpu().numpy())
            assert md == ref.result.marked_detected and t == ref.result.cell_face_tests
            np.testing.assert_array_equal(fl, ll.flags.cpu().numpy())
            np.testing.assert_array_equal(ce, ll.cells.cpu().numpy())
            np.testing.assert_array_equal(qq, ll.q.cpu().numpy())
            np.testing.assert_array_equal(hq, ref.host_q())
            # the first pass of a plan may outgrow the initial forest capacity
            # and finish on the per-level host path (exchanging through the same
            # DeviceComm); the second pass is sized from it and stays on the device
            assert reran == (ref.reran if k == 0 else False)


def test_marking_dense_soup_single_root(ow):
    """One root block next to 12 000 faces: hundreds of bin chunks survive the
    union-box cull per block (grouped chunk rounds); the forest equals the
    oracle's for binned and naive marking."""
    from oracle import forest as of
    from oracle import nearwall as on

    rng = np.random.default_rng(11)
    n = 12000
    anchors = rng.uniform(0.3, 0.7, (n, 3))
    coords = np.zeros((3, 3, n), np.float32)
    for j in range(3):
        coords[j] = (anchors + (rng.uniform(-0.01, 0.01, (n, 3)) if j else 0.0)).T.astype(np.float32)
    from oracle.geometry import first_degenerate

    while first_degenerate(coords) >= 0:
        coords[:, :, first_degenerate(coords)] += np.float32(1e-3)
    for strategy, B in (("binned", 2), ("naive", 1)):
        fo = of.Forest(np.zeros(3), np.ones(3), (1, 1, 1))
        ro = on.refine_near_wall(fo, coords, 0.05, n_levels=3, bins_per_axis=B, strategy=strategy)
        fg = ow.init_root_grid(domain(ow, 3), (1, 1, 1))
        rg = ow.refine_near_wall(fg, ow.CoordListGeometry(3, coords),
                                 ow.NearWallParams(d_spec=0.05, n_levels=3, bins_per_axis=B, strategy=strategy))
        assert rg.marked_detected == ro["marked_detected"]
        np.testing.assert_array_equal(fg._coords, fo.coords)


# --------------------------------------------------------------------------- fused native pass
@pytest.mark.parametrize("capacity", [None, 600])
def test_geometry_to_grid_matches_per_function_path(ow, capacity):
    """ow_geometry_to_grid (one native call from STL records) equals the
    reference call sequence import_stl -> init_root_grid -> refine_near_wall
    -> build_lattice_links, array for array.  capacity=600 (512 roots): the
    device-resident level loop overflows and the pass reruns on the per-level
    host path, which grows the forest."""
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    tris = shapes.icosphere_triangles(3)
    data = shapes.binary_stl_bytes(tris)
    n = int.from_bytes(data[80:84], "little")
    rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8)
    plan = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q27", capacity=capacity)
    g1 = plan.run(rec, n)
    assert g1.reran == (capacity is not None)
    gp = plan.run(rec, n)  # second pass: outputs and capacity sized from the first
    assert not gp.reran
    geom = ow.import_stl_bytes(data)
    f = ow.init_root_grid(dom, (8, 8, 8))
    res = ow.refine_near_wall(f, geom, params)
    ll = ow.build_lattice_links(f, geom, None, "D3Q27")
    assert torch.equal(gp.geometry.coords, geom.coords)
    assert gp.result.marked_detected == res.marked_detected and gp.result.cell_face_tests == res.cell_face_tests
    assert gp.result.marked_refined == res.marked_refined
    for g in (g1, gp):
        assert g.result.marked_detected == res.marked_detected
        np.testing.assert_array_equal(g.forest._coords, f._coords)
        np.testing.assert_array_equal(g.forest._parent, f._parent)
        np.testing.assert_array_equal(g.forest.marks.cpu().numpy(), f.marks.cpu().numpy())
    np.testing.assert_array_equal(gp.forest._coords, f._coords)
    np.testing.assert_array_equal(gp.forest._first_child, f._first_child)
    assert gp.forest.blocks_per_level() == f.blocks_per_level()
    assert torch.equal(gp.result.bins.ids, res.bins.ids)
    for name in ("leaves", "flags", "cells", "q"):
        assert torch.equal(getattr(gp.links, name), getattr(ll, name)), name


def test_grid_plan_reuse_outputs(ow):
    """reuse_outputs=True: passes write into the plan's arrays; each pass
    (consumed before the next) equals a fresh plan's pass."""
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8)
    plan = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19", reuse_outputs=True)
    for sub in (3, 2, 3):  # geometry changes between passes
        tris = shapes.icosphere_triangles(sub)
        data = shapes.binary_stl_bytes(tris)
        n = int.from_bytes(data[80:84], "little")
        rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
        ref = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19").run(rec, n)
        gp = plan.run(rec, n)
        assert gp.result.marked_refined == ref.result.marked_refined
        np.testing.assert_array_equal(gp.forest._coords, ref.forest._coords)
        np.testing.assert_array_equal(gp.forest._parent, ref.forest._parent)
        assert torch.equal(gp.result.bins.ids, ref.result.bins.ids)
        for name in ("leaves", "flags", "cells", "q"):
            assert torch.equal(getattr(gp.links, name), getattr(ref.links, name)), name


def test_grid_plan_reuse_equal_sizes(ow):
    """reuse_outputs=True with equal output sizes between passes (the same
    geometry twice, then its cyclic coordinate permutation: same leaf and
    boundary counts, different faces and links).  The plan hands back the
    same LatticeLinks views (documented aliasing: a pass's results live
    until the next run) and every pass equals a fresh plan's."""
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8)
    plan = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19", reuse_outputs=True)
    tris = shapes.icosphere_triangles(3)
    prev = None
    for k, t in enumerate((tris, tris, tris[:, :, [1, 2, 0]])):
        data = shapes.binary_stl_bytes(t)
        n = int.from_bytes(data[80:84], "little")
        rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
        gp = plan.run(rec, n)
        ref = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19").run(rec, n)
        assert gp.forest.blocks_per_level() == ref.forest.blocks_per_level()
        np.testing.assert_array_equal(gp.forest._coords, ref.forest._coords)
        for name in ("leaves", "flags", "cells", "q"):
            assert torch.equal(getattr(gp.links, name), getattr(ref.links, name)), (k, name)
        if prev is not None and prev[0] == (gp.links.n_boundary, gp.links.leaves.numel()):
            assert gp.links is prev[1]  # same storage, same sizes: the cached views
        prev = ((gp.links.n_boundary, gp.links.leaves.numel()), gp.links)


def test_grid_plan_deferred_host_copies(ow):
    """run(host=True, defer=True) with two plans alternating over a stream of
    geometries (the e2e bench's pipeline): host copies of one pass overlap the
    next pass; after GridPass.wait() every pass's host results equal a
    synchronous pass's, and a plan's next pass does not clobber outputs its
    previous pass is still copying."""
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8)
    plans = [pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19", reuse_outputs=True) for _ in range(2)]
    geoms = [shapes.icosphere_triangles(s, radius=r) for s, r in ((3, 0.3), (3, 0.25), (2, 0.3), (3, 0.3))] * 2
    recs = []
    for t in geoms:
        data = shapes.binary_stl_bytes(t)
        recs.append((torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda(),
                     int.from_bytes(data[80:84], "little")))
    refs = []
    for rec, n in recs:
        r = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19").run(rec, n, host=True)
        torch.cuda.synchronize()
        refs.append({k: (v.clone() if isinstance(v, torch.Tensor) else [c.clone() for c in v])
                     for k, v in r.host.items()})
    pending = []
    deferred = 0
    for k, (rec, n) in enumerate(recs):
        gp = plans[k % 2].run(rec, n, host=True, defer=True)
        # (a pass whose results outgrow the buffers sized from its plan's last
        # pass falls back to synchronous copies; the others are deferred)
        deferred += int(gp.done is not None and bool(gp.host_copied & 8))
        pending.append((k, gp))
        if len(pending) == 2:  # the host reads step k-1 after step k is enqueued
            j, g = pending.pop(0)
            g.wait()
            _check_host(g.host, refs[j], j)
    assert deferred >= 4
    for j, g in pending:
        g.wait()
        _check_host(g.host, refs[j], j)


def _check_host(h, ref, j):
    import torch

    for key in ("level", "parent", "first_child", "marks", "cells", "flags", "q_packed"):
        assert torch.equal(h[key], ref[key]), (j, key)
    for a, b in zip(h["coords"], ref["coords"]):
        assert torch.equal(a, b), (j, "coords")


def test_grid_plan_graph_replay(ow):
    """stage_times=False: the device-resident level loop is captured as a CUDA
    graph on the second pass with unchanged inputs and replayed afterwards
    (ow_graph.cu; scans take their look-back epochs from the device).  Every
    pass — eager, capture, replays, a geometry change (eager again, then a new
    capture) — equals a fresh plan's pass, and the launch accounting counts
    the replayed kernels."""
    import torch

    from paper_2502_16310_b200 import _lib, pipeline, shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=4, bins_per_axis=8)
    plan = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19", reuse_outputs=True, stage_times=False)
    seq = [(3, 0.3)] * 5 + [(3, 0.25)] * 4 + [(3, 0.3)] * 2
    cache = {}
    for k, (sub, r) in enumerate(seq):
        data = shapes.binary_stl_bytes(shapes.icosphere_triangles(sub, radius=r))
        n = int.from_bytes(data[80:84], "little")
        rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
        if (sub, r) not in cache:
            ref = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19").run(rec, n)
            cache[(sub, r)] = (ref.forest._coords.copy(), ref.forest._first_child.copy(),
                               ref.forest.marks.cpu().numpy(), ref.result.marked_detected, ref.result.cell_face_tests,
                               [t.clone() for t in (ref.links.flags, ref.links.cells, ref.links.q)])
        l0 = _lib.launches()
        gp = plan.run(rec, n)
        torch.cuda.synchronize()
        co, fc, mk, md, t, lk = cache[(sub, r)]
        np.testing.assert_array_equal(gp.forest._coords, co, err_msg=f"pass {k}")
        np.testing.assert_array_equal(gp.forest._first_child, fc, err_msg=f"pass {k}")
        np.testing.assert_array_equal(gp.forest.marks.cpu().numpy(), mk, err_msg=f"pass {k}")
        assert gp.result.marked_detected == md and gp.result.cell_face_tests == t, k
        for a, b in zip((gp.links.flags, gp.links.cells, gp.links.q), lk):
            assert torch.equal(a, b), k
        assert _lib.launches() - l0 > 40, k  # replays count their kernels


def test_two_host_threads_concurrently(ow):
    """The entry points are safe to call from several host threads at once
    (SPEC.md:133, 218): each thread gets its own context, so two threads
    binning and linking different geometries on their own streams, many
    times over, reproduce the single-threaded results exactly."""
    import threading

    import torch

    from paper_2502_16310_b200 import shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    geoms = [ow.CoordListGeometry(3, np.ascontiguousarray(np.transpose(
        shapes.icosphere_triangles(s, radius=r).astype(np.float32), (1, 2, 0)))) for s, r in ((3, 0.3), (4, 0.25))]
    grids = [ow.BinGrid(dom, 8), ow.BinGrid(dom, 6)]

    def work(k):
        bins = ow.fill_bins(geoms[k], grids[k])
        f = ow.init_root_grid(dom, (8, 8, 8))
        ll = ow.build_lattice_links(f, geoms[k], None, "D3Q19")
        return [t.cpu() for t in (bins.ids, bins.counts, bins.offsets, ll.flags, ll.cells, ll.q)]

    ref = [work(0), work(1)]
    errors = []

    def thread(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(6):
                    got = work(k)
                    for a, b in zip(got, ref[k]):
                        if not torch.equal(a, b):
                            errors.append(k)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    ts = [threading.Thread(target=thread, args=(k,)) for k in (0, 1)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_geometry_to_grid_errors(ow):
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    tris = shapes.icosphere_triangles(2).astype(np.float32)
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=2, bins_per_axis=4)

    def run(t):
        data = shapes.binary_stl_bytes(t)
        rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
        return pipeline.geometry_to_grid(rec, len(t), dom, (4, 4, 4), params, "D3Q19")

    bad = tris.copy()
    bad[5, 1] = bad[5, 0]
    with pytest.raises(ow.InvalidParameterError, match="degenerate triangle .* at face 5"):
        run(bad)
    out = tris + np.float32(0.9)
    with pytest.raises(ow.InvalidParameterError, match="outside the forest domain"):
        run(out)
    # the face summary is read with the first bin-count readback: binning runs
    # on these faces first and must stay bounded (inf / NaN / huge faces)
    for val, msg in ((np.inf, "non-finite"), (np.nan, "non-finite")):
        bad = tris.copy()
        bad[7, 2, 1] = val
        with pytest.raises(ow.InvalidParameterError, match=msg):
            run(bad)
    bad = tris.copy()
    bad[7] *= np.float32(1e6)  # a valid but enormous face (its sample walk would be ~1e16 samples)
    with pytest.raises(ow.InvalidParameterError, match="outside the forest domain"):
        run(bad)
    # degenerate beats outside (the reference validates faces first)
    bad = tris + np.float32(0.9)
    bad[3, 1] = bad[3, 0]
    with pytest.raises(ow.InvalidParameterError, match="degenerate triangle .* at face 3"):
        run(bad)
    # the plan is usable after errors
    f = run(tris).forest
    assert f.n_blocks > 64


def test_geometry_to_grid_naive_strategy(ow):
    """Fused pass with the naive strategy (no bins, so the face summary is
    settled before the first marking pass) equals the per-function path."""
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    tris = shapes.icosphere_triangles(2).astype(np.float32)
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, strategy="naive")
    data = shapes.binary_stl_bytes(tris)
    rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
    gp = pipeline.geometry_to_grid(rec, len(tris), dom, (4, 4, 4), params, "D3Q19")
    f2 = ow.init_root_grid(dom, (4, 4, 4))
    res = ow.refine_near_wall(f2, gp.geometry, params)
    np.testing.assert_array_equal(gp.forest._coords, f2._coords)
    np.testing.assert_array_equal(gp.forest._level, f2._level)
    assert gp.result.marked_detected == res.marked_detected


def test_native_driver_capacity_fallbacks(ow):
    """A forest created with the minimum capacity overflows inside the device
    refinement: the driver finishes on the host path (grow + rebalance) and the
    forest equals the oracle's."""
    from oracle import forest as of
    from oracle import nearwall as on
    from paper_2502_16310_b200 import shapes

    coords = np.ascontiguousarray(np.transpose(shapes.icosphere_triangles(3).astype(np.float32), (1, 2, 0)))
    fo = of.Forest(np.zeros(3), np.ones(3), (4, 4, 4))
    ro = on.refine_near_wall(fo, coords, 0.08, n_levels=3, bins_per_axis=4)
    fg = ow.init_root_grid(domain(ow, 3), (4, 4, 4), capacity=1)  # minimum capacity (1024 blocks): overflows
    rg = ow.refine_near_wall(fg, ow.CoordListGeometry(3, coords),
                             ow.NearWallParams(d_spec=0.08, n_levels=3, bins_per_axis=4))
    assert fg.n_blocks > 1024
    assert rg.marked_detected == ro["marked_detected"]
    assert rg.marked_refined == ro["marked_refined"]
    np.testing.assert_array_equal(fg._coords, fo.coords)
    np.testing.assert_array_equal(fg._first_child, fo.first_child)


# --------------------------------------------------------------------------- VTK export
def test_export_vtk_byte_identical(ow, tmp_path):
    """export_vtk of GPU-refined forests is byte-identical to the reference's
    export_vtk of the reference's forests (vtk_io.py:17-69)."""
    import hashlib

    from golden_util import GOLDEN, load
    from paper_2502_16310_b200 import shapes

    g = load(os.path.join(GOLDEN, "vtk_cases.npz"))
    geoms = {
        "circle256": lambda: ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.25, 256)),
        "icosphere3": lambda: ow.import_stl_bytes(shapes.binary_stl_bytes(shapes.icosphere_triangles(3))),
    }
    for i in range(2):
        name = str(g[f"case{i}_name"])
        root, d, levels, b = g[f"case{i}_params"]
        geom = geoms[name]()
        f = ow.init_root_grid(domain(ow, geom.dim), (int(root),) * geom.dim)
        ow.refine_near_wall(f, geom, ow.NearWallParams(d_spec=float(d), n_levels=int(levels), bins_per_axis=int(b)))
        path = tmp_path / f"{name}.vtk"
        ow.export_vtk(f, str(path), title=f"case {name}")
        data = path.read_bytes()
        head = bytes(g[f"case{i}_head"])
        assert data[: len(head)] == head, name
        assert len(data) == int(g[f"case{i}_bytes"]), name
        assert hashlib.sha256(data).hexdigest() == str(g[f"case{i}_sha"]), name


def test_bin_density_sweep_csv(ow, tmp_path):
    """sweep() runs one pipeline per B (B=1 naive) and writes the reference's
    CSV schema; blocks_marked / blocks_final match separate runs."""
    from paper_2502_16310_b200 import report

    geom = ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.25, 400))
    dom = ow.Aabb((0, 0), (1, 1))
    rows = report.sweep(geom, dom, (16, 16), 0.1, 3, [1, 2, 4, 8], out_csv=str(tmp_path / "s.csv"), verbose=False)
    lines = (tmp_path / "s.csv").read_text().splitlines()
    assert lines[0] == report.SWEEP_CSV_HEADER and len(lines) == 5
    for r in rows:
        f = ow.init_root_grid(dom, (16, 16))
        res = ow.refine_near_wall(f, geom, ow.NearWallParams(d_spec=0.1, n_levels=3, bins_per_axis=r.bins_per_axis,
                                                             strategy="naive" if r.bins_per_axis == 1 else "binned"))
        assert r.blocks_marked == res.total_marked and r.blocks_final == sum(f.leaves_per_level())
        assert r.bin_setup_ms >= 0 and r.face_detect_ms > 0 and r.total_ms > 0


def test_geometry_to_grid_host_results(ow):
    """run(host=True): the side-stream / tail copies into the plan's pinned
    buffers equal the device results (forest arrays, boundary cells, q), also
    on a first pass whose buffer estimate is too small (host fallback copy)."""
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    data = shapes.binary_stl_bytes(shapes.icosphere_triangles(3))
    n = int.from_bytes(data[80:84], "little")
    rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
    plan = pipeline.GridPlan(ow.Aabb(np.zeros(3), np.ones(3)), (8, 8, 8),
                             ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8), "D3Q19")
    for _ in range(2):
        gp = plan.run(rec, n, host=True)
        torch.cuda.current_stream().synchronize()
        h, f = gp.host, gp.forest
        np.testing.assert_array_equal(h["level"].numpy(), f._level)
        np.testing.assert_array_equal(np.stack([c.numpy() for c in h["coords"]], 1), f._coords)
        np.testing.assert_array_equal(h["parent"].numpy(), f._parent)
        np.testing.assert_array_equal(h["first_child"].numpy(), f._first_child)
        np.testing.assert_array_equal(h["marks"].numpy(), f.marks.cpu().numpy())
        np.testing.assert_array_equal(h["cells"].numpy().view(np.uint32).astype(np.int64), gp.links.cells.cpu().numpy())
        _check_packed_rows(gp)


def _check_packed_rows(gp):
    """Packed host rows (flag word + q of the set bits) == the device links."""
    h, ll = gp.host, gp.links
    cells = ll.cells.cpu().numpy()
    np.testing.assert_array_equal(h["cells"].numpy().view(np.uint32).astype(np.int64), cells)
    flags = ll.flags.cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(h["flags"].numpy().view(np.uint32), flags[cells])
    q = ll.q.cpu().numpy()
    assert h["q_packed"].numel() == int((q >= 0).sum())
    np.testing.assert_array_equal(gp.host_q(), q)


def test_geometry_to_grid_packed_rows_2d(ow):
    """The packed host rows of a 2D pass (16-cell blocks, D2Q9), native and
    first-pass fallback packing."""
    import torch

    from paper_2502_16310_b200 import pipeline

    geom = ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.25, 256))
    plan = pipeline.GridPlan(ow.Aabb((0, 0), (1, 1)), (8, 8),
                             ow.NearWallParams(d_spec=0.1, n_levels=3, bins_per_axis=8), "D2Q9")
    for _ in range(2):
        gp = plan.run(geometry=geom, host=True)
        torch.cuda.current_stream().synchronize()
        assert gp.links.n_boundary > 0
        _check_packed_rows(gp)


# --------------------------------------------------------------------------- predicate vs referee sampler
def test_gpu_referee_sampler_matches_reference_run(ow):
    """GPU predicate-vs-referee sampling reproduces the reference's recorded
    acceptance numbers (test_output.txt:11,14: 1e5 samples, 0 disagreements
    outside the band, 918 / 968 in band) and its FP64 exact distances equal the
    oracle's restatement of the referee bit for bit."""
    from oracle import predicate as op
    from paper_2502_16310_b200 import validate

    assert validate.check_triangle_predicate_oracle(2024, 100000) == (0, 918, 0)
    assert validate.check_edge_predicate_oracle(2025, 100000) == (0, 968, 0)
    tri, pts, d = validate.sample_triangle_cases(7, 3000)
    _, exact = validate.referee_pairs(tri, pts, d)
    ref = [op.exact_point_triangle_distance(pts[i], tri[i, 0], tri[i, 1], tri[i, 2]) for i in range(3000)]
    np.testing.assert_array_equal(exact, np.asarray(ref))
    seg, pts2, d2 = validate.sample_edge_cases(8, 3000)
    _, exact2 = validate.referee_pairs(seg, pts2, d2)
    ref2 = [op.point_segment_distance(pts2[i], seg[i, 0], seg[i, 1]) for i in range(3000)]
    np.testing.assert_array_equal(exact2, np.asarray(ref2))


def test_ascii_stl_native_fast_path(ow, tmp_path):
    """The native ASCII parser gives the reference parser's float32 vertices
    (float() then one rounding) on valid text, including Python-only float
    spellings (underscores, inf/nan, '5.', '.5'), and defers every error to
    the reference-faithful parser (same messages and line numbers)."""
    import ctypes as C

    from paper_2502_16310_b200 import _lib, geometry
    from paper_2502_16310_b200 import shapes

    tris = shapes.icosphere_triangles(2).astype(np.float32)
    lines = ["solid s"]
    for t in tris:
        lines += [" facet normal 0 0 1", "  outer loop"]
        lines += ["   vertex %r %r %r" % (float(v[0]), float(v[1]), float(v[2])) for v in t]
        lines += ["  endloop", " endfacet"]
    lines.append("endsolid s")
    data = ("\n".join(lines) + "\n").encode()
    g = ow.import_stl_bytes(data)
    np.testing.assert_array_equal(g.coords_numpy(), np.ascontiguousarray(np.transpose(tris, (1, 2, 0))))
    odd = (b"solid x facet normal 1_0 0 .5e-1_0 outer loop vertex 1_0.2_5 0.25 1e-4_0 vertex +.5 5. 1e-3 "
           b"vertex 1 2 3 endloop endfacet endsolid x")
    out = np.empty((2, 3, 3), np.float32)
    n = C.c_int64(0)
    err = (C.c_int64 * 5)()
    assert _lib.lib().ow_parse_ascii_stl(odd, len(odd), out.ctypes.data_as(C.c_void_p), 2, C.byref(n), err) == 0
    ref = np.asarray([[float("1_0.2_5"), 0.25, float("1e-4_0")], [0.5, 5.0, 1e-3], [1, 2, 3]], np.float64)
    np.testing.assert_array_equal(out[0], ref.astype(np.float32))
    for bad, msg in ((b"solid x\nfacet normal 0 0 0\nouter loop\nvertex 0x1p3 2 3\n", "expected a number"),
                     (b"solid x\nfacet normal 0 0 0\nouter lop\n", "expected 'loop'"),
                     (b"solid x\nfacet normal 0 0 0\n", "unexpected end of file")):
        with pytest.raises(ow.GeometryParseError, match=msg):
            geometry._parse_ascii(bad, "f.stl")


_PDL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
import paper_2502_16310_b200 as ow
from paper_2502_16310_b200 import pipeline, shapes
data = shapes.binary_stl_bytes(shapes.icosphere_triangles(4))
n = int.from_bytes(data[80:84], "little")
rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
plan = pipeline.GridPlan(ow.Aabb(np.zeros(3), np.ones(3)), (8, 8, 8),
                         ow.NearWallParams(d_spec=0.05, n_levels=3, bins_per_axis=8), "D3Q19")
gp = plan.run(rec, n)
f, ll = gp.forest, gp.links
np.savez(sys.argv[1], level=f._level, coords=f._coords, parent=f._parent, marks=f.marks.cpu().numpy(),
         flags=ll.flags.cpu().numpy(), cells=ll.cells.cpu().numpy(), q=ll.q.cpu().numpy())
"""


def test_pdl_off_matches_pdl_on(ow, tmp_path):
    """Every kernel is launched with programmatic dependent launch (kernels
    wait on griddepcontrol.wait before touching memory); the same fused pass
    launched without it (OW_PDL=0, fresh process) is identical array for array."""
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for pdl in ("1", "0"):
        path = str(tmp_path / f"pdl{pdl}.npz")
        env = dict(os.environ, OW_PDL=pdl)
        r = subprocess.run([sys.executable, "-c", _PDL_SCRIPT, path, repo], env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[pdl] = np.load(path)
    for k in out["1"].files:
        np.testing.assert_array_equal(out["1"][k], out["0"][k], err_msg=k)
    assert len(out["1"]["cells"]) > 0


_PREFILTER_SCRIPT = r"""
import glob, json, os, sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
sys.path.insert(0, os.path.join(sys.argv[2], "tests"))
import paper_2502_16310_b200 as ow
from paper_2502_16310_b200 import pipeline, shapes
import golden_util as gu
from test_gpu_parity import domain, geom_of
stats = {}
for path in gu.files("pipe_"):  # every golden pipeline, bit-exact under this process's launch knobs
    g = gu.load(path)
    geom = geom_of(ow, g)
    dim = geom.dim
    f = ow.init_root_grid(domain(ow, dim), (int(g["root"]),) * dim)
    params = ow.NearWallParams(d_spec=float(g["d_spec"]), n_levels=int(g["n_levels"]),
                               strategy=str(g["strategy"]), bins_per_axis=int(g["bins_per_axis"]))
    res = ow.refine_near_wall(f, geom, params)
    assert res.marked_detected == g["marked_detected"].tolist(), path
    assert res.marked_refined == g["marked_refined"].tolist(), path
    np.testing.assert_array_equal(f._coords, g["coords"], err_msg=path)
    np.testing.assert_array_equal(f.marks.cpu().numpy(), g["marks"], err_msg=path)
    # T per pass (algorithmic); the evaluated / sphere / cull counts depend on
    # when another warp's hit ends a block's remaining items, so not compared
    stats[os.path.basename(path)] = list(map(int, res.cell_face_tests))
data = shapes.binary_stl_bytes(shapes.icosphere_triangles(4))
n = int.from_bytes(data[80:84], "little")
rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
plan = pipeline.GridPlan(ow.Aabb(np.zeros(3), np.ones(3)), (16, 16, 16),
                         ow.NearWallParams(d_spec=0.05, n_levels=3, bins_per_axis=8), "D3Q19")
for _ in range(3):  # sizing, device-sized, graph replay
    gp = plan.run(rec, n)
f, ll = gp.forest, gp.links
np.savez(sys.argv[1], level=f._level, coords=f._coords, parent=f._parent, marks=f.marks.cpu().numpy(),
         flags=ll.flags.cpu().numpy(), q=ll.q.cpu().numpy())
json.dump(stats, open(sys.argv[1] + ".json", "w"))
"""


def test_mark_prefilter_many_blocks_per_warp(ow, tmp_path):
    """The block pass prefilters a warp's leaf blocks one per lane when it has
    more than one (only blocks with a non-empty bin take the warp-wide path),
    under the dynamic schedule (runs of K blocks from a counter) and the
    static stride (OW_MARK_DYN=0).
    With the grid capped at 2 CTAs (8 warps: every level has many blocks per
    warp) the golden pipelines stay bit-exact with their statistics equal to
    the same capped run without the prefilter, and the fused pass is array for
    array the default launch's."""
    import json
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out, st = {}, {}
    for tag, env in (("pf", {"OW_MARK_MAX_CTAS": "2", "OW_MARK_PREFILTER": "1"}),
                     ("nopf", {"OW_MARK_MAX_CTAS": "2", "OW_MARK_PREFILTER": "0"}),
                     ("static", {"OW_MARK_MAX_CTAS": "2", "OW_MARK_DYN": "0"}),
                     ("default", {})):
        path = str(tmp_path / f"{tag}.npz")
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, "-c", _PREFILTER_SCRIPT, path, repo], env=e, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        out[tag] = np.load(path)
        st[tag] = json.load(open(path + ".json"))
    assert st["pf"] == st["nopf"] == st["static"] == st["default"]
    for tag in ("pf", "nopf", "static"):
        for k in out["default"].files:
            np.testing.assert_array_equal(out[tag][k], out["default"][k], err_msg=f"{tag}:{k}")
