"""Parity at BASELINE.json's full configuration sizes (GPU).

The oracle cannot run whole C3/C4-sized pipelines in test time, so these
tests check (a) the C3 forest against SHA-256 digests of the real
reference's own run (tests/golden/bigpipe_*.npz, made by make_golden.py), and
(b) sampled, size-independent restatements: lattice flags and q of random
finest cells recomputed by the oracle's watertight segment test over the faces whose
AABB meets each link's AABB, and level-0 marks of random blocks recomputed by
the oracle's marking.  Every comparison is bit-exact.
"""

import hashlib
import os

import numpy as np
import pytest
import torch

from forest_invariants import check_forest_invariants
from golden_util import GOLDEN, load

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def ow():
    import paper_2502_16310_b200 as ow

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return ow


def _records(tris):
    from paper_2502_16310_b200 import shapes

    data = shapes.binary_stl_bytes(tris)
    n = int.from_bytes(data[80:84], "little")
    return data, n, torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()


def test_c3_forest_matches_reference_digests(ow):
    """C3 (69 936-triangle bumpy sphere, 16^3 root, d=0.05, 4 levels, B=8):
    the fused native pass reproduces the reference's forest arrays bit for bit."""
    from paper_2502_16310_b200 import pipeline, shapes

    g = load(os.path.join(GOLDEN, "bigpipe_bumpy70k_r16_d0.05_L4_binned_B8.npz"))
    data, n, rec = _records(shapes.bumpy_sphere_triangles())
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.05, n_levels=4, bins_per_axis=8)
    gp = pipeline.GridPlan(dom, (16, 16, 16), params, "D3Q27").run(rec, n)
    assert _sha(gp.geometry.coords_numpy()) == str(g["geom_sha"])
    f = gp.forest
    assert gp.result.marked_detected == g["marked_detected"].tolist()
    assert gp.result.marked_refined == g["marked_refined"].tolist()
    assert f.blocks_per_level() == g["blocks_per_level"].tolist()
    assert f.leaves_per_level() == g["leaves_per_level"].tolist()
    n_b = int(g["n_blocks"])
    assert f.n_blocks == n_b
    assert _sha(f._level.astype(np.int16)) == str(g["sha_level"])
    assert _sha(f._coords.astype(np.int64)) == str(g["sha_coords"])
    assert _sha(f._parent.astype(np.int32)) == str(g["sha_parent"])
    assert _sha(f._first_child.astype(np.int32)) == str(g["sha_first_child"])
    assert _sha(f.marks.cpu().numpy().astype(np.int8)) == str(g["sha_marks"])
    assert int(gp.result.bins.ids.numel()) == int(g["n_bin_entries"])
    assert _sha(gp.result.bins.ids.cpu().numpy()) == str(g["sha_bin_ids"])
    assert _sha(gp.result.bins.counts.cpu().numpy()) == str(g["sha_bin_counts"])


def _sampled_lattice(coords, centers, h, dirs):
    """Oracle flags / q of the given cells (oracle/lattice.py definition, with
    candidate faces gathered through a coarse hash of the face boxes)."""
    from oracle import lattice as ol

    F32 = np.float32
    lo = coords.min(axis=0).T
    hi = coords.max(axis=0).T
    G = 128
    glo = np.floor(lo * G).astype(np.int64).clip(0, G - 1)
    ghi = np.floor(hi * G).astype(np.int64).clip(0, G - 1)
    # (bucket, face) pairs of a uniform G^3 hash of the face boxes, sorted by bucket
    ext = ghi - glo + 1
    reps = ext.prod(axis=1)
    face = np.repeat(np.arange(coords.shape[2]), reps)
    k = np.arange(face.size) - np.repeat(np.cumsum(reps) - reps, reps)
    bx = glo[face, 0] + k % ext[face, 0]
    by = glo[face, 1] + (k // ext[face, 0]) % ext[face, 1]
    bz = glo[face, 2] + k // (ext[face, 0] * ext[face, 1])
    key = (bz * G + by) * G + bx
    order = np.argsort(key, kind="stable")
    key, face = key[order], face[order]
    nq = len(dirs)
    flags = np.zeros(len(centers), np.uint32)
    q = np.full((len(centers), nq), F32(-1.0), F32)
    dvs = [(dirs[i].astype(F32) * h).astype(F32) for i in range(nq)]
    for ci, x in enumerate(centers):
        slo = np.floor((x - 2 * h) * G).astype(np.int64).clip(0, G - 1)
        shi = np.floor((x + 2 * h) * G).astype(np.int64).clip(0, G - 1)
        parts = []
        for gz in range(slo[2], shi[2] + 1):
            for gy in range(slo[1], shi[1] + 1):
                k0 = (gz * G + gy) * G
                a, b = np.searchsorted(key, [k0 + slo[0], k0 + shi[0] + 1])
                parts.append(face[a:b])
        cand = np.unique(np.concatenate(parts))
        if cand.size == 0:
            continue
        for i in range(1, nq):
            en = (x + dvs[i]).astype(F32)
            llo, lhi = np.minimum(x, en), np.maximum(x, en)
            ov = np.all((lo[cand] <= lhi) & (hi[cand] >= llo), axis=1)
            fs = cand[ov]
            if fs.size == 0:
                continue
            hit, t = ol.link_hits(np.broadcast_to(x, (fs.size, 3)), dvs[i], coords[:, :, fs])
            if hit.any():
                flags[ci] |= np.uint32(1 << i)
                q[ci, i] = (t[hit] + F32(0.0)).min()
    return flags, q


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_lattice_sampled_cells_full_size(ow, cfg):
    """Flags and q of 1500 random finest cells (a third of them boundary cells)
    of the full C3 / C4 / C5 pass equal the oracle's per-cell restatement."""
    import bench
    from oracle import lattice as ol
    from paper_2502_16310_b200 import pipeline

    c = bench.CONFIGS[cfg]
    data = bench.make_input(c)
    n = int.from_bytes(data[80:84], "little")
    rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=c["d"], n_levels=c["levels"], bins_per_axis=c["B"])
    gp = pipeline.GridPlan(dom, (c["root"],) * 3, params, c["lattice"]).run(rec, n)
    ll, f = gp.links, gp.forest
    flags = ll.flags.cpu().numpy().view(np.uint32)
    cells = ll.cells.cpu().numpy()
    qg = ll.q.cpu().numpy()
    rng = np.random.default_rng(5)
    pick = np.concatenate([rng.choice(cells, 500, replace=False),
                           rng.choice(flags.size, 1000, replace=False)])
    pick = np.unique(pick)
    leaves = ll.leaves.cpu().numpy()
    cen = f.cell_centers_many(torch.from_numpy(leaves[pick // 64])).cpu().numpy()
    cen = cen[np.arange(pick.size), pick % 64]
    level = ll.level
    h = (np.asarray(dom.extent) / (np.asarray(f.root_dims) * (1 << level)) / 4.0).astype(np.float32)
    coords = gp.geometry.coords_numpy()
    dirs = ol.directions(c["lattice"])
    fo, qo = _sampled_lattice(coords, cen.astype(np.float32), h, dirs)
    np.testing.assert_array_equal(flags[pick], fo)
    row = np.searchsorted(cells, pick)
    isb = (row < cells.size) & (cells[np.minimum(row, cells.size - 1)] == pick)
    assert np.array_equal(isb, fo != 0)
    np.testing.assert_array_equal(qg[row[isb]], qo[isb])


def test_marks_sampled_blocks_full_size(ow):
    """Level-0 binned marks of 400 random root blocks of the full C4 pass (1M
    triangles, B=32) equal the oracle's marking of the same blocks."""
    import bench
    from oracle import binning as ob
    from oracle import forest as of
    from oracle import nearwall as on

    c = bench.CONFIGS["C4"]
    data = bench.make_input(c)
    geom = ow.import_stl_bytes(data)
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    grid = ow.BinGrid(dom, c["B"])
    bins = ow.fill_bins(geom, grid)
    f = ow.init_root_grid(dom, (c["root"],) * 3)
    ow.mark_near_wall_binned(f, 0, geom, bins, grid, c["d"])
    marks = f.marks.cpu().numpy()
    rng = np.random.default_rng(9)
    near = np.flatnonzero(marks)
    pick = np.unique(np.concatenate([rng.choice(near, 200, replace=False), rng.choice(marks.size, 200, replace=False)]))
    coords = geom.coords_numpy()
    fo = of.Forest(np.zeros(3), np.ones(3), (c["root"],) * 3)
    go = ob.Grid(np.zeros(3), np.ones(3), c["B"])
    ids, counts, offsets = (a.cpu().numpy() for a in (bins.ids, bins.counts, bins.offsets))
    # hide all other root blocks from the oracle's leaf list: it marks only `pick`
    keep = np.zeros(fo.n, bool)
    keep[pick] = True
    fo.first_child[~keep] = 0
    on.mark(fo, 0, coords, c["d"], (ids, counts, offsets), go)
    np.testing.assert_array_equal(marks[pick], fo.marks[pick])


def _grid_pass(ow, cfg):
    import bench
    from paper_2502_16310_b200 import pipeline

    c = bench.CONFIGS[cfg]
    data = bench.make_input(c)
    n = int.from_bytes(data[80:84], "little")
    rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=c["d"], n_levels=c["levels"], bins_per_axis=c["B"])
    return c, dom, pipeline.GridPlan(dom, (c["root"],) * 3, params, c["lattice"]).run(rec, n)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C5"])
def test_lattice_referee_full_size(ow, cfg):
    """Lattice links of the full C2 / C3 / C5 pass against the FP64 referee
    (oracle/referee.py, independent of the definition's float32 arithmetic)
    on 40 000 finest cells near the closed, star-shaped surface: no link
    whose ends lie on opposite sides of the surface (beyond a 1e-6 band) is
    left unflagged, no link the FP64 test crosses with margin is unflagged,
    q equals the FP64 crossing parameter within 1e-5, and (icospheres,
    convex) no link with both ends inside is flagged.  Prints the counts."""
    from oracle import lattice as ol
    from oracle import referee as rf

    c, dom, gp = _grid_pass(ow, cfg)
    ll, f = gp.links, gp.forest
    flags = ll.flags.cpu().numpy().view(np.uint32)
    cells, qg = ll.cells.cpu().numpy(), ll.q.cpu().numpy()
    leaves = ll.leaves.cpu().numpy()
    h = (np.asarray(dom.extent) / (np.asarray(f.root_dims) * (1 << ll.level)) / 4.0).astype(np.float32)
    coords = gp.geometry.coords_numpy()
    surf = rf.StarSurface(coords)
    rng = np.random.default_rng(17)
    # candidate cells: a radial band around the surface, then the exact side distance
    cen_all = []
    for b0 in range(0, leaves.size, 1 << 16):
        lb = torch.from_numpy(leaves[b0:b0 + (1 << 16)])
        cen_all.append(f.cell_centers_many(lb).cpu().numpy().reshape(-1, 3))
    cen_all = np.concatenate(cen_all)
    r = np.linalg.norm(cen_all.astype(np.float64) - 0.5, axis=1)
    band = np.flatnonzero((r > 0.3 * 0.8) & (r < 0.3 * 1.2))
    band = rng.choice(band, min(band.size, 400000), replace=False)
    sd = surf.signed(cen_all[band])
    near = band[np.abs(sd) < 3.0 * float(h.max())]
    pick = np.sort(rng.choice(near, min(near.size, 40000), replace=False))
    dvs = (ol.directions(c["lattice"]).astype(np.float32) * h).astype(np.float32)
    q = np.full((pick.size, len(dvs)), -1.0, np.float32)
    row = np.searchsorted(cells, pick)
    isb = (row < cells.size) & (cells[np.minimum(row, cells.size - 1)] == pick)
    q[isb] = qg[row[isb]]
    res = rf.check_links(cen_all[pick], dvs, flags[pick], q, coords, surf)
    print(f"{cfg} referee: {res}")
    assert res["crossing"] > 10000 and res["crossing_missed"] == 0
    assert res["unflagged_hit"] == 0
    assert res["q_checked"] > 10000 and res["q_bad"] == 0
    if c["kind"] == "ico":
        assert res["inside_flagged"] == 0


def _forest_arrays(f):
    n = f.n_blocks
    return (f._level[:n].astype(np.int64), f._coords[:n].astype(np.int64), f._parent[:n].astype(np.int64),
            f._first_child[:n].astype(np.int64))


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_forest_invariants_full_size(ow, cfg):
    """The fused C4 / C5 pass produces a consistent forest: parent/child
    links, child coordinates and id allocation, and 2:1 balance across every
    block face, checked over all ~10^5-10^6 blocks."""
    c, dom, gp = _grid_pass(ow, cfg)
    f = gp.forest
    level, coords, parent, fc = _forest_arrays(f)
    check_forest_invariants(level, coords, parent, fc, np.asarray(f.root_dims, np.int64))
    assert f.blocks_per_level()[-1] > 0 and len(f.blocks_per_level()) == c["levels"]


def test_bins_full_size_c5_vs_oracle(ow):
    """C5 (5.24 M triangles, B=64): the device bin CSR equals the oracle's
    fill_bins (binning.py:200-266 restated) array for array."""
    from oracle import binning as ob

    c, dom, gp = _grid_pass(ow, "C5")
    coords = gp.geometry.coords_numpy()
    ids, counts, offsets = ob.fill_bins(coords, ob.Grid(np.zeros(3), np.ones(3), c["B"]))
    b = gp.result.bins
    np.testing.assert_array_equal(b.counts.cpu().numpy(), counts)
    np.testing.assert_array_equal(b.offsets.cpu().numpy(), offsets)
    np.testing.assert_array_equal(b.ids.cpu().numpy(), ids)


def _oracle_forest_of(f):
    from oracle import forest as of

    level, coords, parent, fc = _forest_arrays(f)
    fo = of.Forest(np.asarray(f.domain.min, np.float64), np.asarray(f.domain.max, np.float64), f.root_dims)
    fo.level, fo.coords = level.astype(np.int16), coords
    fo.parent, fo.first_child = parent.astype(np.int32), fc.astype(np.int32)
    fo.marks = np.zeros(level.size, np.int8)
    return fo


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_marks_every_level_sampled_full_size(ow, cfg):
    """Per-function path of the full C4 / C5 configuration (fill_bins ->
    binned marking -> propagation -> refinement per level): after each
    device marking pass, >= 1000 sampled leaves of that level (half of them
    marked) are re-marked by the oracle (nearwall.py:253-311 restated) on the
    device forest's own leaves — every level, bit-exact — and the resulting
    forest equals the fused GridPlan pass's, array for array."""
    from oracle import binning as ob
    from oracle import nearwall as on

    import bench

    c = bench.CONFIGS[cfg]
    geom = ow.import_stl_bytes(bench.make_input(c))
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    grid = ow.BinGrid(dom, c["B"])
    f = ow.init_root_grid(dom, (c["root"],) * 3)
    coords = geom.coords_numpy()
    go = ob.Grid(np.zeros(3), np.ones(3), c["B"])
    rng = np.random.default_rng(23)
    checked = []
    for L in range(c["levels"] - 1):
        bins = ow.fill_bins(geom, grid)
        ow.mark_near_wall_binned(f, L, geom, bins, grid, c["d"])
        marks = f.marks.cpu().numpy()
        leaves = f.leaf_blocks_at(L).cpu().numpy()
        mk = leaves[marks[leaves] == 1]
        pick = np.unique(np.concatenate([rng.choice(mk, min(mk.size, 500), replace=False),
                                         rng.choice(leaves, min(leaves.size, 1000), replace=False)]))
        fo = _oracle_forest_of(f)
        hide = np.ones(fo.n, bool)
        hide[pick] = False
        hide &= fo.first_child == -1
        fo.first_child[hide] = 0  # only the picked leaves are leaves for the oracle
        ib = (a.cpu().numpy() for a in (bins.ids, bins.counts, bins.offsets))
        on.mark(fo, L, coords, c["d"], tuple(ib), go)
        np.testing.assert_array_equal(marks[pick], fo.marks[pick], err_msg=f"level {L}")
        checked.append((L, pick.size, int((marks[pick] == 1).sum())))
        ow.propagate_marks(f, L, c["d"])
        f.refine_marked(L)
    print(f"{cfg} sampled marks (level, blocks, marked): {checked}")
    _, _, gp = _grid_pass(ow, cfg)
    g = gp.forest
    assert f.n_blocks == g.n_blocks
    for a, b in zip(_forest_arrays(f), _forest_arrays(g)):
        np.testing.assert_array_equal(a, b)
