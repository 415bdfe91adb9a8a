"""Generate the golden parity fixtures by running the REAL reference here.

Runs only in the build container, where the reference package is importable
from /root/reference/pkg/src (read-only; never copied).  Every fixture is a
compressed .npz under tests/golden/ holding the reference's outputs for one
case; small geometries are stored inline, large ones by a SHA-256 of their
float32 coordinates plus the recipe that regenerates them, so the fixtures
stay small and the GPU box (which has no /root/reference) can still check.

    python tests/golden/make_golden.py            # regenerate everything
    python tests/golden/make_golden.py bins marks # subsets

Reference calls used (file:line under /root/reference/pkg/src/octowall):
fill_bins binning.py:200, near_triangle_mask distance.py:167,
near_edge_mask distance.py:216, mark_near_wall_naive nearwall.py:217,
mark_near_wall_binned nearwall.py:253, propagate_marks nearwall.py:321,
Forest.refine_marked forest.py:331, refine_near_wall nearwall.py:430,
build_cell_face_links nearwall.py:522, import_stl geometry.py:319,
validate.sample_triangle_cases validate.py:49.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import octowall as ow  # noqa: E402  (the reference)
from octowall import validate as ow_validate  # noqa: E402
from octowall.forest import RefineMark  # noqa: E402

from paper_2502_16310_b200 import shapes  # noqa: E402

UNIT2 = ow.Aabb((0.0, 0.0), (1.0, 1.0))
UNIT3 = ow.Aabb((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))

INLINE_LIMIT = 40_000  # faces; larger geometries are stored by hash + recipe


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# geometry recipes (each must be reproducible from the product package too)
# ---------------------------------------------------------------------------


def edge_geometry(*edges):
    coords = np.zeros((2, 2, len(edges)), np.float32)
    for k, (a, b) in enumerate(edges):
        coords[0, :, k] = a
        coords[1, :, k] = b
    return ow.CoordListGeometry(2, coords)


def random_soup(seed, dim, n_faces, lo=0.1, hi=0.9):
    """Same recipe as the reference's test_backends.random_soup (seeded)."""
    rng = np.random.default_rng(seed)
    anchors = rng.uniform(lo, hi, (n_faces, dim))
    coords = np.empty((dim, dim, n_faces), dtype=np.float32)
    for j in range(dim):
        offs = rng.uniform(-0.05, 0.05, (n_faces, dim))
        pts = np.clip(anchors + (offs if j else 0.0), lo, hi)
        coords[j] = pts.T.astype(np.float32)
    g = ow.CoordListGeometry(dim, coords)
    for _ in range(20):
        try:
            ow.geometry.validate_faces(g)
            return g
        except Exception:
            coords = coords + rng.uniform(1e-4, 2e-4, coords.shape).astype(np.float32)
            coords = np.clip(coords, lo, hi)
            g = ow.CoordListGeometry(dim, coords)
    ow.geometry.validate_faces(g)
    return g


def seam_soup(seed, n_faces, bins_per_axis, ulps=2):
    """Stress soup: small triangles whose vertices sit within a few float32
    ulps of bin seams (SURVEY.md finding 5: samples escaping the vertex-AABB
    bin range)."""
    rng = np.random.default_rng(seed)
    seams = np.arange(1, bins_per_axis) / bins_per_axis
    base = rng.choice(seams, size=(n_faces, 3)).astype(np.float32)
    jitter = rng.integers(-ulps, ulps + 1, size=(n_faces, 3, 3))
    tri = np.repeat(base[:, None, :], 3, axis=1)
    # spread vertices a little, keep several near seams
    spread = rng.uniform(-0.03, 0.03, (n_faces, 3, 3)).astype(np.float32)
    keep_on_seam = rng.random((n_faces, 3, 3)) < 0.6
    tri = np.where(keep_on_seam, tri, tri + spread)
    # ulp jitter
    step = np.spacing(np.abs(tri).astype(np.float32))
    tri = (tri + jitter.astype(np.float32) * step).astype(np.float32)
    tri = np.clip(tri, 0.01, 0.99).astype(np.float32)
    coords = np.transpose(tri, (1, 2, 0)).copy()
    g = ow.CoordListGeometry(3, coords)
    # drop degenerate faces deterministically
    c = coords.astype(np.float64)
    u, v, w = c[1] - c[0], c[2] - c[0], c[2] - c[1]
    scale = np.maximum(np.maximum((u * u).sum(0), (v * v).sum(0)), (w * w).sum(0))
    cr = np.cross(u.T, v.T).T
    area = np.sqrt((cr * cr).sum(0))
    ok = (scale > 0) & (area >= 1e-9 * scale)
    return ow.CoordListGeometry(3, coords[:, :, ok].copy())


def cube_triangles(lo=0.0, hi=1.0):
    quads = [(0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (2, 3, 7, 6), (0, 4, 7, 3), (1, 2, 6, 5)]
    v = np.array([[x, y, z] for z in (lo, hi) for y in (lo, hi) for x in (lo, hi)], np.float64)
    tris = []
    for a, b, c, d in quads:
        tris.append([v[a], v[b], v[c]])
        tris.append([v[a], v[c], v[d]])
    return np.asarray(tris)


def tris_geometry(tris):
    t = np.asarray(tris, np.float32)
    return ow.CoordListGeometry(3, np.transpose(t, (1, 2, 0)).copy())


def stl_geometry(tris):
    """Round-trip through binary STL bytes and the reference importer."""
    data = shapes.binary_stl_bytes(tris)
    with tempfile.NamedTemporaryFile(suffix=".stl", delete=False) as f:
        f.write(data)
        path = f.name
    try:
        return ow.import_stl(path)
    finally:
        os.unlink(path)


GEOMS = {
    "circle16": lambda: ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.25, 16)),
    "circle64": lambda: ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.25, 64)),
    "circle123": lambda: ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.3, 123)),
    "circle128": lambda: ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.25, 128)),
    "circle256": lambda: ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.25, 256)),
    "circle257": lambda: ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.3, 257)),
    "circle400": lambda: ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.3, 400)),
    "circle12800": lambda: ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.25, 12800)),
    "sphere8x12": lambda: ow.index_to_coords(ow.generate_sphere((0.5, 0.5, 0.5), 0.3, 8, 12)),
    "sphere15x18": lambda: ow.index_to_coords(ow.generate_sphere((0.5, 0.5, 0.5), 0.3, 15, 18)),
    "sphere224x250": lambda: ow.index_to_coords(ow.generate_sphere((0.5, 0.5, 0.5), 0.3, 224, 250)),
    "soup2d_0": lambda: random_soup(0, 2, 200),
    "soup2d_7": lambda: random_soup(7, 2, 200),
    "soup2d_3": lambda: random_soup(3, 2, 120),
    "soup2d_4": lambda: random_soup(4, 2, 120),
    "soup2d_11": lambda: random_soup(11, 2, 150),
    "soup2d_12": lambda: random_soup(12, 2, 150),
    "soup3d_1": lambda: random_soup(1, 3, 200),
    "soup3d_9": lambda: random_soup(9, 3, 200),
    "soup3d_5": lambda: random_soup(5, 3, 120),
    "soup3d_13": lambda: random_soup(13, 3, 150),
    "seam3d_b3": lambda: seam_soup(31, 3000, 3),
    "seam3d_b6": lambda: seam_soup(32, 3000, 6),
    "seam2d": lambda: ow.CoordListGeometry(
        2,
        np.array(
            [[[0.5, 0.25, 0.124999], [0.25, 0.5, 0.125]], [[0.5, 0.75, 0.375], [0.75, 0.5, 0.375]]],
            np.float32,
        ),
    ),
    "edge_mid": lambda: edge_geometry(((0.25, 0.25), (0.75, 0.25))),
    "edge_long": lambda: edge_geometry(((0.01, 0.5), (0.99, 0.5))),
    "edge_iso": lambda: edge_geometry(((0.4, 0.4), (0.6, 0.4))),
    "cube": lambda: tris_geometry(cube_triangles()),
    "cube_inset": lambda: tris_geometry(cube_triangles(0.2, 0.8)),
    "icosphere5": lambda: stl_geometry(shapes.icosphere_triangles(5)),
    "icosphere3": lambda: stl_geometry(shapes.icosphere_triangles(3)),
    "bumpy70k": lambda: stl_geometry(shapes.bumpy_sphere_triangles()),
}

_geom_cache = {}


def geom(name):
    if name not in _geom_cache:
        _geom_cache[name] = GEOMS[name]()
    return _geom_cache[name]


def geom_payload(name):
    g = geom(name)
    out = {"geom_name": np.array(name), "geom_dim": np.int64(g.dim), "geom_sha": np.array(sha(g.coords))}
    if g.n_faces <= INLINE_LIMIT:
        out["geom_coords"] = g.coords
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    return path


def forest_payload(f, prefix=""):
    n = f.n_blocks
    return {
        prefix + "n_blocks": np.int64(n),
        prefix + "level": f._level[:n].copy(),
        prefix + "coords": f._coords[:n].copy(),
        prefix + "parent": f._parent[:n].copy(),
        prefix + "first_child": f._first_child[:n].copy(),
        prefix + "marks": f.marks[:n].copy(),
        prefix + "blocks_per_level": np.asarray(f.blocks_per_level(), np.int64),
        prefix + "leaves_per_level": np.asarray(f.leaves_per_level(), np.int64),
    }


def domain_for(dim):
    return UNIT2 if dim == 2 else UNIT3


# ---------------------------------------------------------------------------
# fixture groups
# ---------------------------------------------------------------------------

BIN_CASES = [
    ("circle16", 1, None), ("circle400", 8, None), ("circle400", 7, None), ("circle257", 5, None),
    ("circle123", 4, None), ("circle12800", 8, None), ("circle12800", 16, None),
    ("sphere8x12", 4, None), ("sphere15x18", 1, None), ("sphere224x250", 8, None),
    ("soup2d_0", 1, None), ("soup2d_0", 3, None), ("soup2d_0", 8, None),
    ("soup2d_7", 3, None), ("soup3d_1", 1, None), ("soup3d_1", 3, None), ("soup3d_1", 8, None),
    ("soup3d_9", 8, None), ("seam2d", 2, None), ("seam2d", 4, None), ("seam2d", 8, None),
    ("seam3d_b3", 3, None), ("seam3d_b6", 6, None), ("seam3d_b6", 12, None),
    ("edge_mid", 2, 0.5), ("cube", 2, None), ("cube", 8, None), ("cube_inset", 5, None),
    ("icosphere5", 8, None), ("icosphere5", 16, None), ("icosphere3", 4, None),
    ("circle400", 8, 0.01), ("soup3d_9", 4, 0.02),
]


def gen_bins():
    for gname, b, spacing in BIN_CASES:
        g = geom(gname)
        grid = ow.BinGrid(domain_for(g.dim), b)
        t0 = time.perf_counter()
        bins = ow.fill_bins(g, grid, spacing=spacing, backend="parallel", overlap_factor=10**6)
        dt = time.perf_counter() - t0
        tag = f"bins_{gname}_B{b}" + (f"_h{spacing}" if spacing else "")
        save(tag, **geom_payload(gname), bins_per_axis=np.int64(b),
             spacing=np.float64(spacing if spacing else np.nan),
             ids=bins.ids, counts=bins.counts, offsets=bins.offsets)
        print(f"{tag}: E={bins.ids.size} ({dt:.2f}s)")


PRED_N = 20000


def gen_predicate():
    tri, pts, d = ow_validate.sample_triangle_cases(2024, PRED_N)
    coords = np.transpose(tri, (1, 2, 0)).copy()
    mask = ow.distance.near_triangle_mask(pts[:, 0], pts[:, 1], pts[:, 2], coords, d)
    save("pred_tri", tri=tri, pts=pts, d=d, mask=mask)
    seg, pts2, d2 = ow_validate.sample_edge_cases(2025, PRED_N)
    coords2 = np.transpose(seg, (1, 2, 0)).copy()
    mask2 = ow.distance.near_edge_mask(pts2[:, 0], pts2[:, 1], coords2, d2)
    save("pred_edge", seg=seg, pts=pts2, d=d2, mask=mask2)
    print(f"pred: tri hits {int(mask.sum())}/{PRED_N}, edge hits {int(mask2.sum())}/{PRED_N}")


MARK_CASES = [
    # (geom, root, d, B or None for naive)
    ("soup2d_3", 6, 0.07, None), ("soup2d_3", 6, 0.07, 4), ("soup2d_4", 6, 0.2, None),
    ("soup2d_4", 6, 0.2, 4), ("soup3d_5", 6, 0.1, None), ("soup3d_5", 6, 0.1, 4),
    ("circle256", 32, 0.1, None), ("circle256", 32, 0.1, 1), ("circle128", 16, 0.15, 8),
    ("circle128", 16, 0.15, None), ("sphere15x18", 8, 0.1, None), ("sphere15x18", 8, 0.1, 1),
    ("icosphere3", 8, 0.05, 4), ("icosphere3", 8, 0.05, None), ("cube_inset", 6, 0.07, 3),
    ("circle12800", 64, 0.1, 8),
]


def gen_marks():
    for gname, root, d, b in MARK_CASES:
        g = geom(gname)
        dom = domain_for(g.dim)
        f = ow.init_root_grid(dom, (root,) * g.dim)
        t0 = time.perf_counter()
        if b is None:
            n = ow.mark_near_wall_naive(f, 0, g, d, backend="parallel")
            tag = f"mark_{gname}_r{root}_d{d}_naive"
        else:
            grid = ow.BinGrid(dom, b)
            bins = ow.fill_bins(g, grid, backend="parallel")
            n = ow.mark_near_wall_binned(f, 0, g, bins, grid, d, backend="parallel")
            tag = f"mark_{gname}_r{root}_d{d}_B{b}"
        dt = time.perf_counter() - t0
        save(tag, **geom_payload(gname), root=np.int64(root), d_spec=np.float64(d),
             bins_per_axis=np.int64(-1 if b is None else b), n_marked=np.int64(n),
             marks=f.marks[: f.n_blocks].copy())
        print(f"{tag}: {n} marked ({dt:.2f}s)")


PIPE_CASES = [
    # (geom, root, d, levels, strategy, B)
    ("circle256", 8, 0.1, 3, "binned", 8),
    ("circle256", 16, 0.1, 3, "naive", 1),
    ("circle256", 16, 0.1, 3, "binned", 4),
    ("circle64", 8, 0.1, 2, "binned", 4),
    ("soup2d_11", 4, 0.08, 3, "binned", 4),
    ("soup2d_12", 4, 0.08, 3, "naive", 1),
    ("soup3d_13", 4, 0.08, 3, "binned", 2),
    ("sphere15x18", 8, 0.1, 3, "binned", 4),
    ("icosphere3", 8, 0.05, 3, "binned", 4),
    ("cube_inset", 4, 0.05, 3, "binned", 2),
    ("circle12800", 64, 0.1, 3, "binned", 8),
    ("circle12800", 64, 0.1, 3, "naive", 1),
    ("icosphere5", 16, 0.05, 3, "binned", 8),
]


def gen_pipelines():
    for gname, root, d, levels, strategy, b in PIPE_CASES:
        g = geom(gname)
        dom = domain_for(g.dim)
        f = ow.init_root_grid(dom, (root,) * g.dim)
        params = ow.NearWallParams(d_spec=d, n_levels=levels, strategy=strategy, bins_per_axis=b,
                                   backend="parallel")
        t0 = time.perf_counter()
        res = ow.refine_near_wall(f, g, params)
        dt = time.perf_counter() - t0
        tag = f"pipe_{gname}_r{root}_d{d}_L{levels}_{strategy}_B{b}"
        extra = {}
        if res.bins is not None:
            extra = dict(bin_ids=res.bins.ids, bin_counts=res.bins.counts, bin_offsets=res.bins.offsets)
        save(tag, **geom_payload(gname), root=np.int64(root), d_spec=np.float64(d),
             n_levels=np.int64(levels), strategy=np.array(strategy), bins_per_axis=np.int64(b),
             marked_detected=np.asarray(res.marked_detected, np.int64),
             marked_refined=np.asarray(res.marked_refined, np.int64),
             stages=np.array([t.stage for t in res.timings]),
             **forest_payload(f), **extra)
        print(f"{tag}: blocks {f.blocks_per_level()} detect {res.marked_detected} "
              f"refined {res.marked_refined} ({dt:.1f}s)")


BIG_PIPE_CASES = [
    # C3 of BASELINE.json at full size: bunny-scale bumpy lat-lon sphere (69 936 triangles) as
    # binary STL, 16^3 root, d = 0.05, 4 levels, B = 8.  Arrays are too large to commit, so the
    # fixture holds SHA-256 digests of the forest arrays and the bin CSR plus the counts.
    ("bumpy70k", 16, 0.05, 4, "binned", 8),
]


def gen_bigpipes():
    for gname, root, d, levels, strategy, b in BIG_PIPE_CASES:
        g = geom(gname)
        dom = domain_for(g.dim)
        f = ow.init_root_grid(dom, (root,) * g.dim)
        params = ow.NearWallParams(d_spec=d, n_levels=levels, strategy=strategy, bins_per_axis=b,
                                   backend="parallel")
        t0 = time.perf_counter()
        res = ow.refine_near_wall(f, g, params)
        dt = time.perf_counter() - t0
        n = f.n_blocks
        tag = f"bigpipe_{gname}_r{root}_d{d}_L{levels}_{strategy}_B{b}"
        save(tag, geom_name=np.array(gname), geom_sha=np.array(sha(g.coords)), root=np.int64(root),
             d_spec=np.float64(d), n_levels=np.int64(levels), strategy=np.array(strategy),
             bins_per_axis=np.int64(b), n_blocks=np.int64(n),
             marked_detected=np.asarray(res.marked_detected, np.int64),
             marked_refined=np.asarray(res.marked_refined, np.int64),
             blocks_per_level=np.asarray(f.blocks_per_level(), np.int64),
             leaves_per_level=np.asarray(f.leaves_per_level(), np.int64),
             sha_level=np.array(sha(f._level[:n].astype(np.int16))),
             sha_coords=np.array(sha(f._coords[:n].astype(np.int64))),
             sha_parent=np.array(sha(f._parent[:n].astype(np.int32))),
             sha_first_child=np.array(sha(f._first_child[:n].astype(np.int32))),
             sha_marks=np.array(sha(f.marks[:n].astype(np.int8))),
             sha_bin_ids=np.array(sha(res.bins.ids.astype(np.int32))),
             sha_bin_counts=np.array(sha(res.bins.counts.astype(np.int32))),
             n_bin_entries=np.int64(res.bins.ids.size))
        print(f"{tag}: blocks {f.blocks_per_level()} detect {res.marked_detected} "
              f"refined {res.marked_refined} E={res.bins.ids.size} ({dt:.1f}s)")


VTK_CASES = [
    # (geometry, root, d, levels, B): forests refined by the reference, exported by its export_vtk
    ("circle256", 8, 0.1, 3, 8),
    ("icosphere3", 4, 0.08, 3, 4),
]


def gen_vtk():
    from octowall.vtk_io import export_vtk

    out = {}
    for i, (gname, root, d, levels, b) in enumerate(VTK_CASES):
        g = geom(gname)
        f = ow.init_root_grid(domain_for(g.dim), (root,) * g.dim)
        ow.refine_near_wall(f, g, ow.NearWallParams(d_spec=d, n_levels=levels, bins_per_axis=b, backend="parallel"))
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "f.vtk")
            export_vtk(f, path, title=f"case {gname}")
            data = open(path, "rb").read()
        out[f"case{i}_name"] = np.array(gname)
        out[f"case{i}_params"] = np.array([root, d, levels, b], np.float64)
        out[f"case{i}_sha"] = np.array(hashlib.sha256(data).hexdigest())
        out[f"case{i}_bytes"] = np.int64(len(data))
        out[f"case{i}_head"] = np.frombuffer(data[:2000], np.uint8)
        print(f"vtk {gname}: {len(data)} bytes")
    save("vtk_cases", **out)


def gen_forest_units():
    """Propagation / refinement known answers beyond the reference's own asserts."""
    out = {}
    # propagation on an 8x8 root grid with scattered seeds (test_nearwall.py:149)
    f = ow.init_root_grid(UNIT2, (8, 8))
    f.marks[[3, 17, 44]] = RefineMark.MARKED
    ow.propagate_marks(f, 0, d_spec=0.3)
    out["prop8_marks"] = f.marks[: f.n_blocks].copy()
    # 3D propagation over a mixed-level forest
    f = ow.init_root_grid(UNIT3, (4, 4, 4))
    f.marks[[5, 21, 42]] = RefineMark.MARKED
    f.refine_marked(0)
    lv1 = f.leaf_blocks_at(1)
    f.marks[lv1[::5]] = RefineMark.MARKED
    f.marks[[0, 63]] = RefineMark.MARKED
    ow.propagate_marks(f, 0, d_spec=0.3, rounds=2)
    out.update(forest_payload(f, "prop3d_"))
    # random multi-level refinements (test_forest.py:152 recipe), 2D and 3D
    for dim, seed, rounds, root in ((2, 1, 3, 4), (2, 3, 4, 4), (3, 5, 3, 3), (3, 8, 4, 2)):
        rng = np.random.default_rng(seed)
        f = ow.init_root_grid(domain_for(dim), (root,) * dim)
        splits = []
        for lv in range(rounds):
            leaves = f.leaf_blocks_at(lv)
            if len(leaves) == 0:
                break
            pick = leaves[rng.random(len(leaves)) < 0.4]
            f.marks[pick] = RefineMark.MARKED
            splits.append(f.refine_marked(lv))
        out.update(forest_payload(f, f"rand{dim}d_s{seed}_"))
        out[f"rand{dim}d_s{seed}_splits"] = np.asarray(splits, np.int64)
    save("forest_units", **out)
    print("forest_units:", {k: v.shape for k, v in out.items() if k.endswith("level")})


LINK_CASES = [
    # (geom, root, d_spec, levels, B_refine, B_links, d_link, capacity)
    ("circle64", 8, 0.1, 2, 4, 4, 0.01, 16),
    ("circle64", 8, 0.1, 2, 4, 4, None, 64),
    ("edge_iso", 4, None, 1, None, 2, 0.05, 16),
    ("circle16", 4, None, 1, None, 1, 0.2, 16),
    ("sphere15x18", 8, 0.1, 2, 4, 4, None, 64),
    ("icosphere3", 8, 0.05, 2, 4, 4, None, 64),
    ("circle64", 4, None, 1, None, 1, 0.3, 2),  # capacity error
    ("circle256", 16, 0.1, 3, 8, 8, None, 64),
]


def gen_links():
    for gname, root, d, levels, b_ref, b_link, d_link, cap in LINK_CASES:
        g = geom(gname)
        dom = domain_for(g.dim)
        f = ow.init_root_grid(dom, (root,) * g.dim)
        if levels > 1:
            ow.refine_near_wall(f, g, ow.NearWallParams(d_spec=d, n_levels=levels, bins_per_axis=b_ref,
                                                        backend="parallel"))
        grid = ow.BinGrid(dom, b_link)
        bins = ow.fill_bins(g, grid, backend="parallel")
        tag = f"links_{gname}_r{root}_L{levels}_B{b_link}_dl{d_link}_c{cap}"
        payload = dict(**geom_payload(gname), root=np.int64(root),
                       d_spec=np.float64(np.nan if d is None else d), n_levels=np.int64(levels),
                       bins_refine=np.int64(-1 if b_ref is None else b_ref), bins_per_axis=np.int64(b_link),
                       d_link_arg=np.float64(np.nan if d_link is None else d_link), capacity=np.int64(cap),
                       **forest_payload(f))
        try:
            links = ow.build_cell_face_links(f, g, bins, grid, d_link=d_link, capacity=cap)
            payload.update(d_link=np.float64(links.d_link), block_ids=links.block_ids,
                           cell_indices=links.cell_indices, offsets=links.offsets, face_ids=links.face_ids,
                           error=np.array(""))
            msg = f"{links.n_linked_cells} cells / {links.face_ids.size} links"
        except ow.CapacityError as e:
            payload.update(error=np.array(str(e)))
            msg = f"CapacityError: {e}"
        save(tag, **payload)
        print(f"{tag}: {msg}")


GROUPS = {
    "bins": gen_bins,
    "predicate": gen_predicate,
    "marks": gen_marks,
    "pipelines": gen_pipelines,
    "forest": gen_forest_units,
    "links": gen_links,
    "bigpipes": gen_bigpipes,
    "vtk": gen_vtk,
}


def main(argv):
    which = argv or list(GROUPS)
    manifest_path = os.path.join(HERE, "MANIFEST.json")
    for w in which:
        GROUPS[w]()
    files = sorted(p for p in os.listdir(HERE) if p.endswith(".npz"))
    with open(manifest_path, "w") as f:
        json.dump({"numpy": np.__version__, "python": sys.version.split()[0],
                   "reference": "/root/reference/pkg (octowall 0.1.0)", "files": files}, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
