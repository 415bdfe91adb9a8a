"""Device-sized fused passes (ow_pipeline.cu: g2g_device): after a plan's
first pass has sized its output buffers, ``GridPlan.run`` enqueues the whole
geometry-to-grid pass without a host round trip and reads every count back
once at the end.  Each pass must equal the synchronous path array for array;
a pass whose capacities or assumptions do not hold (more bin entries than the
estimate, slow bin faces, a near-wall reach the domain does not predict,
larger outputs) falls back to the synchronous pass and is still exact."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ow():
    import paper_2502_16310_b200 as m
    from paper_2502_16310_b200 import _build

    _build.build()
    return m


def _records(tris):
    import torch

    from paper_2502_16310_b200 import shapes

    data = shapes.binary_stl_bytes(tris)
    return torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda(), int.from_bytes(data[80:84], "little")


def _snapshot(gp):
    out = dict(coords=gp.forest._coords.copy(), first_child=gp.forest._first_child.copy(),
               parent=gp.forest._parent.copy(), level=gp.forest._level.copy(),
               marks=gp.forest.marks.cpu().numpy().copy(), detected=list(gp.result.marked_detected),
               refined=list(gp.result.marked_refined), tests=list(gp.result.cell_face_tests),
               evaluated=list(gp.result.pairs_evaluated), entries=gp.result.bins.ids.numel(),
               ids=gp.result.bins.ids.cpu().numpy().copy(), counts=gp.result.bins.counts.cpu().numpy().copy())
    if gp.links is not None:
        for name in ("leaves", "flags", "cells", "q"):
            out[name] = getattr(gp.links, name).cpu().numpy().copy()
    return out


def _equal(a, b, tag):
    assert a.keys() == b.keys()
    for k in a:
        if isinstance(a[k], np.ndarray):
            np.testing.assert_array_equal(a[k], b[k], err_msg=f"{tag}: {k}")
        else:
            assert a[k] == b[k], (tag, k, a[k], b[k])


def _run_both(ow, dom, root, params, lattice, inputs, stage_times=False):
    """The same pass sequence through a device-sized plan and a synchronous one."""
    import torch

    from paper_2502_16310_b200 import _lib, pipeline

    snaps, modes = [], []
    for dev in (True, False):
        _lib.set_device_pass(dev)
        try:
            plan = pipeline.GridPlan(dom, root, params, lattice, reuse_outputs=True, stage_times=stage_times)
            run = []
            for inp in inputs:
                gp = plan.run(*inp) if isinstance(inp, tuple) else plan.run(geometry=inp)
                torch.cuda.synchronize()
                run.append(_snapshot(gp))
                if dev:
                    modes.append(gp.device_sized)
            snaps.append(run)
        finally:
            _lib.set_device_pass(True)
    for k, (a, b) in enumerate(zip(*snaps)):
        _equal(a, b, f"pass {k}")
    return modes


def test_device_pass_matches_sync_3d(ow):
    from paper_2502_16310_b200 import _lib, shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8)
    a = _records(shapes.icosphere_triangles(3))
    b = _records(shapes.icosphere_triangles(3, radius=0.25))
    c = _records(shapes.icosphere_triangles(4, radius=0.32))  # more entries / rows than the estimates
    n0 = _lib.device_pass_stats()
    modes = _run_both(ow, dom, (8, 8, 8), params, "D3Q19", [a, a, a, a, b, a, c, c, a])
    assert modes[0] == 0  # the first pass sizes the outputs
    assert modes[1:4] == [1, 1, 1]  # device-sized: eager, graph capture, graph replay
    assert modes[-1] == 1
    assert 2 in modes[6:8]  # the larger geometry outgrew an estimate once: synchronous re-run
    n1 = _lib.device_pass_stats()
    assert n1[0] - n0[0] >= 5


def test_device_pass_matches_sync_stage_events_and_d3q27(ow):
    """Stage-timing events on (the level loop runs eagerly, no graph) and a
    27-direction lattice with 4 levels."""
    from paper_2502_16310_b200 import shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.05, n_levels=4, bins_per_axis=8)
    a = _records(shapes.bumpy_sphere_triangles(40, 41))
    modes = _run_both(ow, dom, (8, 8, 8), params, "D3Q27", [a, a, a], stage_times=True)
    assert modes == [0, 1, 1]


def test_device_pass_matches_sync_2d(ow):
    dom = ow.Aabb(np.zeros(2), np.ones(2))
    params = ow.NearWallParams(d_spec=0.1, n_levels=3, bins_per_axis=8)
    g1 = ow.index_to_coords(ow.generate_circle((0.5, 0.5), 0.25, 256))
    g2 = ow.index_to_coords(ow.generate_circle((0.45, 0.5), 0.3, 700))
    modes = _run_both(ow, dom, (8, 8), params, "D2Q9", [g1, g1, g1, g2, g2, g1])
    assert modes[1:3] == [1, 1]


def test_device_pass_falls_back_on_slow_faces(ow):
    """Faces spanning more bins than the bitmask path handles need the slow
    path's readback: the device-sized attempt falls back, exactly."""
    import torch

    # a closed octahedron of 8 large faces: each spans many of the 16^3 bins
    c, r = 0.5, 0.3
    v = np.array([[c + r, c, c], [c - r, c, c], [c, c + r, c], [c, c - r, c], [c, c, c + r], [c, c, c - r]])
    faces = [(0, 2, 4), (2, 1, 4), (1, 3, 4), (3, 0, 4), (2, 0, 5), (1, 2, 5), (3, 1, 5), (0, 3, 5)]
    tris = np.array([[v[i] for i in f] for f in faces], np.float64)
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.05, n_levels=3, bins_per_axis=16, overlap_factor=1000)
    a = _records(tris)
    modes = _run_both(ow, dom, (8, 8, 8), params, "D3Q19", [a, a, a])
    assert modes[1:] == [2, 2]
    torch.cuda.synchronize()


def test_device_pass_falls_back_on_reach(ow):
    """A vertex slightly beyond the domain's largest |bound| (inside the
    reference's 1e-6 tolerance) changes the near-wall reach the pass predicts
    from the domain: fall back, exactly."""
    from paper_2502_16310_b200 import shapes

    tris = shapes.icosphere_triangles(2)
    tris = np.concatenate([tris, np.array([[[0.999, 0.5, 0.5], [1.0 + 4e-7, 0.5, 0.5], [0.999, 0.51, 0.5]]])])
    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8)
    a = _records(tris)
    modes = _run_both(ow, dom, (8, 8, 8), params, "D3Q19", [a, a])
    assert modes[1] == 2


def test_device_pass_errors_match_sync(ow):
    """Invalid geometry through a device-sized plan raises the synchronous
    path's error (message and type)."""
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8)
    plan = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19", reuse_outputs=True, stage_times=False)
    tris = shapes.icosphere_triangles(3)
    rec, n = _records(tris)
    plan.run(rec, n)
    plan.run(rec, n)
    bad = tris.copy()
    bad[7, 1] = bad[7, 0]  # degenerate triangle 7
    rb, nb = _records(bad)
    with pytest.raises(ow.InvalidParameterError, match="degenerate"):
        plan.run(rb, nb)
    out = tris.copy() + 0.6  # outside the domain
    ro, no = _records(out)
    with pytest.raises(ow.InvalidParameterError, match="outside"):
        plan.run(ro, no)
    gp = plan.run(rec, n)  # and the plan recovers
    torch.cuda.synchronize()
    assert gp.device_sized == 1


def test_run_async_two_plans_stream(ow):
    """run_async: two plans alternate over a stream of geometries with the
    next pass submitted before the previous one is finished (the e2e bench's
    pipeline); every pass's device arrays and host copies equal a fresh
    synchronous pass's, including a pass that outgrows its plan's estimates
    (finished on the synchronous path after the next pass was submitted)."""
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8)
    geoms = [shapes.icosphere_triangles(s, radius=r) for s, r in
             ((3, 0.3), (3, 0.3), (3, 0.25), (3, 0.3), (3, 0.3), (4, 0.32), (3, 0.3), (4, 0.32), (3, 0.3))]
    recs = [_records(t) for t in geoms]
    refs = []
    for rec, n in recs:
        r = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19").run(rec, n, host=True)
        torch.cuda.synchronize()
        refs.append((_snapshot(r), {k: (v.clone() if isinstance(v, torch.Tensor) else [c.clone() for c in v])
                                    for k, v in r.host.items()}))
    plans = [pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19", reuse_outputs=True, stage_times=False)
             for _ in range(2)]
    prev, modes = None, []
    for k, (rec, n) in enumerate(recs):
        pend = plans[k % 2].run_async(rec, n, host=True, defer=True)
        if prev is not None:
            j, p = prev
            g = p.result()
            g.wait()
            modes.append(g.device_sized)
            _equal(_snapshot(g), refs[j][0], f"pass {j}")
            for key in ("level", "parent", "first_child", "marks", "cells", "flags", "q_packed"):
                assert torch.equal(g.host[key], refs[j][1][key]), (j, key)
        prev = (k, pend)
    j, p = prev
    g = p.result()
    g.wait()
    _equal(_snapshot(g), refs[j][0], f"pass {j}")
    assert 1 in modes and 2 in modes


def test_run_async_same_plan_and_in_flight_limit(ow):
    """A plan's pending pass is finished before its next submit (results of
    both equal synchronous passes); at most 8 passes may be in flight on one
    context — a 9th submit raises, and the pending ones still finish exactly."""
    import torch

    from paper_2502_16310_b200 import pipeline, shapes

    dom = ow.Aabb(np.zeros(3), np.ones(3))
    params = ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8)
    rec, n = _records(shapes.icosphere_triangles(3))
    ref = _snapshot(pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19").run(rec, n))
    plan = pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19", reuse_outputs=True, stage_times=False)
    plan.run(rec, n)
    p1 = plan.run_async(rec, n)
    p2 = plan.run_async(rec, n)  # finishes p1 first
    g1 = p1.result()
    assert g1.device_sized == 1
    g2 = p2.result()
    torch.cuda.synchronize()
    _equal(_snapshot(g2), ref, "same plan")
    plans = [pipeline.GridPlan(dom, (8, 8, 8), params, "D3Q19", reuse_outputs=True, stage_times=False)
             for _ in range(9)]
    for p in plans:
        p.run(rec, n)  # (sizes every plan's outputs)
    pend = [p.run_async(rec, n) for p in plans[:8]]
    with pytest.raises(ow.InvalidParameterError, match="in flight"):
        plans[8].run_async(rec, n)
    for q in pend:
        g = q.result()
        assert g.device_sized == 1
    torch.cuda.synchronize()
    _equal(_snapshot(g), ref, "after the in-flight limit")
    g9 = plans[8].run(rec, n)
    torch.cuda.synchronize()
    _equal(_snapshot(g9), ref, "the refused plan afterwards")
