#!/usr/bin/env python
"""Geometry-to-grid benchmark (BASELINE.json metric) on B200.

One step = the whole hot path on one geometry: binary-STL records -> SoA
import -> face binning -> per level {near-wall marking, propagation,
refinement / block allocation} -> lattice boundary links + q on the finest
level.  ``value`` is cell-face tests / s (T of SURVEY.md §8d over the step's
marking passes divided by the step's device time) with the STL records
resident in HBM; ``e2e`` repeats the step from pinned host bytes with the
H2D copy and the D2H of the results (forest arrays, link flags, q) inside the
timed region.  ``ms_per_step`` is the geometry-to-grid time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (strong scaling, NCCL)
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    "C1": dict(workload="C1 circle text primitive 12800 edges, 64^2 root, d=0.1, 3 levels, B=8, D2Q9",
               kind="text", text="circle 0.5 0.5 0.25 12800\n", dim=2, root=64, d=0.1, levels=3, B=8,
               lattice="D2Q9"),
    "C2": dict(workload="C2 icosphere 20480 triangles (binary STL), 16^3 root, d=0.05, 3 levels, B=8, D3Q19",
               kind="ico", subdiv=5, dim=3, root=16, d=0.05, levels=3, B=8, lattice="D3Q19"),
    "C3": dict(workload="C3 bumpy lat-lon sphere 69936 triangles (binary STL), 16^3 root, d=0.05, 4 levels, "
                        "B=8, D3Q27", kind="bumpy", dim=3, root=16, d=0.05, levels=4, B=8, lattice="D3Q27"),
    "C4": dict(workload="C4 torus knot 1M triangles (binary STL), 16^3 root, d=0.02, 5 levels, B=32, D3Q19",
               kind="knot", dim=3, root=16, d=0.02, levels=5, B=32, lattice="D3Q19"),
    "C5": dict(workload="C5 icosphere 5.24M triangles (binary STL), 64^3 root, d=0.01, 3 levels, B=64, D3Q19",
               kind="ico", subdiv=9, dim=3, root=64, d=0.01, levels=3, B=64, lattice="D3Q19"),
}

FP32_OPS_PER_TEST = {3: 130, 2: 21}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def make_input(cfg):
    from paper_2502_16310_b200 import shapes

    if cfg["kind"] == "text":
        return cfg["text"].encode()
    if cfg["kind"] == "ico":
        tris = shapes.icosphere_triangles(cfg["subdiv"])
    elif cfg["kind"] == "bumpy":
        tris = shapes.bumpy_sphere_triangles()
    else:
        tris = shapes.torus_knot_triangles()
    return shapes.binary_stl_bytes(tris)


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled by an ``nvidia-smi -lms`` child
    process during the timed region (a separate process: no GIL contention
    with the host side of the pipeline being timed)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index, period_ms=20):
        self.index, self.period_ms = index, period_ms
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.proc = None

    def __enter__(self):
        import subprocess
        import tempfile

        self.out = tempfile.TemporaryFile(mode="w+")
        try:
            dev = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[self.index] \
                if os.environ.get("CUDA_VISIBLE_DEVICES") else str(self.index)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", dev, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 f"-lms={self.period_ms}"], stdout=self.out, stderr=subprocess.DEVNULL)
            time.sleep(0.3)  # let the sampler start before the timed region
        except Exception as e:  # pragma: no cover
            log("clock sampling unavailable:", e)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            self.proc.wait()
            self.out.seek(0)
            for line in self.out.read().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) != 6:
                    continue
                try:
                    self.samples.append(float(parts[0]))
                    self.max_mhz = float(parts[1])
                except ValueError:
                    continue
                for name, v in zip(self.NAMES, parts[2:]):
                    if v.lower().startswith("active"):
                        self.reasons.add(name)

    def summary(self):
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples),
                "sampler": f"nvidia-smi -lms {self.period_ms} (child process) over the timed region"}


# ---------------------------------------------------------------------------- GPU arm
def e2e_stream(plan, rec_host, n_faces, args, l2_flush, barrier):
    """End-to-end steps through the public API with pinned host bytes in and
    the results out, as a stream of geometries: two plans alternate so the
    transfers of one step overlap the device work of its neighbours.  Returns
    (total ms of the timed steps minus the L2 flushes, per-pass ms, H2D bytes
    per step, D2H bytes per step, slow-path steps)."""
    import torch

    from paper_2502_16310_b200 import pipeline

    plans = [plan, pipeline.GridPlan(plan.domain, plan.root_dims, plan.params, plan.lattice, reuse_outputs=True,
                                     comm=plan.comm, stage_times=plan.stage_times)]
    dev = torch.device("cuda", torch.cuda.current_device())
    cs = torch.cuda.current_stream()
    hs = torch.cuda.Stream()
    bufs = [torch.empty_like(rec_host, device=dev) for _ in range(2)]
    loaded = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    for e in consumed:
        e.record(cs)
    # (each of the two plans needs 3 passes before its pass is a replayed graph:
    # sizing, the first device-sized pass, the capture — at least 6 stream steps)
    W, K = max(args.warmup, 6), args.steps

    def h2d(k):
        with torch.cuda.stream(hs):
            hs.wait_event(consumed[k % 2])  # the pass that read this buffer has finished
            bufs[k % 2].copy_(rec_host, non_blocking=True)
            loaded[k % 2].record(hs)

    flushes = []
    passes = []
    slow, h2d_b, d2h_b = [], 0, 0
    prev = None  # (step, PendingGridPass) submitted, not yet finished by the host
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def finish(k, pend):
        # the host finishes step k (its counts, errors, host copies) while
        # step k+1 already runs on the device, then waits for step k-1's
        # results to reach host memory (their copies overlapped step k)
        nonlocal h2d_b, d2h_b
        gp = pend.result()
        if k >= 0:
            h2d_b = rec_host.numel()
            hres = gp.host
            d2h_b = sum(t.numel() * t.element_size() for k2, t in hres.items() if k2 != "coords")
            d2h_b += sum(t.numel() * t.element_size() for t in hres["coords"])
            if gp.reran or gp.host_copied & 5 != 5 or gp.done is None:
                slow.append(k)
        return gp

    sync_steps = os.environ.get("OW_E2E_SYNC") == "1"
    barrier()
    h2d(-W)
    done_prev = None
    for k in range(-W, K):
        if k == 0:
            if prev is not None:
                finish(*prev).wait()  # warm-up results out of the way: the timed stream starts empty
                prev = None
            if done_prev is not None:
                done_prev.wait()
                done_prev = None
            torch.cuda.synchronize()
            start.record(cs)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(cs)
        l2_flush()
        f1.record(cs)
        if k + 1 < K:  # step k+1's bytes start while step k computes
            h2d(k + 1)
        cs.wait_event(loaded[k % 2])
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(cs)
        pend = plans[k % 2].run_async(bufs[k % 2], n_faces, host=True, defer=True)
        if sync_steps:  # (A/B: the host finishes each step before submitting the next)
            pend.result()
        p1.record(cs)
        consumed[k % 2].record(cs)
        if k >= 0:
            flushes.append((f0, f1))
            passes.append((p0, p1))
        if prev is not None:
            gp = finish(*prev)  # step k-1, while step k runs
            if done_prev is not None:
                done_prev.wait()  # the host has step k-2's results
            done_prev = gp
        prev = (k, pend)
    if prev is not None:
        gp = finish(*prev)
        if done_prev is not None:
            done_prev.wait()
        done_prev = gp
    if done_prev is not None and done_prev.done is not None:
        cs.wait_event(done_prev.done)
    end.record(cs)
    torch.cuda.synchronize()
    total = start.elapsed_time(end) - sum(a.elapsed_time(b) for a, b in flushes)
    return total, [a.elapsed_time(b) for a, b in passes], h2d_b, d2h_b, slow


def gpu_arm(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2502_16310_b200 as ow
    from paper_2502_16310_b200 import _lib, parallel

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    numa = _lib.bind_host_numa(local_rank)  # pinned staging buffers on the GPU's socket (no-op on one node)
    data = make_input(cfg)
    dim = cfg["dim"]
    dom = ow.Aabb(np.zeros(dim), np.ones(dim))
    params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
    grid = ow.BinGrid(dom, cfg["B"])
    text = cfg["kind"] == "text"
    if text:  # C1: the text primitive's geometry stays resident for `value`; e2e re-parses it every step
        ig = ow.geometry.parse_text_primitives(data.decode())
        n_faces = ig.n_faces
        geom_dev = ow.index_to_coords(ig)
    else:
        n_faces = int.from_bytes(data[80:84], "little")
        rec_host = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).pin_memory()
        rec_dev = rec_host.to(dev)

    from paper_2502_16310_b200 import pipeline

    # N > 1: the fused pass shards on the device (parallel.DeviceComm: marks,
    # statistics, lattice flag words and q rows exchanged over peer memory by
    # the native level loop, no host round trip per level)
    comm = None
    if world > 1:
        cap_blocks = 32 * cfg["root"] ** dim
        comm = parallel.DeviceComm(max(64 << 20, 4 * (4 ** dim) * cap_blocks))
    # (stage-timing events off in the timed loops: an event between two kernels
    # stops their programmatic overlap; the profiled pass below records them)
    plan = pipeline.GridPlan(dom, (cfg["root"],) * dim, params, cfg["lattice"], reuse_outputs=True, comm=comm,
                             stage_times=False)

    def submit(records):
        # fused native pass: STL records (C1: the resident text-primitive
        # geometry) -> grid -> lattice links (ow_geometry_to_grid_submit)
        return plan.run_async(geometry=geom_dev) if text else plan.run_async(records, n_faces)

    def done(pend):
        gp = pend.result()  # (the host's checks and results: ow_geometry_to_grid_finish)
        return gp.result, gp.forest, gp.links

    def step(records):
        return done(submit(records))

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def l2_flush():
        flush.zero_()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # >= 3 untimed steps: the first sizes every buffer, the second is the first
    # device-sized pass, the third captures its CUDA graph (replayed when timed)
    for _ in range(max(args.warmup, 3)):
        res, forest, ll = step(rec_dev if not text else None)
    T_step = int(sum(res.cell_face_tests))
    evaluated = int(sum(res.pairs_evaluated))
    blocks = forest.blocks_per_level()
    n_boundary = ll.n_boundary

    # ---- value: inputs resident in HBM
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    fallback_steps = []
    gc.collect()
    gc.disable()  # no collector pauses inside the timed regions (re-enabled after e2e)
    launches0 = _lib.launches()
    with ClockSampler(local_rank) as clk:
        barrier()
        for k in range(args.steps):
            l2_flush()
            ev[k][0].record()
            pend = submit(rec_dev if not text else None)
            ev[k][1].record()  # after the submitted pass's last kernel
            res, forest, ll = done(pend)
            ev[k][2].record()  # (a pass that fell back to the synchronous path is timed to here)
            if pend.result().device_sized == 2:
                fallback_steps.append(k)
        barrier()
    launches = _lib.launches() - launches0
    lat_stats = _lib.lattice_stats()
    ms = sum(e0.elapsed_time(e2 if k in fallback_steps else e1) for k, (e0, e1, e2) in enumerate(ev))
    # per-kernel-family device times (roofline): the same steps again with the
    # library's CUDA-event brackets on, outside the timed loop above
    _lib.profile(True)
    if plan is not None:
        plan.stage_times = True
    barrier()
    for k in range(args.steps):
        l2_flush()
        pres, _, _ = step(rec_dev if not text else None)
    barrier()
    if plan is not None:
        plan.stage_times = False
    for s in pres.timings:
        log("stage", s.csv_row())
    prof = _lib.profile_read()
    _lib.profile(False)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps

    # ---- e2e: pinned host bytes in, results out
    e2e = None
    if not args.no_e2e:
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        h2d = d2h = 0
        pinned = []
        slow_path = []  # steps that reran the level loop or copied results from Python
        barrier()
        # C1: the text primitive parsed on the host every step (the reference's
        # import_text_primitives + index_to_coords: the vertices and faces go
        # host -> device), the fused pass, every result back to pinned memory.
        # Two plans alternate: step k is parsed and submitted while step k-1
        # runs, then the host finishes step k-1 (k < 0: untimed warm-up).
        if text:
            tplans = [plan, pipeline.GridPlan(dom, (cfg["root"],) * dim, params, cfg["lattice"], reuse_outputs=True,
                                              stage_times=False)]
            W2 = max(args.warmup, 6)  # (3 untimed passes per plan: sizing, first device-sized pass, capture)
            tprev, tdone = None, None
            tstart, tend = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tflush = []

            def tfinish(pend):
                nonlocal d2h, res, forest, ll
                gp = pend.result()
                res, forest, ll = gp.result, gp.forest, gp.links
                hres = gp.host
                d2h = sum(t.numel() * t.element_size() for k2, t in hres.items() if k2 != "coords")
                d2h += sum(t.numel() * t.element_size() for t in hres["coords"])
                return gp

            for k in range(-W2, args.steps):
                if k == 0:
                    if tprev is not None:
                        tfinish(tprev).wait()
                        tprev = None
                    if tdone is not None:
                        tdone.wait()
                        tdone = None
                    torch.cuda.synchronize()
                    tstart.record()
                f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                f0.record()
                l2_flush()
                f1.record()
                if k >= 0:
                    tflush.append((f0, f1))
                igk = ow.geometry.parse_text_primitives(data.decode())
                h2d = igk.vertices.nbytes + igk.faces.nbytes
                pend = tplans[k % 2].run_async(geometry=ow.index_to_coords(igk), host=True, defer=True)
                if tprev is not None:
                    gp = tfinish(tprev)
                    if tdone is not None:
                        tdone.wait()
                    tdone = gp
                tprev = pend
            gp = tfinish(tprev)
            if tdone is not None:
                tdone.wait()
            if gp.done is not None:
                torch.cuda.current_stream().wait_event(gp.done)
            tend.record()
            torch.cuda.synchronize()
            ms2_total = tstart.elapsed_time(tend) - sum(a.elapsed_time(b) for a, b in tflush)
            per = [ms2_total / args.steps] * args.steps  # (a stream: no per-step split)
            ev2 = None
        if not text:
            ms2_total, per, h2d, d2h, slow_path = e2e_stream(plan, rec_host, n_faces, args, l2_flush, barrier)
            ev2 = None
        barrier()
        ms2 = sum(a.elapsed_time(b) for a, b in ev2) if ev2 else ms2_total
        t2 = torch.tensor([ms2], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        ms2 = float(t2.item()) / args.steps
        if ev2:
            per = [a.elapsed_time(b) for a, b in ev2]
        log("e2e steps ms", " ".join(f"{x:.3f}" for x in per))
        per = sorted(per)
        e2e = {"value": T_step / (ms2 / 1e3), "unit": "cell-face tests/s", "ms_per_step": ms2,
               "ms_step_median": per[len(per) // 2], "ms_step_max": per[-1],
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "result": ("forest arrays (level, coords, parent, first_child, marks) + boundary rows packed: cell "
                          "ids, flag words and the q of the set bits (GridPass.host_q() expands to the dense rows)")}
        if text:
            e2e["pipeline"] = ("two GridPlans alternate: step k's text primitive is parsed on the host and its "
                               "vertices / faces go host->device (index_to_coords, pinned staging, no host wait) "
                               "while step k-1 runs; step k is submitted (run_async(host=True, defer=True)) before "
                               "the host finishes step k-1; ms_per_step = (device time of the stream - the L2 "
                               "flushes) / steps")
        if not text:
            e2e["slow_path_steps"] = slow_path
            e2e["pipeline"] = ("two GridPlans alternate: step k+1's STL bytes go host->device on a copy stream while "
                               "step k computes; step k+1 is submitted (GridPlan.run_async(host=True, defer=True)) "
                               "before the host finishes step k (PendingGridPass.result(): its counts, checks and "
                               "device->host copies on the library's copy stream, which overlap step k+1), and the "
                               "host waits for step k-1's results (GridPass.wait()) after that; "
                               "ms_per_step = (device time from the first H2D to the last D2H - the L2 flushes "
                               "between passes) / steps; ms_step_* = per-pass compute-stream times; the stream "
                               "runs max(warmup, 6) untimed steps first (3 per plan: sizing, first device-sized "
                               "pass, graph capture)")

    gc.enable()

    # ---- roofline of the dominant kernel family
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    sm_mhz = clk.summary()["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * 128 * sm_mhz * 1e6 / 1e12  # non-FMA issue rate (-fmad=false), TOP/s
    traffic = {}
    try:
        traffic = json.load(open(os.path.join(REPO, "profiles", "traffic.json"))).get(args.config, {})
    except Exception:
        pass
    peak_note = ("148 SMs x 128 FP32 lanes x max SM clock = non-FMA (FMUL/FADD/FSETP) issue rate; "
                 "MEASURED_PEAKS.json has no FP32 entry")

    def entry(kernel, ms, n, ops, algorithmic, tkey):
        achieved = ops / (ms / 1e3) / 1e12 if ms > 0 else 0.0
        t = traffic.get(tkey)
        return {"kernel": kernel, "bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": achieved / fp32_peak if fp32_peak else None, "traffic": t, "traffic_unit": "bytes/launch",
                "algorithmic": algorithmic, "launches": n, "avg_launch_ms": ms / max(n, 1), "peak_note": peak_note}

    mark_ms, mark_n = prof["mark"]
    spheres = int(sum(res.sphere_tests))
    sphere_ops = 8 if dim == 3 else 5  # (dx, dy[, dz]) sub, squares, sums
    mark = entry("k_mark_blocks + k_mark_items (near-wall marking)", mark_ms, mark_n,
                 (FP32_OPS_PER_TEST[dim] * evaluated + sphere_ops * spheres) * args.steps,
                 f"per step: {spheres} cell-face bounding-sphere tests x {sphere_ops} FP32 ops + {evaluated} "
                 f"full predicates x {FP32_OPS_PER_TEST[dim]} FP32 ops (the reference's _scan_block cascade on the "
                 f"pairs surviving its FP64 box cull; {int(sum(res.box_culls))} FP64 box culls not counted)", "mark")
    sw_ms, sw_n = prof["lattice_sweep"]
    n_cb, n_pairs, mt = lat_stats
    # FP32 arithmetic of one watertight link-face test (oracle/lattice.py:wt_hits):
    # 3D: per vertex 3 translations, 2 shear products, 2 shear differences (21),
    # edge functions 6 + 3, det 2, T 3 + 3 + 2 = 40 (the division t = T / det
    # only for candidate crossings, not counted); 2D (wt_hits2): 14
    per_test = 40 if dim == 3 else 14
    lattice = entry("k_lat_faces (boundary-link intersection sweep)", sw_ms, sw_n, per_test * mt * args.steps,
                    f"per step: {mt} watertight link-face tests x {per_test} FP32 ops ({n_pairs} (block, face, "
                    f"direction) rows over {n_cb} candidate blocks; every test is a link whose AABB meets the face "
                    f"AABB)", "lattice")
    dominant = lattice if sw_ms >= mark_ms else mark
    roofline = dict(dominant)
    roofline["secondary"] = mark if dominant is lattice else lattice
    # HBM roofline of the binning family: per fill_bins call the
    # algorithmic bytes are the coordinates read (4 D^2 F), the face ids
    # written (4 E) and counts + offsets (8 B^D); the family's device time is
    # the sample walk, the pair emission, the stable radix sort and the scans
    # (events around the device work only, not the host readback between them)
    bins_ms, bins_n = prof["fill_bins"]
    n_bins = cfg["B"] ** dim
    E = int(res.bins.ids.numel()) if res.bins is not None else 0
    calls = max(1, bins_n // 2)  # (count, emit) brackets per call
    bin_bytes = (4 * dim * dim * n_faces + 4 * E + 8 * n_bins) * calls
    hbm_peak = float(peaks.get("hbm_gbs") or 6542.7)
    achieved_gbs = bin_bytes / (bins_ms / 1e3) / 1e9 if bins_ms > 0 else 0.0
    roofline["hbm"] = {
        "kernel": "fill_bins family (k_count_fast, k_count_walk, k_emit_fast, k_radix_hist/k_radix_scatter, k_scan)",
        "bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
        "frac": achieved_gbs / hbm_peak, "traffic": traffic.get("fill_bins"), "traffic_unit": "bytes/call",
        "algorithmic": f"per call: 4*D^2*F coords read + 4*E ids + 8*B^D counts/offsets = {4 * dim * dim * n_faces} + "
                       f"{4 * E} + {8 * n_bins} B (F={n_faces}, E={E}, B^D={n_bins}); {calls // args.steps} call(s) "
                       f"per step",
        "launches": bins_n, "avg_call_ms": bins_ms / calls,
        "peak_note": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read + write bytes)"}
    roofline["families_ms"] = {k: round(v[0] / args.steps, 4) for k, v in prof.items()}
    out = {
        "metric": "geometry-to-grid time (ms) & cell-face tests/s at 1/2/4/8 B200 vs CPU",
        "value": T_step / (ms_step / 1e3),
        "unit": "cell-face tests/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "geometry_to_grid_ms": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (procedural geometry, deterministic)",
        # (main() sets "config" to bench_config(): the same object as the reference arm's)
        "run": {"cell_face_tests_per_step": T_step, "pairs_evaluated_per_step": evaluated,
                "value_timing": ("per pass: CUDA events before the submit and after its last kernel "
                                 "(GridPlan.run_async); the host's finish step runs after; a pass that fell "
                                 "back to the synchronous path is timed through its finish"),
                "fallback_steps": fallback_steps,
                "blocks_per_level": blocks, "boundary_cells": n_boundary,
                "parallelism": (f"octree-block shards x{world}: work-balanced marking slices and finest-leaf "
                                f"lattice slices per rank, marks / statistics / flag words / q rows exchanged "
                                f"over CUDA-IPC peer memory inside the native level loop; bins and forest "
                                f"replicated" if world > 1 else "single GPU")},
        "roofline": roofline,
        "gpu_launches": int(launches),
        "host_numa_node": numa,
        "clocks": clk.summary(),
    }
    if e2e:
        out["e2e"] = e2e
    return out


# ---------------------------------------------------------------------------- CPU arms
# T and faces of each configuration: properties of the
# workload, identical for both arms (tests/test_gpu_parity.py checks the GPU
# pass against this table; the oracle / reference reproduce the same forests)
FACES = {"C1": 12800, "C2": 20480, "C3": 69936, "C4": 1000000, "C5": 5242880}
TESTS_PER_STEP = {"C1": 65607680, "C2": 114183168, "C3": 2883791872, "C4": 5029797240, "C5": 3326663808}
FULL_CPU = ("C1", "C2")  # configs whose whole pass one CPU step runs (C3-C5: bounded samples)


def bench_config(name):
    """The ``config`` object of both arms' JSON lines (identical dicts)."""
    cfg = CONFIGS[name]
    return {"workload": cfg["workload"], "faces": FACES[name], "cell_face_tests_per_step": TESTS_PER_STEP[name],
            "step": "geometry-to-grid pass: STL (C1: text primitive) import -> refine_near_wall over all levels "
                    "(fill_bins, near-wall marking, propagation, refinement); the GPU arm also builds the "
                    "finest-level lattice links + q, which the reference does not have",
            "l2": "GPU arm: L2 flushed (256 MB write) before every step; CPU arm: host caches as they are"}


def _ref_module():
    from oracle import stage_ref

    return stage_ref.import_reference() if stage_ref.available() else None


def _write_input(name):
    import tempfile

    cfg = CONFIGS[name]
    fd, path = tempfile.mkstemp(suffix=".txt" if cfg["kind"] == "text" else ".stl")
    with os.fdopen(fd, "wb") as fh:
        fh.write(make_input(cfg))
    return path


def _ref_full_step(name, path):
    """One whole geometry-to-grid pass of the reference's own serial path
    (cli.py:87-101: load_geometry -> init_root_grid -> refine_near_wall,
    backend "serial") from the staged oracle/_ref, else the NumPy port.
    Returns (seconds, cell-face tests, kind)."""
    cfg = CONFIGS[name]
    dim = cfg["dim"]
    ow = _ref_module()
    t0 = time.perf_counter()
    if ow is not None:
        if cfg["kind"] == "text":
            geom = ow.index_to_coords(ow.import_text_primitives(path, dim=dim))
        else:
            geom = ow.import_stl(path)
        forest = ow.init_root_grid(ow.Aabb(np.zeros(dim), np.ones(dim)), (cfg["root"],) * dim)
        ow.refine_near_wall(forest, geom, ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"],
                                                           bins_per_axis=cfg["B"]))
        return time.perf_counter() - t0, TESTS_PER_STEP[name], "reference"
    from oracle import forest as of
    from oracle import geometry as og
    from oracle import nearwall as on

    with open(path, "rb") as fh:
        data = fh.read()
    coords = og.index_to_coords(*og.parse_primitives(data.decode())) if cfg["kind"] == "text" else og.stl(data)
    f = of.Forest(np.zeros(dim), np.ones(dim), (cfg["root"],) * dim)
    r = on.refine_near_wall(f, coords, cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
    return time.perf_counter() - t0, int(sum(r["cell_face_tests"])), "port"


CPU_SAMPLE_TESTS = 1.5e8  # ~25 s of the oracle's marking at ~6e6 tests/s


def _port_sample(name):
    """Bounded sample for configurations whose whole pass takes minutes to
    hours on one core (C3-C5; DNF at C4/C5): the level-0
    face-detection stage of the NumPy port over a uniform spread of level-0
    blocks (every k-th one, so the near-wall share is kept), import and
    fill_bins untimed.  Returns (seconds, tests, what)."""
    from oracle import binning as ob
    from oracle import forest as of
    from oracle import geometry as og
    from oracle import nearwall as on

    cfg = CONFIGS[name]
    dim = cfg["dim"]
    coords = og.stl(make_input(cfg))
    f = of.Forest(np.zeros(dim), np.ones(dim), (cfg["root"],) * dim)
    grid = ob.Grid(np.zeros(dim), np.ones(dim), cfg["B"])
    bins = ob.fill_bins(coords, grid)
    T = on.cell_face_tests(f, 0, grid, bins[1], coords.shape[2])
    leaves = f.leaves_at(0)
    stride = max(1, int(np.ceil(T / CPU_SAMPLE_TESTS)))
    sample = leaves[::stride]
    skip = np.ones(len(f.marks), bool)
    skip[sample] = False
    f.marks[skip] = of.MARKED  # mark() skips MARKED leaves: only the sample is evaluated
    T = int(np.asarray(bins[1], np.int64)[grid.bin_of(f.cell_centers(sample))].sum())
    t1 = time.perf_counter()
    on.mark(f, 0, coords, cfg["d"], bins, grid)
    return time.perf_counter() - t1, T, (f"NumPy port: level-0 binned marking (face-detection stage; import and "
                                         f"fill_bins untimed) of every {stride}th level-0 block "
                                         f"({len(sample)} of {len(leaves)})")


def _pool_step(args):
    name, path = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    if name in FULL_CPU:
        return _ref_full_step(name, path)
    s, T, what = _port_sample(name)
    return s, T, "port"


def cpu_baseline(name):
    """One bounded CPU step on one core (rank 0, N=1): the whole pass of the
    reference's serial path for C1/C2, a level-0 sample of the port beyond."""
    path = _write_input(name)
    try:
        if name in FULL_CPU:
            s, T, kind = _ref_full_step(name, path)
            what = (f"one whole {name} geometry-to-grid pass ({'reference octowall serial backend, staged in oracle/_ref' if kind == 'reference' else 'NumPy port of octowall'}: "
                    f"import -> refine_near_wall over {CONFIGS[name]['levels']} levels), {s:.1f} s")
        else:
            s, T, what = _port_sample(name)
            kind = "port"
    finally:
        os.unlink(path)
    return {"value": T / s, "unit": "cell-face tests/s", "cores": 1, "kind": kind, "sample": what}


def reference_arm(args, name):
    """--impl reference: the reference's CPU implementation of the path on the
    host cores.  Each step is one whole pass of the configuration (C1/C2; a
    bounded level-0 sample beyond) in its own single-threaded worker process
    (the serial backend is one core by construction); steps run concurrently
    on up to all host cores, and ``value`` is the whole job's tests / wall
    time of the K timed steps (W untimed warm-up steps first, also pooled)."""
    import multiprocessing as mp

    path = _write_input(name)
    cores = max(1, min(args.steps, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                       else os.cpu_count() or 1))
    try:
        ctx = mp.get_context("fork")
        with ctx.Pool(cores) as pool:
            if args.warmup:
                pool.map(_pool_step, [(name, path)] * min(args.warmup, cores))
            t0 = time.perf_counter()
            res = pool.map(_pool_step, [(name, path)] * args.steps, chunksize=1)
            wall = time.perf_counter() - t0
    finally:
        os.unlink(path)
    tests = sum(r[1] for r in res)
    kind = res[0][2]
    v = tests / wall
    what = (f"{args.steps} whole {name} passes (import -> refine_near_wall, all levels) of "
            f"{'the reference octowall serial backend (oracle/_ref)' if kind == 'reference' else 'the NumPy port'}"
            if name in FULL_CPU else f"{args.steps} level-0 samples of the NumPy port")
    cb = {"value": v, "unit": "cell-face tests/s", "cores": cores, "kind": kind,
          "sample": f"{what}, one single-threaded process per step, {cores} concurrent; "
                    f"{wall:.1f} s wall for the timed steps, {statistics.mean(r[0] for r in res):.2f} s per step"}
    return {
        "metric": "geometry-to-grid time (ms) & cell-face tests/s at 1/2/4/8 B200 vs CPU",
        "impl": "reference", "value": v, "unit": "cell-face tests/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(r[0] for r in res), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (procedural geometry, deterministic)",
        "config": bench_config(name), "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "cell-face tests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(reference_arm(args, args.config)), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist

        # one rank per GPU over NCCL; OW_BENCH_BACKEND=gloo with more ranks than
        # GPUs (ranks share devices) only exercises the N>1 code path on a small box
        backend = os.environ.get("OW_BENCH_BACKEND", "nccl")
        local_rank %= max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    from paper_2502_16310_b200 import _build

    if rank == 0:
        _build.build()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    out = gpu_arm(args, cfg, rank, world, local_rank)
    out["config"] = bench_config(args.config)
    if out["run"]["cell_face_tests_per_step"] != TESTS_PER_STEP[args.config]:
        log("WARNING: T of the GPU pass differs from the workload table")
        out["run"]["tests_mismatch"] = True
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
