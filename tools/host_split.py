"""Host-side split of one GridPlan.run (GPU box helper): Python before the
native call, the native call (which ends at its last readback), Python after.

    python tools/host_split.py [C2] [steps] [host]

``host``: run(host=True) from pinned STL bytes (the bench's e2e step).
"""

import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402
from paper_2502_16310_b200 import _lib, pipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = bench.CONFIGS[name]
data = bench.make_input(cfg)
n = int.from_bytes(data[80:84], "little")
rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
dim = cfg["dim"]
dom = ow.Aabb(np.zeros(dim), np.ones(dim))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
plan = pipeline.GridPlan(dom, (cfg["root"],) * dim, params, cfg["lattice"], reuse_outputs=True)

marks = []
_orig = _lib.call


def timed_call(name, *a):
    t0 = time.perf_counter()
    r = _orig(name, *a)
    marks.append((name, t0, time.perf_counter()))
    return r


_lib.call = timed_call
HOST = len(sys.argv) > 3 and sys.argv[3] == "host"
rec_host = rec.cpu().pin_memory()
_run = plan.run


def run_step(r, nf):
    if HOST:
        _run(rec_host.to("cuda", non_blocking=True), nf, host=True)
        torch.cuda.current_stream().synchronize()
    else:
        _run(r, nf)


plan_run = run_step
for _ in range(5):
    plan_run(rec, n)
torch.cuda.synchronize()
tot = pre = nat = post = 0.0
for _ in range(steps):
    marks.clear()
    t0 = time.perf_counter()
    plan_run(rec, n)
    t1 = time.perf_counter()
    g = [m for m in marks if m[0] == "ow_geometry_to_grid"][0]
    tot += t1 - t0
    pre += g[1] - t0
    nat += g[2] - g[1]
    post += t1 - g[2]
    torch.cuda.synchronize()
print(f"{name}: run {1e6 * tot / steps:.1f} us = python before {1e6 * pre / steps:.1f} + native "
      f"{1e6 * nat / steps:.1f} + python after {1e6 * post / steps:.1f}")
pr = cProfile.Profile()
pr.enable()
for _ in range(steps):
    plan_run(rec, n)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
