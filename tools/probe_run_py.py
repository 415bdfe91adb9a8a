"""Where the Python time of GridPlan.run goes (GPU box helper): times the
pieces run() calls, outside the native call, by wrapping them.

    python tools/probe_run_py.py [C2] [steps]
"""

import os
import sys
import time
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402
from paper_2502_16310_b200 import _lib, geometry, lattice, nearwall, pipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = bench.CONFIGS[name]
data = bench.make_input(cfg)
n = int.from_bytes(data[80:84], "little")
rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
dom = ow.Aabb(np.zeros(3), np.ones(3))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
plan = pipeline.GridPlan(dom, (cfg["root"],) * 3, params, cfg["lattice"], reuse_outputs=True)
acc = defaultdict(float)


def wrap(mod, attr, label):
    f = getattr(mod, attr)

    def w(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        acc[label] += time.perf_counter() - t0
        return r

    setattr(mod, attr, w)


wrap(_lib, "call", "native call")
wrap(pipeline, "_driver_result", "_driver_result")
wrap(pipeline, "_driver_done", "_driver_done")
wrap(pipeline, "LatticeLinks", "LatticeLinks()")
wrap(pipeline.CoordListGeometry, "_validated", "_validated")
wrap(torch, "empty", "torch.empty")
wrap(pipeline.GridPass, "__init__", "GridPass()")
for _ in range(10):
    plan.run(rec, n)
torch.cuda.synchronize()
acc.clear()
t0 = time.perf_counter()
for _ in range(steps):
    plan.run(rec, n)
tot = time.perf_counter() - t0
torch.cuda.synchronize()
print(f"{name}: run {1e6 * tot / steps:.1f} us per call")
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"  {1e6 * v / steps:8.1f} us  {k}")
rest = tot - sum(acc.values())
print(f"  {1e6 * rest / steps:8.1f} us  (rest of run's own Python)")
