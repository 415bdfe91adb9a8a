"""Host time of the e2e stream's pieces (no profiler): GridPlan.run split into
the native call and the Python around it, and the bench loop's own
bookkeeping (GPU box helper):  python tools/probe_e2e_host.py [C2]"""

import os
import sys
import time
import types
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402
from paper_2502_16310_b200 import _lib, pipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = bench.CONFIGS[name]
data = bench.make_input(cfg)
n = int.from_bytes(data[80:84], "little")
rec_host = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).pin_memory()
dim = cfg["dim"]
dom = ow.Aabb(np.zeros(dim), np.ones(dim))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
plan = pipeline.GridPlan(dom, (cfg["root"],) * dim, params, cfg["lattice"], reuse_outputs=True, stage_times=False)
flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
acc = defaultdict(list)
orig_call = _lib.call


def call(name, *a, **k):
    t0 = time.perf_counter()
    r = orig_call(name, *a, **k)
    acc["native " + name].append(time.perf_counter() - t0)
    return r


_lib.call = call
orig_run = pipeline.GridPlan.run


def run(self, *a, **k):
    t0 = time.perf_counter()
    r = orig_run(self, *a, **k)
    acc["run total"].append(time.perf_counter() - t0)
    return r


pipeline.GridPlan.run = run
args = types.SimpleNamespace(warmup=3, steps=40)
t0 = time.perf_counter()
tot, per, *_ = bench.e2e_stream(plan, rec_host, n, args, lambda: flush_buf.zero_(), lambda: None)
wall = time.perf_counter() - t0
print(f"e2e device ms/step {tot / args.steps:.4f}; wall per step {wall / (args.steps + args.warmup) * 1e3:.4f} ms")
for k in sorted(acc):
    v = np.array(acc[k][-args.steps:]) * 1e6
    print(f"{k:40s} median {np.median(v):8.1f} us  min {v.min():8.1f}  max {v.max():8.1f}  (last {len(v)})")
