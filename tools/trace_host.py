"""Merged host/GPU timeline of one warm fused pass (torch.profiler / CUPTI):
runtime API calls on the host (launches, graph launches, synchronisations)
next to the GPU ops, offsets from the step start (GPU box helper).

    python tools/trace_host.py [C2] [e2e]
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402
from paper_2502_16310_b200 import pipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = bench.CONFIGS[name]
data = bench.make_input(cfg)
n = int.from_bytes(data[80:84], "little")
rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
dim = cfg["dim"]
dom = ow.Aabb(np.zeros(dim), np.ones(dim))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
plan = pipeline.GridPlan(dom, (cfg["root"],) * dim, params, cfg["lattice"], reuse_outputs=True, stage_times=False)
for _ in range(5):
    plan.run(rec, n)
torch.cuda.synchronize()
out = os.path.join("gpurun_out", f"trace_host_{name}.json")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        with torch.profiler.record_function("step"):
            plan.run(rec, n)
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
steps = sorted([e for e in ev if e.get("name") == "step" and e.get("ph") == "X" and e.get("cat") == "user_annotation"], key=lambda e: e["ts"])
s = steps[-1]
t0, t1 = s["ts"], s["ts"] + s["dur"]
rows = []
for e in ev:
    if e.get("ph") != "X" or not (t0 <= e["ts"] <= t1):
        continue
    cat = e.get("cat", "")
    if cat in ("kernel", "gpu_memcpy", "gpu_memset"):
        rows.append((e["ts"] - t0, e["dur"], "GPU", e["name"].replace("(anonymous namespace)::", "")[:60]))
    elif cat == "cuda_runtime" or cat == "cuda_driver":
        rows.append((e["ts"] - t0, e["dur"], "CPU", e["name"][:60]))
rows.sort()
print(f"step wall {s['dur']:.1f} us")
for ts, d, who, nm in rows:
    print(f"{ts:9.1f} {d:7.1f}  {who}  {nm}")
