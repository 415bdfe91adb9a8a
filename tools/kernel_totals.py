"""Per-kernel GPU time of one warm fused pass (torch.profiler / CUPTI) for
A/B comparisons (GPU box helper):  python tools/kernel_totals.py C5"""

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
for _ in range(4):
    gp = plan.run(rec, n)
torch.cuda.synchronize()
print("device_sized", gp.device_sized)
out = os.path.join("gpurun_out", f"ktot_{name}.json")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    with torch.profiler.record_function("step"):
        plan.run(rec, n)
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and e.get("ph") == "X"]
t0 = min(k["ts"] for k in ks)
t1 = max(k["ts"] + k["dur"] for k in ks)
agg = {}
for k in ks:
    nm = k["name"].replace("(anonymous namespace)::", "").split("(")[0][:60]
    c, t = agg.get(nm, (0, 0.0))
    agg[nm] = (c + 1, t + k["dur"])
print(f"span {t1 - t0:.1f} us, busy {sum(k['dur'] for k in ks):.1f} us")
for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{t:9.1f} us {c:4d}x  {nm}")
