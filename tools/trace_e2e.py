"""Merged host/GPU timeline of the bench's e2e stream (two plans alternating,
pinned STL bytes in, results out; torch.profiler / CUPTI), offsets from the
first op of the last traced steps (GPU box helper):

    python tools/trace_e2e.py [C2]
"""

import json
import os
import sys
import types

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
rec_host = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).pin_memory()
dim = cfg["dim"]
dom = ow.Aabb(np.zeros(dim), np.ones(dim))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
plan = pipeline.GridPlan(dom, (cfg["root"],) * dim, params, cfg["lattice"], reuse_outputs=True, stage_times=False)
flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def l2_flush():
    flush_buf.fill_(1.0)


args = types.SimpleNamespace(warmup=3, steps=4)
bench.e2e_stream(plan, rec_host, n, args, l2_flush, lambda: None)
torch.cuda.synchronize()
out = os.path.join("gpurun_out", f"trace_e2e_{name}.json")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    bench.e2e_stream(plan, rec_host, n, args, l2_flush, lambda: None)
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
rows = []
for e in ev:
    if e.get("ph") != "X":
        continue
    cat = e.get("cat", "")
    if cat in ("kernel", "gpu_memcpy", "gpu_memset"):
        who = "GPU" if cat == "kernel" else "CPY"
        rows.append((e["ts"], e["dur"], who, e["name"].replace("(anonymous namespace)::", "")[:50]))
    elif cat in ("cuda_runtime", "cuda_driver") and e["dur"] > 4:
        rows.append((e["ts"], e["dur"], "CPU", e["name"][:50]))
rows.sort()
# the last two steps: from the second-to-last k_stl_to_soa
starts = [r[0] for r in rows if r[2] == "GPU" and r[3].startswith("k_stl_to_soa")]
t0 = starts[-2]
for ts, d, who, nm in rows:
    if ts >= t0 - 120:
        if who == "GPU" and d < 6 and not nm.startswith(("k_stl", "k_lat", "k_mark", "k_g2g", "void at::")):
            continue
        print(f"{ts - t0:9.1f} {d:7.1f}  {who}  {nm}")
