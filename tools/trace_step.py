"""GPU timeline of bench steps with torch.profiler (CUPTI): kernel gaps and the
host call that was running during each gap (GPU box helper).

    python tools/trace_step.py [C2] [steps] [e2e]

``e2e``: the bench's e2e step (pinned STL bytes in, run(host=True), results
out, stream synchronised) instead of the HBM-resident step.
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = bench.CONFIGS[name]
data = bench.make_input(cfg)
n = int.from_bytes(data[80:84], "little")
e2e = len(sys.argv) > 3 and sys.argv[3] == "e2e"
rec_host = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).pin_memory()
rec = rec_host.cuda()
dim = cfg["dim"]
dom = ow.Aabb(np.zeros(dim), np.ones(dim))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])


from paper_2502_16310_b200 import pipeline  # noqa: E402


plan = pipeline.GridPlan(dom, (cfg["root"],) * dim, params, cfg["lattice"], reuse_outputs=True,
                         stage_times=False)  # as the bench's timed loops


def step():
    if e2e:
        rd = rec_host.to("cuda", non_blocking=True)
        plan.run(rd, n, host=True)
        torch.cuda.current_stream().synchronize()
    else:
        plan.run(rec, n)


for _ in range(3):
    step()
torch.cuda.synchronize()
out = os.path.join("gpurun_out", f"trace_{name}{'_e2e' if e2e else ''}.json")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        with torch.profiler.record_function("step"):
            step()
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
kern = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")], key=lambda e: e["ts"])
steps_ev = sorted([e for e in ev if e.get("name") == "step" and e.get("ph") == "X" and e.get("cat") == "user_annotation"], key=lambda e: e["ts"])
s = steps_ev[-1]
t0, t1 = s["ts"], s["ts"] + s["dur"]
ks = [k for k in kern if t0 <= k["ts"] <= t1]
busy = sum(k["dur"] for k in ks)
print(f"last step: wall {s['dur']:.1f} us, GPU busy {busy:.1f} us in {len(ks)} GPU ops")
gaps = []
for a, b in zip(ks, ks[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    if g > 5:
        gaps.append((g, a["name"][:50], b["name"][:50], b["ts"]))
print(f"idle between GPU ops: {sum(g for g, *_ in gaps):.1f} us in {len(gaps)} gaps > 5 us; first op at +{ks[0]['ts'] - t0:.1f} us")
cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("cpu_op", "user_annotation", "python_function")]
for g, a, b, ts in sorted(gaps, reverse=True)[:8]:
    print(f"{g:8.1f} us  after {a:50s} before {b}")
agg = {}
for k in ks:
    nm = k["name"].replace("(anonymous namespace)::", "").split("(")[0][:60]
    c, t = agg.get(nm, (0, 0.0))
    agg[nm] = (c + 1, t + k["dur"])
print("per kernel (last step):")
for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{t:9.1f} us {c:4d}x  {nm}")
print("copies (last step, offset from step start):")
for k in ks:
    if k.get("cat") in ("gpu_memcpy", "gpu_memset"):
        b = k.get("args", {}).get("bytes", 0)
        print(f"  +{k['ts'] - t0:8.1f} us {k['dur']:7.1f} us {b:>10} B  {k['name'][:40]}")
print(f"last GPU op ends at +{max(k['ts'] + k['dur'] for k in ks) - t0:.1f} us of a {s['dur']:.1f} us step")
