"""Break down bench.py's e2e step on the GPU box: the same loop as the bench
(event-bracketed GridPlan.run(host=True) from pinned STL bytes, stream
synchronised) with and without the L2 flush, and the H2D / D2H legs alone.

    python tools/probe_e2e.py [C2] [steps]
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402
from paper_2502_16310_b200 import pipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = bench.CONFIGS[name]
from paper_2502_16310_b200 import _lib  # noqa: E402

nodes = [d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")]
print(f"numa nodes {len(nodes)}, GPU node {_lib.device_numa_node(0)}, cpus allowed {len(os.sched_getaffinity(0))}")
if os.environ.get("OW_BIND"):
    print("bound to node", _lib.bind_host_numa(0), "cpus", len(os.sched_getaffinity(0)))
data = bench.make_input(cfg)
n = int.from_bytes(data[80:84], "little")
rec_host = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).pin_memory()
dim = cfg["dim"]
dom = ow.Aabb(np.zeros(dim), np.ones(dim))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
plan = pipeline.GridPlan(dom, (cfg["root"],) * dim, params, cfg["lattice"], reuse_outputs=True)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def loop(with_flush, host=True):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    wall = 0.0
    torch.cuda.synchronize()
    for k in range(steps):
        if with_flush:
            flush.zero_()
        ev[k][0].record()
        t0 = time.perf_counter()
        rd = rec_host.to("cuda", non_blocking=True)
        plan.run(rd, n, host=host)
        torch.cuda.current_stream().synchronize()
        wall += time.perf_counter() - t0
        ev[k][1].record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / steps, 1e3 * wall / steps


for _ in range(3):
    loop(True)
for fl in (True, False, True):
    for host in (True, False):
        ms, wall = loop(fl, host)
        print(f"flush={fl} host={host}: event {ms:.3f} ms/step, host wall {wall:.3f} ms/step")
gp = plan.run(rec_host.to("cuda"), n, host=True)
torch.cuda.synchronize()
q = gp.links.q
hq = torch.empty(q.numel(), dtype=torch.float32, pin_memory=True)
for _ in range(3):
    hq.copy_(q.reshape(-1), non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    hq.copy_(q.reshape(-1), non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"q D2H alone: {q.numel() * 4} B in {1e3 * dt:.3f} ms = {q.numel() * 4 / dt / 1e9:.1f} GB/s")
d = torch.empty(rec_host.numel(), dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d.copy_(rec_host, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"records H2D alone: {rec_host.numel()} B in {1e3 * dt:.3f} ms = {rec_host.numel() / dt / 1e9:.1f} GB/s")
