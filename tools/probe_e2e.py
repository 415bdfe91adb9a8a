"""Break down the e2e step of bench.py (H2D, step, D2H) on the GPU box."""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402

cfg = bench.CONFIGS["C2"]
data = bench.make_input(cfg)
n = int.from_bytes(data[80:84], "little")
host = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).pin_memory()
dom = ow.Aabb(np.zeros(3), np.ones(3))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
pinned = {}
for it in range(6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    rd = host.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    geom = ow.geometry.stl_records_to_coords(rd, n)
    f = ow.init_root_grid(dom, (16, 16, 16), capacity=8 * 4096)
    res = ow.refine_near_wall(f, geom, params)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    ll = ow.build_lattice_links(f, geom, None, cfg["lattice"])
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    outs = [f.level_tensor, f.coords_tensor, f._parent_t[: f.n_blocks], f._first_child_t[: f.n_blocks], f.marks,
            ll.flags, ll.cells, ll.q]
    for i, o in enumerate(outs):
        nb = o.numel() * o.element_size()
        if i not in pinned or pinned[i].numel() < nb:
            pinned[i] = torch.empty(2 * nb + 64, dtype=torch.uint8, pin_memory=True)
        pinned[i][:nb].copy_(o.contiguous().view(-1).view(torch.uint8), non_blocking=True)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    d = np.diff(np.array(t)) * 1e3
    print(f"h2d {d[0]:.3f}  refine {d[1]:.3f}  lattice {d[2]:.3f}  d2h {d[3]:.3f} ms")
