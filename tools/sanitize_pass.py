"""Small workloads for compute-sanitizer (GPU box helper): a 2D pass through
the per-function API (text primitive -> refine_near_wall -> lattice links)
and a 3D fused GridPlan pass with host outputs, plus fill_bins and the
cell-face links.  tools/sanitize.sh runs it under memcheck, racecheck,
synccheck and initcheck."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16310_b200 as ow  # noqa: E402
from paper_2502_16310_b200 import pipeline, shapes  # noqa: E402

torch.cuda.set_device(0)
ig = ow.generate_circle((0.5, 0.5), 0.25, 256)
geom = ow.index_to_coords(ig)
f = ow.init_root_grid(ow.Aabb((0, 0), (1, 1)), (8, 8))
ow.refine_near_wall(f, geom, ow.NearWallParams(d_spec=0.1, n_levels=3, bins_per_axis=8))
grid = ow.BinGrid(ow.Aabb((0, 0), (1, 1)), 8)
ll = ow.build_lattice_links(f, geom, grid, "D2Q9")
links = ow.build_cell_face_links(f, geom, ow.fill_bins(geom, grid), grid, capacity=64)
data = shapes.binary_stl_bytes(shapes.icosphere_triangles(3))
n = int.from_bytes(data[80:84], "little")
rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
plan = pipeline.GridPlan(ow.Aabb(np.zeros(3), np.ones(3)), (8, 8, 8),
                         ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8), "D3Q19", reuse_outputs=True)
for _ in range(2):
    gp = plan.run(rec, n, host=True)
torch.cuda.synchronize()
# device-sized passes (single readback, graph capture and replay) through two
# plans with the next pass submitted before the previous one is finished, a
# pass that outgrows the estimates (synchronous fallback) and deferred copies
plans = [pipeline.GridPlan(ow.Aabb(np.zeros(3), np.ones(3)), (8, 8, 8),
                           ow.NearWallParams(d_spec=0.06, n_levels=3, bins_per_axis=8), "D3Q19", reuse_outputs=True,
                           stage_times=False) for _ in range(2)]
big = shapes.binary_stl_bytes(shapes.icosphere_triangles(4, radius=0.32))
recs = [(rec, n)] * 4 + [(torch.frombuffer(bytearray(big[84:]), dtype=torch.uint8).cuda(),
                          int.from_bytes(big[80:84], "little"))] * 2 + [(rec, n)] * 2
prev, modes = None, []
for k, (r, nn) in enumerate(recs):
    pend = plans[k % 2].run_async(r, nn, host=True, defer=True)
    if prev is not None:
        g = prev.result()
        g.wait()
        modes.append(g.device_sized)
    prev = pend
g = prev.result()
g.wait()
torch.cuda.synchronize()
print("sanitize pass OK:", f.blocks_per_level(), ll.n_boundary, gp.forest.blocks_per_level(), gp.links.n_boundary,
      "device-sized modes", modes + [g.device_sized])
