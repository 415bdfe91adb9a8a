"""Stage-by-stage wall-clock probe of one bench configuration (GPU box helper).

    python tools/probe_stages.py [C2]
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402
from paper_2502_16310_b200 import _lib  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = bench.CONFIGS[name]
    data = bench.make_input(cfg)
    dim = cfg["dim"]
    dom = ow.Aabb(np.zeros(dim), np.ones(dim))
    rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
    n = int.from_bytes(data[80:84], "little")
    params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
    for it in range(4):
        torch.cuda.synchronize()
        t = {}
        t0 = time.perf_counter()
        geom = ow.geometry.stl_records_to_coords(rec, n)
        torch.cuda.synchronize()
        t["import"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        f = ow.init_root_grid(dom, (cfg["root"],) * dim, capacity=32 * cfg["root"] ** dim)
        torch.cuda.synchronize()
        t["init"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        res = ow.refine_near_wall(f, geom, params)
        torch.cuda.synchronize()
        t["refine_near_wall"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        ll = ow.build_lattice_links(f, geom, ow.BinGrid(dom, cfg["B"]), cfg["lattice"])
        torch.cuda.synchronize()
        t["lattice"] = time.perf_counter() - t0
        if it == 3:
            for k, v in t.items():
                print(f"{k:18s} {1e3 * v:8.3f} ms")
            for s in res.timings:
                print("   ", s.csv_row())
            print("blocks", f.blocks_per_level(), "boundary", ll.n_boundary, "launches", _lib.launches())
    # refinement cost with and without forest growth
    for cap in (8 * cfg["root"] ** dim, 64 * cfg["root"] ** dim):
        f = ow.init_root_grid(dom, (cfg["root"],) * dim, capacity=cap)
        geom = ow.geometry.stl_records_to_coords(rec, n)
        grid = ow.BinGrid(dom, cfg["B"])
        bins = ow.fill_bins(geom, grid)
        for level in range(cfg["levels"] - 1):
            ow.mark_near_wall_binned(f, level, geom, bins, grid, cfg["d"])
            ow.propagate_marks(f, level, cfg["d"])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ns = f.refine_marked(level)
            torch.cuda.synchronize()
            print(f"cap {cap:8d} level {level} refine {1e3 * (time.perf_counter() - t0):8.3f} ms split {ns}")


if __name__ == "__main__":
    main()
