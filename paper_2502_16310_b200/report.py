"""Bin-density sweep: the reference's `sweep` (cli.py:137-174) over the GPU
pipeline, with its CSV schema (report.py:16-41).  Figures (matplotlib) are
out of scope; the CSV is the canonical artifact.

A sweep is also the C3 benchmark configuration of BASELINE.json (bunny-scale
STL, 4 levels, bin-density sweep): ``tools/sweep_c3.py`` runs it (``profiles/r01_sweep_c3.csv``).
"""

from __future__ import annotations

import sys
import time
from dataclasses import dataclass

import torch

from .errors import OctowallError
from .forest import DEFAULT_MAX_LEVEL, init_root_grid
from .nearwall import NearWallParams, refine_near_wall

SWEEP_CSV_HEADER = "B,bin_setup_ms,face_detect_ms,total_ms,blocks_marked,blocks_final"


@dataclass
class SweepRow:
    bins_per_axis: int
    bin_setup_ms: float
    face_detect_ms: float
    total_ms: float
    blocks_marked: int
    blocks_final: int
    error: str = ""

    def csv_row(self):
        return (f"{self.bins_per_axis},{self.bin_setup_ms:.3f},{self.face_detect_ms:.3f},"
                f"{self.total_ms:.3f},{self.blocks_marked},{self.blocks_final}")


def write_sweep_csv(path, rows):
    with open(path, "w", encoding="utf-8") as f:
        f.write(SWEEP_CSV_HEADER + "\n")
        for r in rows:
            if not r.error:
                f.write(r.csv_row() + "\n")


def sweep(geom, domain, root_dims, d_spec, n_levels, bin_densities, bin_fraction=None, backend="serial",
          max_level=DEFAULT_MAX_LEVEL, out_csv=None, verbose=True):
    """One pipeline run per bin density; B=1 runs the naive strategy.  Stage
    times are device-event milliseconds; total_ms is the wall time of the
    refine_near_wall call (synchronised)."""
    rows = []
    for b in bin_densities:
        strategy = "naive" if b == 1 else "binned"
        try:
            forest = init_root_grid(domain, root_dims, max_level=max_level)
            params = NearWallParams(d_spec=d_spec, n_levels=n_levels, strategy=strategy, bins_per_axis=b,
                                    bin_fraction=bin_fraction, backend=backend)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            result = refine_near_wall(forest, geom, params)
            torch.cuda.synchronize()
            total = 1e3 * (time.perf_counter() - t0)
            rows.append(SweepRow(bins_per_axis=b, bin_setup_ms=result.total_ms("bin_setup"),
                                 face_detect_ms=result.total_ms("face_detection"), total_ms=total,
                                 blocks_marked=result.total_marked, blocks_final=sum(forest.leaves_per_level())))
            if verbose:
                print(f"B={b}: total {total:.1f} ms, marked {result.total_marked}", file=sys.stderr)
        except OctowallError as e:
            rows.append(SweepRow(b, 0, 0, 0, 0, 0, error=str(e)))
            if verbose:
                print(f"B={b}: FAILED: {e}", file=sys.stderr)
    if out_csv:
        write_sweep_csv(out_csv, rows)
    return rows
