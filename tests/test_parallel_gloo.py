"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

The marking slice of each rank is played by the CPU oracle (test-only), and
the gather of per-leaf marks goes through the same ``parallel`` functions the
NCCL path uses; the gathered forest must equal a single-process run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import binning as ob
        from oracle import forest as of
        from oracle import nearwall as on
        from paper_2502_16310_b200 import parallel

        from oracle.geometry import circle, index_to_coords

        coords = index_to_coords(*circle(0.5, 0.5, 0.25, 400))
        f = of.Forest((0, 0), (1, 1), (16, 16))
        grid = ob.Grid((0, 0), (1, 1), 8)
        bins = ob.fill_bins(coords, grid)
        for level in range(2):
            leaves = f.leaves_at(level)
            lo, hi = parallel.partition(len(leaves), rank, world)
            # rank-local marking on a private copy restricted to its slice
            sub = of.Forest((0, 0), (1, 1), (16, 16))
            sub.__dict__.update({k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in f.__dict__.items()})
            keep = np.zeros(f.n, bool)
            keep[leaves[lo:hi]] = True
            others = np.flatnonzero(~keep & (sub.level == level))
            saved = sub.first_child[others].copy()
            sub.first_child[others] = 0  # hide other ranks' leaves from leaves_at()
            on.mark(sub, level, coords, 0.1, bins, grid)
            sub.first_child[others] = saved
            mine = torch.from_numpy(sub.marks[leaves[lo:hi]].copy())
            allm, _ = parallel.gather_slices(mine, len(leaves), world)
            f.marks[leaves] = allm.numpy()
            on.propagate(f, level, 0.1)
            f.refine_marked(level)
        q.put((rank, f.level.copy(), f.coords.copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_marking_gather_matches_single_process():
    from oracle import binning as ob
    from oracle import forest as of
    from oracle import nearwall as on
    from oracle.geometry import circle, index_to_coords

    coords = index_to_coords(*circle(0.5, 0.5, 0.25, 400))
    ref = of.Forest((0, 0), (1, 1), (16, 16))
    on.refine_near_wall(ref, coords, 0.1, n_levels=3, bins_per_axis=8)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, level, co in got:
        np.testing.assert_array_equal(level, ref.level)
        np.testing.assert_array_equal(co, ref.coords)


def test_partition_covers_and_balances():
    from paper_2502_16310_b200.parallel import partition

    for n in (0, 1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            spans = [partition(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
    w = torch.ones(100, dtype=torch.float64)
    w[:10] = 50.0
    spans = [partition(100, r, 4, w) for r in range(4)]
    assert spans[0][1] <= 10  # heavy head goes to rank 0 alone
