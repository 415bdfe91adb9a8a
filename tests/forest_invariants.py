"""Size-independent invariants of a forest of octrees / quadtrees
(forest.py:300-370): used on full-size device forests (tests/test_gpu_fullsize.py)
and checked here against oracle forests (tests/test_oracle_golden.py)."""

import numpy as np


def check_forest_invariants(level, coords, parent, first_child, root):
    """Parent/child consistency, child-id allocation, and 2:1 balance across
    every face (forest.py:300-370), vectorised over all blocks."""
    n, dim = coords.shape
    nc = 1 << dim
    R = int(np.prod(root))
    # roots: x-fastest lattice, level 0, no parent
    assert np.all(level[:R] == 0) and np.all(parent[:R] == -1)
    assert np.all(level[R:] > 0) and np.all(parent[R:] >= 0)
    # parent / child consistency: each split block owns 2^D consecutive ids
    sp = np.flatnonzero(first_child >= 0)
    fc = first_child[sp]
    assert np.all((fc - R) % nc == 0)
    assert np.unique(fc).size == fc.size  # no two parents share children
    assert fc.size * nc == n - R  # the child groups tile [R, n)
    for ci in range(nc):
        ch = fc + ci
        assert np.all(parent[ch] == sp)
        assert np.all(level[ch] == level[sp] + 1)
        for a in range(dim):
            np.testing.assert_array_equal(coords[ch, a], 2 * coords[sp, a] + ((ci >> a) & 1))
    # ids are allocated by split calls that take their parents in ascending id
    # (forest.py:300-329, _split_many): in allocation order (ascending first
    # child) the parent ids form ascending runs, at most one per split call
    # (one marking split and at most RS_MAX_ITERS = 26 rebalance sweeps per level)
    order = sp[np.argsort(fc, kind="stable")]
    runs = 1 + int(np.sum(np.diff(order) < 0)) if order.size else 0
    assert runs <= 27 * (int(level.max()) + 1), f"{runs} allocation runs"
    # 2:1 balance: for a block b at level l >= 1 and every face, the level
    # l-1 lattice block holding b's neighbour cell exists (no leaf coarser
    # than l-1 touches b)
    key = lambda lv, c: ((lv << 58) | sum(c[:, a] << (29 * a) for a in range(dim)) if dim == 2 else  # noqa: E731
                         (lv << 60) | (c[:, 0]) | (c[:, 1] << 20) | (c[:, 2] << 40))
    keys = np.sort(key(level, coords))
    nb = np.flatnonzero(level >= 1)
    lv = level[nb]
    for a in range(dim):
        for step in (-1, 1):
            c = coords[nb].copy()
            c[:, a] += step
            ext = root[a] << lv
            ok = (c[:, a] >= 0) & (c[:, a] < ext)
            k = key(lv[ok] - 1, c[ok] >> 1)
            pos = np.searchsorted(keys, k)
            found = (pos < keys.size) & (keys[np.minimum(pos, keys.size - 1)] == k)
            assert found.all(), f"2:1 balance violated at {int((~found).sum())} block faces"
