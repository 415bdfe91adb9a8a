"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain NumPy restatement of the reference (`octowall`, /root/reference/pkg)
algorithm for the geometry-to-grid hot path, used exclusively as the parity
checker by ``tests/``, by ``__graft_entry__.smoke()`` and by the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  The product
package (``paper_2502_16310_b200``) never imports it: the product path runs
the sm_100a CUDA library or fails loudly.

Parity pinning: every function here is checked bit-for-bit against golden
vectors produced by running the real reference in the build container
(``tests/golden/make_golden.py``; fixtures ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.  The lattice-link / q extension
(``oracle.lattice``) has no reference counterpart: it is pinned by analytic
known-answer tests only ("parity unpinned by reference").

Modules
    geometry   STL / primitive import, index->coords gather, face validation
    binning    BinGrid constants, face discretisation, fill_bins (CSR)
    predicate  FP32 near-face predicates (Algorithm 1), fixed op order
    forest     forest-of-octrees SoA, descent lookup, split, 2:1 balance
    nearwall   marking (naive / binned), propagation, refine driver, links
    lattice    D2Q9 / D3Q19 / D3Q27 boundary links + q (extension)
"""

from . import binning, forest, geometry, lattice, nearwall, predicate  # noqa: F401
