"""Loading of the reference-generated golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import glob
import hashlib
import os

import numpy as np

from oracle import geometry as og

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# geometries too large to store inline are regenerated from their recipe and
# checked against the SHA-256 recorded by make_golden.py
_RECIPES = {
    "sphere224x250": lambda: og.index_to_coords(*og.latlon_sphere(0.5, 0.5, 0.5, 0.3, 224, 250)),
}


def files(prefix):
    return sorted(glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def ids(paths):
    return [os.path.basename(p)[:-4] for p in paths]


def load(path):
    z = np.load(path, allow_pickle=False)
    return {k: z[k] for k in z.files}


def geometry(g):
    """float32 coords (D, D, F) of a fixture, verified against its hash."""
    if "geom_coords" in g:
        c = np.ascontiguousarray(g["geom_coords"], np.float32)
    else:
        c = np.ascontiguousarray(_RECIPES[str(g["geom_name"])](), np.float32)
    assert hashlib.sha256(c.tobytes()).hexdigest() == str(g["geom_sha"]), "geometry recipe drifted"
    return c


def unit_domain(dim):
    return np.zeros(dim), np.ones(dim)
