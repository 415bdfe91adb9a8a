"""Stage the real reference package for the CPU baseline (test / bench
infrastructure; the recipe oracle/_ref is built from).

The reference (``octowall``) is pure Python + NumPy: there is nothing to
compile, and ``/root/reference`` exists only in the build container.  This
recipe copies its package sources, unmodified, from
``/root/reference/pkg/src/octowall`` into the git-ignored ``oracle/_ref/``,
which travels to the GPU box with the repository snapshot like a built
``.so``.  ``bench.py --impl reference`` (and the ``cpu_baseline`` leg) then
time the reference's own serial code path there (``cpu_baseline.kind =
"reference"``); where ``oracle/_ref`` is absent they fall back to the NumPy
restatement in ``oracle/`` (``kind = "port"``).  Nothing in the product
imports either.

    python -m oracle.stage_ref          # (also run by __graft_entry__.build())
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/pkg/src/octowall"
DST = os.path.join(HERE, "_ref", "octowall")
MANIFEST = os.path.join(HERE, "_ref", "MANIFEST.json")
# the geometry-to-grid path (cli.py:87-113) needs only these modules; the CLI
# and the matplotlib report are left out (matplotlib is not installed)
MODULES = ("__init__.py", "backends.py", "binning.py", "distance.py", "errors.py", "forest.py", "geometry.py",
           "nearwall.py", "validate.py", "vtk_io.py")


def _sha(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def stage(force=False):
    """Copy the reference modules into oracle/_ref/octowall; returns the
    staged directory, or None when the reference is not present here."""
    if not os.path.isdir(SRC):
        return DST if os.path.isdir(DST) else None
    want = {m: _sha(os.path.join(SRC, m)) for m in MODULES}
    if not force and os.path.exists(MANIFEST):
        try:
            with open(MANIFEST) as fh:
                if json.load(fh).get("sha256") == want:
                    return DST
        except (OSError, ValueError):
            pass
    tmp = DST + ".tmp"
    shutil.rmtree(tmp, ignore_errors=True)
    os.makedirs(tmp)
    for m in MODULES:
        shutil.copyfile(os.path.join(SRC, m), os.path.join(tmp, m))
    shutil.rmtree(DST, ignore_errors=True)
    os.replace(tmp, DST)
    with open(MANIFEST, "w") as fh:
        json.dump({"source": SRC, "sha256": want}, fh, indent=1)
    return DST


def available():
    return os.path.exists(os.path.join(DST, "__init__.py"))


def import_reference():
    """The staged ``octowall`` module (its directory on sys.path first)."""
    import importlib
    import sys

    if not available():
        raise ImportError("oracle/_ref/octowall is not staged (python -m oracle.stage_ref)")
    root = os.path.dirname(DST)
    if root not in sys.path:
        sys.path.insert(0, root)
    return importlib.import_module("octowall")


if __name__ == "__main__":
    print(stage(force=True))
