"""Legacy ASCII VTK export of the forest's leaf blocks (vtk_io.py:17-69).

Written natively (``ow_export_vtk``): one device->host copy of the block
arrays, FP64 leaf boxes with the reference's formula, parallel host
formatting.  The file is byte-identical to the reference's.
"""

from __future__ import annotations

import ctypes as C
import os

from . import _lib
from .forest import Forest


def export_vtk(forest: Forest, path, title="octowall leaf blocks"):
    """Write the forest's leaves as a VTK unstructured grid."""
    _lib.call("ow_export_vtk", _lib.ctx(), C.byref(forest.view()), os.fsencode(path), title.encode("utf-8"),
              _lib.stream())
