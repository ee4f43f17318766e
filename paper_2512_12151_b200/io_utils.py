"""Frame export (intact/io_utils.py:1-43) through the native writer.

`export_frame` writes the same bytes as the reference — the vertices the
triangles use, in ascending id order, coordinates as repr(float), then the
faces renumbered 1-based — with the formatting spread over host threads
(csrc/export.cpp).  It needs libibf.so but no GPU; positions may be a CUDA
tensor (copied to the host first).
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib


def surface_subset(positions, triangles):
    """(vertex ids into positions, faces renumbered against them) —
    intact/io_utils.py:22-32 (host numpy; the writer does this natively)."""
    triangles = np.asarray(triangles, dtype=np.int64)
    used = np.unique(triangles)
    remap = np.zeros(int(used.max()) + 1 if len(used) else 0, dtype=np.int64)
    remap[used] = np.arange(len(used))
    return used, remap[triangles]


def export_frame(positions, triangles, path, threads: int = 0) -> None:
    """Write the surface at `positions` as an OBJ mesh (intact/io_utils.py:35-43)."""
    if hasattr(positions, "detach"):
        positions = positions.detach().cpu().numpy()
    x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, dtype=np.int64).reshape(-1, 3)
    _lib.check(_lib.lib().ibf_export_obj(os.fsencode(path), _lib.host_ptr(x), len(x), _lib.host_ptr(t), len(t),
                                         int(threads)), "ibf_export_obj")
