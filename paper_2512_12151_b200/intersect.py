"""Penetration certificate on the device (intact/intersect.py; SURVEY.md
§8(f) f1): the reference's static triangle-triangle intersection test, and
a nearest-pair monitor, both over the CCD handle's LBVH broad phase."""

from __future__ import annotations

import numpy as np

from .ccd import CCD
from .device import to_dev


def static_intersection_test(x, tris) -> np.ndarray:
    """All intersecting surface triangle pairs (k,2), a < b, shared-vertex
    pairs excluded (intact/intersect.py:125-140), ascending."""
    tris = np.ascontiguousarray(tris, dtype=np.int64).reshape(-1, 3)
    if len(tris) == 0:
        return np.empty((0, 2), dtype=np.int64)
    handle = CCD(tris, np.zeros((0, 2), dtype=np.int64), np.zeros(0, dtype=np.int64))
    xd = to_dev(np.ascontiguousarray(x, dtype=np.float64)) if isinstance(x, np.ndarray) else x
    n, pairs = handle.static_intersections(xd, cap=1 << 20)
    if n > len(pairs):
        n, pairs = handle.static_intersections(xd, cap=n)
    return pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))] if len(pairs) else pairs.reshape(0, 2)
