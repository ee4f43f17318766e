"""Oracle: boundary-surface extraction and OBJ frame text.

Restates `extract_surface_arrays` (intact/mesh.py:106-124) and
`surface_subset` / `export_frame` (intact/io_utils.py:22-43), paths relative
to /root/reference/pkg/src.  Test infrastructure only —
see oracle/__init__.py.
"""

from __future__ import annotations

import numpy as np

# face r of a tet is opposite vertex r, wound outward (intact/mesh.py _TET_FACES)
TET_FACES = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]], dtype=np.int64)


def extract_surface_arrays(tets):
    """(boundary tris in face order, unique sorted edges, unique vertices,
    non-manifold edge count) — intact/mesh.py:106-124."""
    tets = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    if len(tets) == 0:
        return (np.zeros((0, 3), np.int64), np.zeros((0, 2), np.int64), np.zeros(0, np.int64), 0)
    faces = tets[:, TET_FACES].reshape(-1, 3)
    _, inverse, counts = np.unique(np.sort(faces, axis=1), axis=0, return_inverse=True, return_counts=True)
    boundary = faces[counts[inverse.ravel()] == 1]
    edges = np.sort(boundary[:, [[0, 1], [1, 2], [2, 0]]].reshape(-1, 2), axis=1)
    uniq, ecount = np.unique(edges, axis=0, return_counts=True)
    return boundary, uniq.reshape(-1, 2), np.unique(boundary), int((ecount > 2).sum())


def surface_subset(triangles):
    """(used vertex ids, faces renumbered against them) — intact/io_utils.py:22-32."""
    triangles = np.asarray(triangles, dtype=np.int64)
    used = np.unique(triangles)
    remap = np.zeros(int(used.max()) + 1 if len(used) else 0, dtype=np.int64)
    remap[used] = np.arange(len(used))
    return used, remap[triangles]


def obj_text(positions, triangles) -> str:
    """The bytes export_frame writes (intact/io_utils.py:35-43)."""
    used, faces = surface_subset(triangles)
    lines = [f"v {float(p[0])!r} {float(p[1])!r} {float(p[2])!r}" for p in np.asarray(positions)[used]]
    lines += [f"f {a + 1} {b + 1} {c + 1}" for a, b, c in faces.reshape(-1, 3)]
    return "\n".join(lines) + ("\n" if lines else "")
