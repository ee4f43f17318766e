"""Tet meshes, rest data and simulation state (intact/mesh.py:23-152).

One-time host-side preprocessing (out of the hot path): the outputs —
shape rows, volumes, lumped masses, surface triangles/edges/vertices — are
the inputs the device system is built from.  Same conventions as the
reference so scenes built here and there are interchangeable.
"""

from __future__ import annotations

import dataclasses
import logging

import numpy as np

log = logging.getLogger(__name__)

# faces opposite vertices 0..3 of a positively oriented tet, wound outward
_TET_FACES = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]], dtype=np.int64)
DEGENERATE_VOLUME_FRACTION = 1e-12


class MeshError(ValueError):
    """Malformed mesh input."""


@dataclasses.dataclass
class TetMesh:
    rest_positions: np.ndarray
    tets: np.ndarray
    surface_tris: np.ndarray
    surface_edges: np.ndarray
    surface_verts: np.ndarray

    @property
    def n_verts(self) -> int:
        return self.rest_positions.shape[0]

    @property
    def n_tets(self) -> int:
        return self.tets.shape[0]


@dataclasses.dataclass
class RestData:
    inv_rest_shape: np.ndarray
    volumes: np.ndarray
    shape_rows: np.ndarray
    masses: np.ndarray


@dataclasses.dataclass
class SimState:
    """Positions and velocities of every vertex, (n,3) float64 each."""

    x: np.ndarray
    v: np.ndarray

    def copy(self) -> "SimState":
        return SimState(self.x.copy(), self.v.copy())


def tet_volumes(positions, tets):
    p = positions[tets]
    return np.linalg.det((p[:, 1:] - p[:, :1]).transpose(0, 2, 1)) / 6.0


def surface_of(tets):
    """Boundary faces (seen once), their unique sorted edges and vertices."""
    if len(tets) == 0:
        return (np.zeros((0, 3), dtype=np.int64), np.zeros((0, 2), dtype=np.int64),
                np.zeros(0, dtype=np.int64))
    faces = tets[:, _TET_FACES].reshape(-1, 3)
    _, inv, cnt = np.unique(np.sort(faces, axis=1), axis=0, return_inverse=True, return_counts=True)
    bnd = faces[cnt[inv.ravel()] == 1]
    e = np.sort(bnd[:, [[0, 1], [1, 2], [2, 0]]].reshape(-1, 2), axis=1)
    edges, ecnt = np.unique(e, axis=0, return_counts=True)
    if (ecnt > 2).any():
        log.warning("non-manifold surface: %d edge(s) shared by >2 boundary faces", int((ecnt > 2).sum()))
    return bnd, edges, np.unique(bnd)


def extract_surface_arrays(tets):
    """Boundary faces, their unique sorted edges and vertices, computed on
    the device (csrc/surface.cu): drop-in for intact/mesh.py:106-124 with
    bit-identical outputs.  `tets` is (m,4) int64, numpy or a CUDA tensor;
    the results are numpy int64 arrays.  Needs the GPU (no host fallback;
    `surface_of` is the host preprocessing path of build_tet_mesh)."""
    import ctypes as C
    from . import _lib
    from .device import require_cuda
    torch = require_cuda()
    if isinstance(tets, torch.Tensor):
        td = tets.to(device="cuda", dtype=torch.int64).contiguous()
    else:
        td = torch.from_numpy(np.ascontiguousarray(tets, dtype=np.int64).reshape(-1, 4)).cuda()
    h = C.c_void_p()
    nt, ne, nv, nbad = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().ibf_surface_extract(td.shape[0] if td.numel() else 0, _lib.dev_ptr(td), C.byref(h),
                                              C.byref(nt), C.byref(ne), C.byref(nv), C.byref(nbad), _lib.stream()),
               "ibf_surface_extract")
    try:
        tris = np.empty((nt.value, 3), dtype=np.int64)
        edges = np.empty((ne.value, 2), dtype=np.int64)
        verts = np.empty(nv.value, dtype=np.int64)
        _lib.check(_lib.lib().ibf_surface_get(h, _lib.host_ptr(tris), _lib.host_ptr(edges), _lib.host_ptr(verts),
                                              _lib.stream()), "ibf_surface_get")
    finally:
        _lib.lib().ibf_surface_destroy(h)
    if nbad.value:
        log.warning("non-manifold surface: %d edge(s) shared by >2 boundary faces", nbad.value)
    return tris, edges, verts


def extract_surface(mesh: TetMesh):
    """(surface_tris, surface_edges, surface_verts) recomputed on the device
    (intact/mesh.py:127-129)."""
    return extract_surface_arrays(mesh.tets)


def build_tet_mesh(positions, tets) -> TetMesh:
    """Validate, re-orient negative tets, extract the surface."""
    positions = np.ascontiguousarray(positions, dtype=np.float64)
    tets = np.ascontiguousarray(tets, dtype=np.int64)
    if positions.ndim != 2 or positions.shape[1] != 3:
        raise MeshError(f"positions must be (n, 3), got {positions.shape}")
    if tets.ndim != 2 or tets.shape[1] != 4:
        raise MeshError(f"tets must be (m, 4), got {tets.shape}")
    if tets.size and (tets.min() < 0 or tets.max() >= len(positions)):
        raise MeshError("tet index out of range")
    vols = tet_volumes(positions, tets)
    neg = vols < 0.0
    if neg.any():
        tets = tets.copy()
        tets[neg, 1], tets[neg, 2] = tets[neg, 2], tets[neg, 1].copy()
        vols = np.abs(vols)
    if tets.size:
        floor = DEGENERATE_VOLUME_FRACTION * float(vols.mean())
        bad = np.nonzero(vols <= floor)[0]
        if bad.size:
            raise MeshError(f"degenerate tet(s) {bad.tolist()[:8]}: volume <= {floor:.3e}")
    t, e, v = surface_of(tets)
    return TetMesh(positions, tets, t, e, v)


def _morton3(points, bits=21):
    """Interleaved 3 x `bits`-bit Morton codes of points normalised to their box."""
    lo = points.min(axis=0)
    ext = np.maximum(points.max(axis=0) - lo, 1e-300)
    q = np.minimum(((points - lo) / ext * ((1 << bits) - 1)).astype(np.uint64), (1 << bits) - 1)
    code = np.zeros(len(points), dtype=np.uint64)
    for b in range(bits):
        for a in range(3):
            code |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    return code


def reorder_for_locality(mesh: TetMesh) -> TetMesh:
    """The same mesh with vertices renumbered along a Morton curve of their
    rest positions and tets sorted by their smallest vertex.

    Pure data layout (no reference counterpart; the reference is order
    agnostic): the symmetric SpMV reads each stored block twice (row and
    transposed) and gathers p at the block columns, so both stay L2 hits only
    if a block's rows and columns are near in index.  Lattice-index numbering
    of a sparse lattice (hollow cores, thin strands) puts neighbours up to a
    lattice plane apart; on the squishy-ball scene the PCG's DRAM traffic was
    1.42x its algorithmic bytes with that numbering."""
    perm = np.argsort(_morton3(mesh.rest_positions), kind="stable")
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    tets = inv[mesh.tets]
    tets = tets[np.lexsort((tets.max(axis=1), tets.min(axis=1)))]
    return build_tet_mesh(mesh.rest_positions[perm], tets)


def sell_numbering(n_verts: int, tets: np.ndarray, window: int = 1024, rounds: int = 4) -> np.ndarray:
    """new_of_old: a vertex renumbering that keeps the given order's
    locality at the scale of `window` vertices but sorts each window by
    (upper count, lower count) descending, so the 32 rows of a sliced-ELL
    slice (internal.cuh) have near-equal upper and lower block counts.

    The upper / lower counts of a vertex depend on the numbering itself
    (upper = neighbours numbered after it), so the sort is repeated `rounds`
    times on the counts of the previous round.  On the squishy ball (lattice
    order) this takes the SpMV's upper padding from 26 % to 3 % and the
    lower-list padding from 29 % to 12 % (the upper stream alone reads every
    padded slot's sectors: ncu, 508 MB of DRAM reads for 373 MB of upper
    blocks and columns) — but k_pcg measured 200 vs 185 us per CG iteration
    on it, the standalone SpMV unchanged (rejected), so the
    squishy scene keeps the lattice numbering.  Pure data layout; the
    reference is order agnostic."""
    tets = np.asarray(tets, dtype=np.int64)
    n = int(n_verts)
    pairs = np.concatenate([tets[:, [i, j]] for i in range(4) for j in range(i + 1, 4)])
    lo, hi = pairs.min(axis=1), pairs.max(axis=1)
    key = np.unique(lo * n + hi)
    e0, e1 = key // n, key % n
    new_of = np.arange(n, dtype=np.int64)
    win = np.arange(n, dtype=np.int64) // max(int(window), 1)
    for _ in range(max(int(rounds), 1)):
        a, b = new_of[e0], new_of[e1]
        up = np.bincount(np.minimum(a, b), minlength=n)       # by new position
        low = np.bincount(np.maximum(a, b), minlength=n)
        old_at = np.empty(n, dtype=np.int64)
        old_at[new_of] = np.arange(n)
        k = up * 4096 + low                                    # by new position
        order = np.lexsort((-k, win))                          # positions, window-major, key descending
        new_of = np.empty(n, dtype=np.int64)
        new_of[old_at[order]] = np.arange(n)
    return new_of


def reorder_for_sell(mesh: TetMesh, window: int = 0, rounds: int = 4) -> TetMesh:
    """The same mesh with its vertices renumbered by `sell_numbering`
    (tets keep their order).  window 0: IBF_SELL_NUMBERING_WINDOW or 1024."""
    import os
    window = window or int(os.environ.get("IBF_SELL_NUMBERING_WINDOW", "1024"))
    new_of = sell_numbering(mesh.n_verts, mesh.tets, window, rounds)
    perm = np.empty_like(new_of)
    perm[new_of] = np.arange(len(new_of))
    return build_tet_mesh(mesh.rest_positions[perm], new_of[mesh.tets])


def compute_rest_data(mesh: TetMesh, density: float) -> RestData:
    """Dm^-1, volumes, shape rows A_i (dF = sum dx_i A_i), lumped masses."""
    if density <= 0.0:
        raise MeshError(f"density must be positive, got {density}")
    p = mesh.rest_positions[mesh.tets]
    dm = (p[:, 1:] - p[:, :1]).transpose(0, 2, 1)
    vol = np.linalg.det(dm) / 6.0
    inv = np.linalg.inv(dm)
    rows = np.empty((mesh.n_tets, 4, 3))
    rows[:, 1:] = inv
    rows[:, 0] = -inv.sum(axis=1)
    masses = np.zeros(mesh.n_verts)
    np.add.at(masses, mesh.tets.ravel(), np.repeat(density * vol / 4.0, 4))
    if mesh.n_tets and not (masses[np.unique(mesh.tets)] > 0.0).all():
        raise MeshError("non-positive lumped mass")
    return RestData(inv, vol, rows, masses)
