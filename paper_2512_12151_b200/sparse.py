"""Symmetric 3x3-block matrices and block-Jacobi PCG (intact/sparse.py) on the GPU.

`BlockSparseMatrix` keeps the reference's constructor (COO triplets,
duplicates coalesced in key order) and storage (diagonal + strict upper);
the blocks live on the device and `matvec` / `pcg_solve` run there
(csrc/pcg.cu).  numpy in, numpy out, so the reference's tests read the same.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import empty, to_dev, to_host

PCG_RESTART_INTERVAL = 250


def clique_contributions(vertex_ids, blocks):
    """Per-clique (M,k,k,3,3) grids -> upper-triangle COO triplets, transposing
    blocks whose global row > col (host-side index bookkeeping,
    intact/sparse.py:17-36)."""
    vertex_ids = np.asarray(vertex_ids)
    m, k = vertex_ids.shape
    li, lj = np.triu_indices(k)
    r = vertex_ids[:, li].ravel()
    c = vertex_ids[:, lj].ravel()
    v = np.asarray(blocks)[:, li, lj].reshape(-1, 3, 3)
    sw = r > c
    return (np.where(sw, c, r), np.where(sw, r, c),
            np.where(sw[:, None, None], v.transpose(0, 2, 1), v))


@dataclass
class PCGInfo:
    iterations: int
    converged: bool
    rel_residual: float


class BlockSparseMatrix:
    """Symmetric 3Nx3N matrix as coalesced 3x3 blocks, diagonal plus upper."""

    def __init__(self, n_vertices, rows, cols, blocks):
        rows = np.ascontiguousarray(rows, dtype=np.int64).ravel()
        cols = np.ascontiguousarray(cols, dtype=np.int64).ravel()
        blocks = np.ascontiguousarray(blocks, dtype=np.float64).reshape(-1, 3, 3)
        self.n_vertices = int(n_vertices)
        h = C.c_void_p()
        _lib.check(_lib.lib().ibf_bsr_create(self.n_vertices, len(rows), _lib.host_ptr(rows), _lib.host_ptr(cols),
                                             _lib.host_ptr(blocks), C.byref(h)), "BlockSparseMatrix")
        self.handle = h
        self._sync_host()

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h and _lib._lib is not None:
                _lib.lib().ibf_bsr_destroy(h)
                self.handle = None
        except (AttributeError, TypeError):
            pass  # interpreter shutdown: module globals already cleared

    def _sync_host(self):
        nb = int(_lib.lib().ibf_bsr_size(self.handle))
        self.rows = np.empty(nb, dtype=np.int64)
        self.cols = np.empty(nb, dtype=np.int64)
        self.blocks = np.empty((nb, 3, 3))
        _lib.check(_lib.lib().ibf_bsr_export(self.handle, _lib.host_ptr(self.rows), _lib.host_ptr(self.cols),
                                             _lib.host_ptr(self.blocks), _lib.stream()), "ibf_bsr_export")
        self._off = self.rows != self.cols

    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(self.n_vertices, 3)
        xd, yd = to_dev(x), empty((self.n_vertices, 3))
        _lib.check(_lib.lib().ibf_bsr_matvec(self.handle, _lib.dev_ptr(xd), _lib.dev_ptr(yd), _lib.stream()),
                   "matvec")
        return to_host(yd)

    def diagonal_blocks(self):
        diag = np.zeros((self.n_vertices, 3, 3))
        on = ~self._off
        diag[self.rows[on]] = self.blocks[on]
        return diag

    def mask_dirichlet(self, vertex_mask, diag_replacement):
        m = np.ascontiguousarray(vertex_mask, dtype=np.uint8)
        d = np.ascontiguousarray(diag_replacement, dtype=np.float64).reshape(self.n_vertices, 3, 3)
        _lib.check(_lib.lib().ibf_bsr_mask_dirichlet(self.handle, _lib.host_ptr(m), _lib.host_ptr(d),
                                                     _lib.stream()), "mask_dirichlet")
        self._sync_host()

    def to_dense(self):
        n = self.n_vertices * 3
        dense = np.zeros((n, n))
        for r, c, b in zip(self.rows, self.cols, self.blocks):
            dense[3 * r:3 * r + 3, 3 * c:3 * c + 3] += b
            if r != c:
                dense[3 * c:3 * c + 3, 3 * r:3 * r + 3] += b.T
        return dense


def pcg_solve(matrix: BlockSparseMatrix, rhs, rel_tol, max_iters=None):
    """Block-Jacobi PCG (intact/sparse.py:99-150) as one persistent kernel.
    `matrix` is a BlockSparseMatrix or the AssembledMatrix that `assemble`
    returns (solved on its device operator, contacts matrix-free)."""
    fast = getattr(matrix, "pcg", None)
    if fast is not None:
        out = fast(rhs, rel_tol, max_iters)
        if out is not None:
            p, its, conv, rel = out
            return p, PCGInfo(its, conv, rel)
    rhs = np.ascontiguousarray(rhs, dtype=np.float64).reshape(matrix.n_vertices, 3)
    bd, xd = to_dev(rhs), empty((matrix.n_vertices, 3))
    info = np.zeros(3)
    _lib.check(_lib.lib().ibf_bsr_pcg(matrix.handle, _lib.dev_ptr(bd), _lib.dev_ptr(xd), float(rel_tol),
                                      int(max_iters) if max_iters else 0, _lib.host_ptr(info), _lib.stream()),
               "pcg_solve")
    return to_host(xd), PCGInfo(int(info[0]), bool(info[1]), float(info[2]))
