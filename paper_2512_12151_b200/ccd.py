"""Continuous collision detection (intact/ccd.py) on the GPU.

`CCD` is the device handle the stepper keeps per System (surface primitives
resident, LBVH scratch reused).  The module-level functions keep the
reference's numpy signatures for drop-in use and parity tests.
"""

from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from . import _lib
from .device import empty, to_dev, to_host
from .distance import PairKind

S_ACCD = 0.1
ACCD_MAX_ITERS = 100


@dataclasses.dataclass
class BlockingPairs:
    """Pairs whose TOI along the queried motion is below 1 (intact/ccd.py:148-165)."""

    kinds: np.ndarray
    indices: np.ndarray
    tois: np.ndarray

    @staticmethod
    def empty() -> "BlockingPairs":
        return BlockingPairs(np.empty(0, dtype=np.int64), np.empty((0, 4), dtype=np.int64), np.empty(0))

    def __len__(self):
        return len(self.tois)


class CCD:
    """Device handle over fixed surface primitives (tris, edges, verts)."""

    def __init__(self, tris, edges, verts):
        self.tris = np.ascontiguousarray(tris, dtype=np.int64).reshape(-1, 3)
        self.edges = np.ascontiguousarray(edges, dtype=np.int64).reshape(-1, 2)
        self.verts = np.ascontiguousarray(verts, dtype=np.int64).reshape(-1)
        h = C.c_void_p()
        _lib.check(_lib.lib().ibf_ccd_create(len(self.tris), _lib.host_ptr(self.tris), len(self.edges),
                                             _lib.host_ptr(self.edges), len(self.verts),
                                             _lib.host_ptr(self.verts), C.byref(h)), "ibf_ccd_create")
        self.handle = h
        self.n_blocking = 0

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h and _lib._lib is not None:
                _lib.lib().ibf_ccd_destroy(h)
                self.handle = None
        except (AttributeError, TypeError):
            pass  # interpreter shutdown: module globals already cleared

    def max_step_size(self, x_dev, x_hat_dev, min_gap, cap=1.0):
        """alpha on the host; blocking pairs stay on the device."""
        a = C.c_double()
        nb = C.c_int64()
        _lib.check(_lib.lib().ibf_max_step_size(self.handle, _lib.dev_ptr(x_dev), _lib.dev_ptr(x_hat_dev),
                                                float(min_gap), float(cap), C.byref(a), C.byref(nb),
                                                _lib.stream()), "ibf_max_step_size")
        self.n_blocking = int(nb.value)
        return float(a.value)

    def blocking(self) -> BlockingPairs:
        n = self.n_blocking
        k = np.empty(n, dtype=np.int64)
        q = np.empty((n, 4), dtype=np.int64)
        t = np.empty(n)
        if n:
            _lib.check(_lib.lib().ibf_ccd_get_blocking(self.handle, _lib.host_ptr(k), _lib.host_ptr(q),
                                                       _lib.host_ptr(t), _lib.stream()), "ibf_ccd_get_blocking")
        return BlockingPairs(k, q, t)

    def static_intersections(self, x_dev, cap: int = 1 << 16):
        """(n_hits, pairs (k,2)) of intersecting surface triangles at x
        (intact/intersect.py:125-140); pairs truncated to `cap`."""
        nh = C.c_int64()
        out = np.empty((max(cap, 1), 2), dtype=np.int64)
        _lib.check(_lib.lib().ibf_static_intersection(self.handle, _lib.dev_ptr(x_dev), C.byref(nh),
                                                      _lib.host_ptr(out), int(cap), _lib.stream()),
                   "ibf_static_intersection")
        k = min(int(nh.value), cap)
        return int(nh.value), out[:k]

    def min_distance(self, x_dev, radius):
        """(d, kind, quad) of the nearest non-adjacent VF/EE pair whose boxes
        come within `radius`; (inf, -1, None) without candidates."""
        d = C.c_double()
        pr = np.full(5, -1, dtype=np.int64)
        _lib.check(_lib.lib().ibf_min_distance(self.handle, _lib.dev_ptr(x_dev), float(radius), C.byref(d),
                                               _lib.host_ptr(pr), _lib.stream()), "ibf_min_distance")
        if pr[0] < 0:
            return float(d.value), -1, None
        return float(d.value), int(pr[0]), pr[1:].copy()

    def candidates(self, x0_dev, x1_dev, min_gap):
        nvf, nee = C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().ibf_ccd_candidates(self.handle, _lib.dev_ptr(x0_dev), _lib.dev_ptr(x1_dev),
                                                 float(min_gap), C.byref(nvf), C.byref(nee), _lib.stream()),
                   "ibf_ccd_candidates")
        vf = np.empty((nvf.value, 4), dtype=np.int64)
        ee = np.empty((nee.value, 4), dtype=np.int64)
        _lib.check(_lib.lib().ibf_ccd_get_candidates(self.handle, _lib.host_ptr(vf), _lib.host_ptr(ee),
                                                     _lib.stream()), "ibf_ccd_get_candidates")
        return vf, ee


def accd_batch(kind, x0, x1, min_gap):
    """Conservative TOI per pair (intact/ccd.py:37-91), bit-identical."""
    x0 = np.ascontiguousarray(x0, dtype=np.float64).reshape(-1, 4, 3)
    x1 = np.ascontiguousarray(x1, dtype=np.float64).reshape(-1, 4, 3)
    n = len(x0)
    if n == 0:
        return np.ones(0)
    a, b, t = to_dev(x0), to_dev(x1), empty((n,))
    _lib.check(_lib.lib().ibf_accd(int(kind), n, _lib.dev_ptr(a), _lib.dev_ptr(b), float(min_gap),
                                   _lib.dev_ptr(t), _lib.stream()), "ibf_accd")
    return to_host(t)


def accd_toi(kind, x0, x1, min_gap) -> float:
    return float(accd_batch(kind, np.asarray(x0, float)[None], np.asarray(x1, float)[None], min_gap)[0])


def candidate_pairs(x0, x1, tris, edges, verts, min_gap):
    """Broad phase (intact/ccd.py:113-145): same pair sets, ordered ascending."""
    ccd = CCD(tris, edges, verts)
    return ccd.candidates(to_dev(x0), to_dev(x1), min_gap)


def max_step_size(x, x_hat, tris, edges, verts, min_gap, cap: float = 1.0):
    """(alpha, BlockingPairs) — intact/ccd.py:168-193."""
    ccd = CCD(tris, edges, verts)
    alpha = ccd.max_step_size(to_dev(x), to_dev(x_hat), min_gap, cap)
    return alpha, ccd.blocking()


__all__ = ["BlockingPairs", "CCD", "PairKind", "S_ACCD", "ACCD_MAX_ITERS", "accd_batch", "accd_toi",
           "candidate_pairs", "max_step_size"]
