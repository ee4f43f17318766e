"""Pair distances (intact/distance.py) — numpy in, numpy out, computed on the GPU.

Same names, shapes and conventions as the reference: pts (n,4,3) stacked as
(vertex, tri0, tri1, tri2) or (a0, a1, b0, b1); returns d (n,), grad (n,12),
signed weights (n,4), degenerate (n,) bool.  Bit-identical to the reference
(csrc/geometry.cuh).
"""

from __future__ import annotations

import dataclasses
from enum import IntEnum

import numpy as np

from . import _lib
from .device import empty, to_dev, to_host, torch


class PairKind(IntEnum):
    VERTEX_FACE = 0
    EDGE_EDGE = 1


@dataclasses.dataclass
class DistanceEval:
    d: float
    grad: np.ndarray
    weights: np.ndarray
    degenerate: bool


def _eval(kind, pts):
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 4, 3)
    n = len(pts)
    if n == 0:
        return np.zeros(0), np.zeros((0, 12)), np.zeros((0, 4)), np.zeros(0, dtype=bool)
    P = to_dev(pts)
    d, g, w = empty((n,)), empty((n, 12)), empty((n, 4))
    dg = empty((n,), dtype=torch().uint8)
    _lib.check(_lib.lib().ibf_pair_eval(int(kind), n, _lib.dev_ptr(P), _lib.dev_ptr(d), _lib.dev_ptr(g),
                                        _lib.dev_ptr(w), _lib.dev_ptr(dg), _lib.stream()), "ibf_pair_eval")
    return to_host(d), to_host(g), to_host(w), to_host(dg).astype(bool)


def vf_eval(pts):
    return _eval(PairKind.VERTEX_FACE, pts)


def ee_eval(pts):
    return _eval(PairKind.EDGE_EDGE, pts)


def pair_distances(kind, pts):
    return _eval(kind, pts)[0]


def unsigned_distance(kind, p0, p1, p2, p3) -> DistanceEval:
    d, g, w, dg = _eval(kind, np.asarray([p0, p1, p2, p3], dtype=np.float64)[None])
    return DistanceEval(float(d[0]), g[0], w[0], bool(dg[0]))
