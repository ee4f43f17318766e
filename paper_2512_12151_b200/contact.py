"""Augmented-Lagrangian contact constraints (intact/contact.py) with a
device-resident active set.

`ActiveSet` keeps the reference's interface (len, iteration in insertion
order, membership by (kind, sorted ids), add, update, refresh_anchors,
batch, dual_update_sweep) over an `ibf_contacts` handle whose SoA lives in
HBM (csrc/contact.cu).  Iterating materialises `Constraint` copies for
inspection; mutating them does not write back (use `add`/`import_state`).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .ccd import CCD, BlockingPairs
from .distance import PairKind

GAMMA_PRUNE_THRESHOLD = 0.01


def constraint_key(kind, indices) -> tuple:
    return (int(kind), tuple(sorted(int(i) for i in indices)))


@dataclass
class Constraint:
    kind: PairKind
    indices: np.ndarray
    lam: float = 0.0
    gamma: float = 1.0
    s: float = 0.0
    anchor_d: float = 0.0
    anchor_grad: np.ndarray = field(default_factory=lambda: np.zeros((4, 3)))
    anchor_x: np.ndarray = field(default_factory=lambda: np.zeros((4, 3)))

    @property
    def key(self) -> tuple:
        return constraint_key(self.kind, self.indices)


@dataclass
class ConstraintBatch:
    """Host snapshot of the SoA (intact/contact.py:109-141)."""

    kinds: np.ndarray
    indices: np.ndarray
    lam: np.ndarray
    gamma: np.ndarray
    anchor_d: np.ndarray
    anchor_grad: np.ndarray
    anchor_x: np.ndarray

    def __len__(self) -> int:
        return len(self.kinds)


class ActiveSet:
    """Insertion-ordered constraint set in device memory."""

    def __init__(self, admit_all: bool = False):
        self.admit_all = admit_all
        self.handle = None
        self.n_verts = 0

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h and _lib._lib is not None:
                _lib.lib().ibf_contacts_destroy(h)
                self.handle = None
        except (AttributeError, TypeError):
            pass  # interpreter shutdown: module globals already cleared

    # -- handle management: the reference's ActiveSet() does not know N
    def ensure(self, n_verts: int):
        n_verts = max(int(n_verts), 1)
        if self.handle is not None and n_verts <= self.n_verts:
            return self.handle
        state = self.export_state() if self.handle is not None else None
        if self.handle is not None:
            _lib.lib().ibf_contacts_destroy(self.handle)
        h = C.c_void_p()
        _lib.check(_lib.lib().ibf_contacts_create(n_verts, 1 if self.admit_all else 0, C.byref(h)),
                   "ibf_contacts_create")
        self.handle, self.n_verts = h, n_verts
        if state is not None:
            self.import_state(*state)
        return self.handle

    def __len__(self) -> int:
        return int(_lib.lib().ibf_contacts_size(self.handle)) if self.handle is not None else 0

    def export_state(self):
        n = len(self)
        kind = np.empty(n, dtype=np.int64)
        quad = np.empty((n, 4), dtype=np.int64)
        lam, gamma, s, ad = (np.empty(n) for _ in range(4))
        ag, ax = np.empty((n, 4, 3)), np.empty((n, 4, 3))
        if n:
            _lib.check(_lib.lib().ibf_contacts_export(
                self.handle, *(_lib.host_ptr(a) for a in (kind, quad, lam, gamma, s, ad, ag, ax)),
                _lib.stream()), "ibf_contacts_export")
        return kind, quad, lam, gamma, s, ad, ag, ax

    def import_state(self, kind, quad, lam, gamma, s, ad, ag, ax):
        kind = np.ascontiguousarray(kind, dtype=np.int64)
        quad = np.ascontiguousarray(quad, dtype=np.int64).reshape(-1, 4)
        self.ensure(int(quad.max()) + 1 if quad.size else 1)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (lam, gamma, s, ad, ag, ax)]
        _lib.check(_lib.lib().ibf_contacts_import(
            self.handle, len(kind), _lib.host_ptr(kind), _lib.host_ptr(quad),
            *(_lib.host_ptr(a) for a in arrs), _lib.stream()), "ibf_contacts_import")

    def __iter__(self):
        kind, quad, lam, gamma, s, ad, ag, ax = self.export_state()
        for j in range(len(kind)):
            yield Constraint(PairKind(int(kind[j])), quad[j].copy(), float(lam[j]), float(gamma[j]), float(s[j]),
                             float(ad[j]), ag[j].copy(), ax[j].copy())

    def __contains__(self, key) -> bool:
        kind, quad = self.export_state()[:2]
        return any(constraint_key(k, q) == key for k, q in zip(kind, quad))

    def add(self, constraint: Constraint) -> bool:
        """Append unless the key is resident (intact/contact.py:172-177)."""
        if constraint.key in self:
            return False
        st = list(self.export_state())
        new = [np.array([int(constraint.kind)]), np.asarray(constraint.indices, dtype=np.int64)[None],
               np.array([constraint.lam]), np.array([constraint.gamma]), np.array([constraint.s]),
               np.array([constraint.anchor_d]), np.asarray(constraint.anchor_grad, dtype=float)[None],
               np.asarray(constraint.anchor_x, dtype=float)[None]]
        self.import_state(*[np.concatenate([a, b]) for a, b in zip(st, new)])
        return True

    def update(self, blocking) -> tuple[int, int]:
        """Dedup, earliest-TOI admission, prune (intact/contact.py:179-205).
        `blocking` is a BlockingPairs (host) or a CCD handle (device-resident
        blocking set of its last max_step_size)."""
        adm, pr = C.c_int64(), C.c_int64()
        if isinstance(blocking, CCD):
            self.ensure(self.n_verts)
            _lib.check(_lib.lib().ibf_contacts_update(self.handle, blocking.handle, C.byref(adm), C.byref(pr),
                                                      _lib.stream()), "ibf_contacts_update")
        else:
            b = blocking if blocking is not None else BlockingPairs.empty()
            k = np.ascontiguousarray(b.kinds, dtype=np.int64)
            q = np.ascontiguousarray(b.indices, dtype=np.int64).reshape(-1, 4)
            t = np.ascontiguousarray(b.tois, dtype=np.float64)
            self.ensure(max(self.n_verts, int(q.max()) + 1 if q.size else 1))
            _lib.check(_lib.lib().ibf_contacts_update_host(self.handle, len(k), _lib.host_ptr(k), _lib.host_ptr(q),
                                                           _lib.host_ptr(t), C.byref(adm), C.byref(pr),
                                                           _lib.stream()), "ibf_contacts_update")
        return int(adm.value), int(pr.value)

    def refresh_anchors(self, x) -> int:
        """Re-linearise at x (numpy (n,3) or device tensor); returns the
        degenerate count (intact/contact.py:207-235)."""
        from .device import to_dev
        xd = to_dev(x) if isinstance(x, np.ndarray) else x
        self.ensure(max(self.n_verts, xd.shape[0]))
        nd = C.c_int64()
        _lib.check(_lib.lib().ibf_contacts_refresh_anchors(self.handle, _lib.dev_ptr(xd), C.byref(nd),
                                                           _lib.stream()), "refresh_anchors")
        return int(nd.value)

    def batch(self) -> ConstraintBatch | None:
        if len(self) == 0:
            return None
        kind, quad, lam, gamma, _s, ad, ag, ax = self.export_state()
        return ConstraintBatch(kind, quad, lam, gamma, ad, ag, ax)

    def dual_update_sweep(self, x_hat, offset, mu, decay) -> float:
        from .device import to_dev
        if len(self) == 0:
            return 0.0
        xd = to_dev(x_hat) if isinstance(x_hat, np.ndarray) else x_hat
        w = C.c_double()
        _lib.check(_lib.lib().ibf_contacts_dual_sweep(self.handle, _lib.dev_ptr(xd), float(offset), float(mu),
                                                      float(decay), C.byref(w), _lib.stream()), "dual_update_sweep")
        return float(w.value)
