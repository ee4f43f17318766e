"""Semi-implicit smoothed Coulomb friction (intact/friction.py) with the
frozen terms resident in HBM.

`friction_precompute` keeps the reference's signature and returns a
`FrictionTerms` whose arrays (indices, weights, frames, coeff, ref, eps —
the reference's dataclass fields) live in an `ibf_friction` handle and are
copied to the host only when read.  Terms enter the next step's assembly,
energy and SpMV matrix-free (csrc/friction.cu); `Simulation` threads them
from step to step like the reference (intact/stepper.py:361-396).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


class FrictionTerms:
    """Frozen per-contact friction data (intact/friction.py:56-73)."""

    def __init__(self):
        h = C.c_void_p()
        _lib.check(_lib.lib().ibf_friction_create(C.byref(h)), "ibf_friction_create")
        self.handle = h
        self._host = None

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h and _lib._lib is not None:
                _lib.lib().ibf_friction_destroy(h)
                self.handle = None
        except (AttributeError, TypeError):
            pass  # interpreter shutdown: module globals already cleared

    def __len__(self) -> int:
        return int(_lib.lib().ibf_friction_size(self.handle))

    @classmethod
    def from_arrays(cls, indices, weights, frames, coeff, ref, eps) -> "FrictionTerms":
        """Device copy of host terms (e.g. a reference FrictionTerms)."""
        ft = cls()
        q = np.ascontiguousarray(indices, dtype=np.int64).reshape(-1, 4)
        w = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1, 4)
        fr = np.ascontiguousarray(frames, dtype=np.float64).reshape(-1, 3, 2)
        cf = np.ascontiguousarray(coeff, dtype=np.float64).reshape(-1)
        rf = np.ascontiguousarray(ref, dtype=np.float64).reshape(-1, 3)
        _lib.check(_lib.lib().ibf_friction_import(ft.handle, len(cf), _lib.host_ptr(q), _lib.host_ptr(w),
                                                  _lib.host_ptr(fr), _lib.host_ptr(cf), _lib.host_ptr(rf),
                                                  float(eps), _lib.stream()), "ibf_friction_import")
        return ft

    def _export(self):
        if self._host is None:
            n = len(self)
            q = np.empty((n, 4), dtype=np.int64)
            w, fr = np.empty((n, 4)), np.empty((n, 3, 2))
            cf, rf = np.empty(n), np.empty((n, 3))
            eps = C.c_double()
            _lib.check(_lib.lib().ibf_friction_export(self.handle, _lib.host_ptr(q), _lib.host_ptr(w),
                                                      _lib.host_ptr(fr), _lib.host_ptr(cf), _lib.host_ptr(rf),
                                                      C.byref(eps), _lib.stream()), "ibf_friction_export")
            self._host = (q, w, fr, cf, rf, float(eps.value))
        return self._host

    indices = property(lambda self: self._export()[0])
    weights = property(lambda self: self._export()[1])
    frames = property(lambda self: self._export()[2])
    coeff = property(lambda self: self._export()[3])
    ref = property(lambda self: self._export()[4])
    eps = property(lambda self: self._export()[5])


def as_device(friction):
    """A FrictionTerms handle for any object with the reference's fields."""
    if friction is None or isinstance(friction, FrictionTerms):
        return friction
    return FrictionTerms.from_arrays(friction.indices, friction.weights, friction.frames, friction.coeff,
                                     friction.ref, friction.eps)


def friction_precompute(x, active_set, mu, offset, h, friction_coefficient, eps_v):
    """Friction anchors from a converged step (intact/friction.py:103-151);
    None when disabled or no contact carries a positive normal force."""
    from .device import to_dev
    if friction_coefficient <= 0.0 or len(active_set) == 0:
        return None
    xd = to_dev(x) if isinstance(x, np.ndarray) else x
    ft = FrictionTerms()
    n = C.c_int64()
    _lib.check(_lib.lib().ibf_friction_precompute(ft.handle, active_set.handle, _lib.dev_ptr(xd), float(mu),
                                                  float(offset), float(h), float(friction_coefficient),
                                                  float(eps_v), C.byref(n), _lib.stream()),
               "ibf_friction_precompute")
    return ft if n.value else None
