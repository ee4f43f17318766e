"""AL subproblem solver (intact/solver.py) on the GPU.

`DeviceSystem` owns an `ibf_system` handle: the static symmetric BSR pattern
of mass + elasticity, gather maps, workspaces.  `solve_subproblem` is the
reference's Newton loop, executed by libibf's native loop
(ibf_solve_subproblem, csrc/newton.cu) with one host sync per iteration.
The numpy-signature functions (`assemble`, `incremental_energy`,
`solve_subproblem`) keep the reference's arguments; the device system they
need is built once per (masses, regions, dbc_mask) and cached.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .contact import ActiveSet, ConstraintBatch
from .device import empty, to_dev, to_host
from .elasticity import Material, MaterialModel

NEWTON_CAP = 64
LINE_SEARCH_MAX_HALVINGS = 30


class NonFiniteEnergyError(RuntimeError):
    """Assembly saw a non-finite elastic energy (intact/solver.py:35-37)."""


@dataclass(frozen=True)
class ElasticRegion:
    """A material-homogeneous group of tets addressing global vertex ids."""

    material: Material
    tets: np.ndarray
    shape_rows: np.ndarray
    volumes: np.ndarray


@dataclass
class SubproblemResult:
    x_hat: np.ndarray
    newton_iters: int
    cg_iters: int
    stalled: bool
    worst_violation: float


class DeviceSystem:
    """Device-resident elastic system (masses, regions, DBC mask)."""

    def __init__(self, masses, regions, dbc_mask=None):
        self._friction = None
        self._assembly_serial = 0
        masses = np.ascontiguousarray(masses, dtype=np.float64)
        n = len(masses)
        self.n = n
        self.regions = list(regions)
        models = np.array([_lib.MODELS[MaterialModel(r.material.model).value] for r in regions], dtype=np.int32)
        mus = np.array([r.material.mu for r in regions], dtype=np.float64)
        lams = np.array([r.material.lam for r in regions], dtype=np.float64)
        counts = np.array([len(r.tets) for r in regions], dtype=np.int64)
        tets = (np.concatenate([np.asarray(r.tets, dtype=np.int64).reshape(-1, 4) for r in regions])
                if regions else np.zeros((0, 4), dtype=np.int64))
        rows = (np.concatenate([np.asarray(r.shape_rows, dtype=np.float64).reshape(-1, 4, 3) for r in regions])
                if regions else np.zeros((0, 4, 3)))
        vols = (np.concatenate([np.asarray(r.volumes, dtype=np.float64).reshape(-1) for r in regions])
                if regions else np.zeros(0))
        dbc = np.zeros(n, dtype=np.uint8) if dbc_mask is None else np.ascontiguousarray(dbc_mask, dtype=np.uint8)
        self.has_nh = any(MaterialModel(r.material.model) == MaterialModel.NH and len(r.tets) for r in regions)
        h = C.c_void_p()
        _lib.check(_lib.lib().ibf_system_create(
            n, _lib.host_ptr(masses), _lib.host_ptr(dbc), len(regions), _lib.host_ptr(models), _lib.host_ptr(mus),
            _lib.host_ptr(lams), _lib.host_ptr(counts), _lib.host_ptr(np.ascontiguousarray(tets)),
            _lib.host_ptr(np.ascontiguousarray(rows)), _lib.host_ptr(np.ascontiguousarray(vols)), C.byref(h)),
            "ibf_system_create")
        self.handle = h
        self.n_tets = len(tets)
        nb, nl = C.c_int64(), C.c_int64()
        _lib.lib().ibf_system_pattern(h, C.byref(nb), C.byref(nl))
        self.n_blocks, self.n_upper = int(nb.value), int(nl.value)

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h and _lib._lib is not None:
                _lib.lib().ibf_system_destroy(h)
                self.handle = None
        except (AttributeError, TypeError):
            pass  # interpreter shutdown: module globals already cleared

    # ---- device-tensor entry points (used by the stepper)
    def solve_subproblem(self, aset: ActiveSet | None, x_tilde, x, x_hat, mu, offset, h, cg_tol, decay):
        self._assembly_serial += 1          # the native loop re-assembles
        res = np.zeros(4)
        ch = aset.ensure(self.n) if aset is not None else None
        _lib.check(_lib.lib().ibf_solve_subproblem(self.handle, ch, _lib.dev_ptr(x_tilde), _lib.dev_ptr(x),
                                                   _lib.dev_ptr(x_hat), float(mu), float(offset), float(h),
                                                   float(cg_tol), float(decay), _lib.host_ptr(res), _lib.stream()),
                   "solve_subproblem")
        return int(res[0]), int(res[1]), bool(res[2]), float(res[3])

    def set_dist(self, partition):
        """Row-partition this system's PCG solves over `partition`
        (dist.Partition; None: the single-GPU kernel again).  Keeps a
        reference so the communicator outlives the system's use of it."""
        self._dist = partition
        _lib.check(_lib.lib().ibf_system_set_dist(self.handle, partition.handle if partition is not None else None),
                   "ibf_system_set_dist")

    def set_friction(self, friction):
        """Frozen friction terms for the following assemble / energy / solve
        calls (None removes them); keeps a reference to the handle."""
        from .friction import as_device
        self._assembly_serial += 1          # the operator's friction part changes
        self._friction = as_device(friction)
        h = self._friction.handle if self._friction is not None and len(self._friction) else None
        _lib.check(_lib.lib().ibf_system_set_friction(self.handle, h), "ibf_system_set_friction")

    def stiffness_diagonal_max(self, x, h) -> float:
        out = C.c_double()
        _lib.check(_lib.lib().ibf_stiffness_diagonal_max(self.handle, _lib.dev_ptr(x), float(h), C.byref(out),
                                                         _lib.stream()), "stiffness_diagonal_max")
        return float(out.value)

    def inversion_safe_step(self, x, p) -> float:
        out = C.c_double()
        _lib.check(_lib.lib().ibf_inversion_safe_step(self.handle, _lib.dev_ptr(x), _lib.dev_ptr(p), C.byref(out),
                                                      _lib.stream()), "inversion_safe_step")
        return float(out.value)

    def assemble(self, aset, x_hat, x_tilde, mu, offset, h, apply_dbc, grad_out):
        self._assembly_serial += 1
        ch = aset.ensure(self.n) if (aset is not None and len(aset)) else None
        _lib.check(_lib.lib().ibf_assemble(self.handle, ch, _lib.dev_ptr(x_hat), _lib.dev_ptr(x_tilde), float(mu),
                                           float(offset), float(h), 1 if apply_dbc else 0, _lib.dev_ptr(grad_out),
                                           _lib.stream()), "assemble")

    def energy(self, aset, x_hat, x_tilde, mu, offset, h, p=None, rs=(1.0,)) -> np.ndarray:
        rs = np.ascontiguousarray(rs, dtype=np.float64)
        out = np.zeros(max(len(rs), 1))
        ch = aset.ensure(self.n) if (aset is not None and len(aset)) else None
        _lib.check(_lib.lib().ibf_incremental_energy(self.handle, ch, _lib.dev_ptr(x_hat), _lib.dev_ptr(p),
                                                     len(rs), _lib.host_ptr(rs), _lib.dev_ptr(x_tilde), float(mu),
                                                     float(offset), float(h), _lib.host_ptr(out), _lib.stream()),
                   "incremental_energy")
        return out

    def matvec(self, x, y):
        _lib.check(_lib.lib().ibf_system_matvec(self.handle, _lib.dev_ptr(x), _lib.dev_ptr(y), _lib.stream()),
                   "matvec")

    def pcg(self, rhs, x_out, rel_tol, max_iters=0):
        info = np.zeros(3)
        _lib.check(_lib.lib().ibf_system_pcg(self.handle, _lib.dev_ptr(rhs), _lib.dev_ptr(x_out), float(rel_tol),
                                             int(max_iters), _lib.host_ptr(info), _lib.stream()), "pcg")
        return int(info[0]), bool(info[1]), float(info[2])

    def export_bsr(self):
        rows = np.empty(self.n_blocks, dtype=np.int64)
        cols = np.empty(self.n_blocks, dtype=np.int64)
        blocks = np.empty((self.n_blocks, 3, 3))
        _lib.check(_lib.lib().ibf_system_export_bsr(self.handle, _lib.host_ptr(rows), _lib.host_ptr(cols),
                                                    _lib.host_ptr(blocks), _lib.stream()), "export_bsr")
        return rows, cols, blocks

    def export_terms(self):
        """Explicit upper cliques (rows, cols, blocks (k,3,3)) of the contact
        and friction terms of the last assembly, unmasked and uncoalesced."""
        nb = C.c_int64()
        _lib.check(_lib.lib().ibf_system_export_terms(self.handle, C.byref(nb), None, None, None, _lib.stream()),
                   "export_terms")
        rows = np.empty(nb.value, dtype=np.int64)
        cols = np.empty(nb.value, dtype=np.int64)
        blocks = np.empty((nb.value, 3, 3))
        if nb.value:
            _lib.check(_lib.lib().ibf_system_export_terms(self.handle, C.byref(nb), _lib.host_ptr(rows),
                                                          _lib.host_ptr(cols), _lib.host_ptr(blocks), _lib.stream()),
                       "export_terms")
        return rows, cols, blocks

    def spmv_bytes(self) -> float:
        b = C.c_double()
        _lib.lib().ibf_system_spmv_stats(self.handle, C.byref(b))
        return float(b.value)


_CACHE: dict = {}


def device_system(masses, regions, dbc_mask=None) -> DeviceSystem:
    """Cached DeviceSystem for a (masses, regions, dbc_mask) triple."""
    key = (id(masses), tuple(id(r.tets) for r in regions),
           None if dbc_mask is None else hash(np.asarray(dbc_mask, dtype=bool).tobytes()))
    hit = _CACHE.get(key)
    if hit is None or hit[1] is not masses:
        if len(_CACHE) > 8:
            _CACHE.clear()
        hit = (DeviceSystem(masses, regions, dbc_mask), masses, list(regions))
        _CACHE[key] = hit
    return hit[0]


def _batch_set(batch: ConstraintBatch | None, n):
    if batch is None or len(batch) == 0:
        return None
    aset = ActiveSet()
    aset.ensure(n)
    aset.import_state(batch.kinds, batch.indices, batch.lam, batch.gamma, np.zeros(len(batch)), batch.anchor_d,
                      batch.anchor_grad, batch.anchor_x)
    return aset


class AssembledMatrix:
    """H of `assemble`: the reference's BlockSparseMatrix (intact/sparse.py:46-96)
    as returned by intact/solver.py:109-156 — mass + h^2 PSD elasticity +
    mu*gamma grad_d grad_d^T contact cliques + friction cliques, DBC-masked.

    The elastic part is the device system's BSR; the contact and friction
    parts stay matrix-free on the device.  `matvec` and `pcg_solve(H, ...)`
    run on that device operator.  `rows` / `cols` / `blocks`,
    `diagonal_blocks()` and `to_dense()` see the explicit matrix: the term
    cliques are exported by the device (ibf_system_export_terms), masked like
    the reference masks them, and coalesced with the elastic blocks into a
    standalone `BlockSparseMatrix` on first use.  After `mask_dirichlet` the
    explicit matrix is authoritative for every operation.

    The device operator is that of the owning system's LAST assembly: a later
    `assemble` on the same system makes earlier matrices stale (reading one
    raises)."""

    def __init__(self, dev: DeviceSystem, keep, dbc_mask, serial):
        self.dev, self._keep, self._serial = dev, keep, serial
        self.n_vertices = dev.n
        self._dbc = None if dbc_mask is None or not np.any(dbc_mask) else np.asarray(dbc_mask, dtype=bool)
        self._explicit = None
        self._detached = False

    def _live(self):
        if self.dev._assembly_serial != self._serial:
            raise RuntimeError("stale AssembledMatrix: its DeviceSystem was assembled again")

    def explicit(self):
        """The explicit BlockSparseMatrix (built once, on first use)."""
        if self._explicit is None:
            from .sparse import BlockSparseMatrix
            self._live()
            rows, cols, blocks = self.dev.export_bsr()
            tr, tc, tb = self.dev.export_terms()
            if self._dbc is not None and len(tr):
                # intact/sparse.py:81-87 zeroes (and keeps) every block touching a
                # masked vertex; the masked diagonals are already mass * I
                tb = tb.copy()
                tb[self._dbc[tr] | self._dbc[tc]] = 0.0
            self._explicit = BlockSparseMatrix(self.n_vertices, np.concatenate([rows, tr]),
                                               np.concatenate([cols, tc]), np.concatenate([blocks, tb]))
        return self._explicit

    rows = property(lambda self: self.explicit().rows)
    cols = property(lambda self: self.explicit().cols)
    blocks = property(lambda self: self.explicit().blocks)

    @property
    def handle(self):
        return self.explicit().handle

    def diagonal_blocks(self):
        return self.explicit().diagonal_blocks()

    def mask_dirichlet(self, vertex_mask, diag_replacement):
        self.explicit().mask_dirichlet(vertex_mask, diag_replacement)
        self._detached = True

    def matvec(self, x):
        if self._detached:
            return self._explicit.matvec(x)
        self._live()
        xd, yd = to_dev(np.asarray(x, dtype=np.float64).reshape(self.n_vertices, 3)), empty((self.n_vertices, 3))
        self.dev.matvec(xd, yd)
        return to_host(yd)

    def pcg(self, rhs, rel_tol, max_iters=None):
        """Block-Jacobi PCG on the device operator (pcg_solve's fast path);
        None once mask_dirichlet detached the explicit matrix."""
        if self._detached:
            return None
        self._live()
        bd, xd = to_dev(np.asarray(rhs, dtype=np.float64).reshape(self.n_vertices, 3)), empty((self.n_vertices, 3))
        its, conv, rel = self.dev.pcg(bd, xd, rel_tol, int(max_iters) if max_iters else 0)
        return to_host(xd), its, conv, rel

    def to_dense(self):
        return self.explicit().to_dense()


def assemble(x_hat, x_tilde, masses, regions, batch, mu, offset, h, dbc_mask=None, friction=None):
    """(grad (n,3), H) of the AL objective at x_hat (intact/solver.py:109-156).
    H keeps the friction terms it was assembled with (matrix-free)."""
    dev = device_system(masses, regions, dbc_mask)
    aset = _batch_set(batch, dev.n)
    xd, xt = to_dev(x_hat), to_dev(x_tilde)
    g = empty((dev.n, 3))
    dev.set_friction(friction)
    dev.assemble(aset, xd, xt, mu, offset, h, dbc_mask is not None and np.any(dbc_mask), g)
    return to_host(g), AssembledMatrix(dev, (aset, dev._friction), dbc_mask, dev._assembly_serial)


def incremental_energy(x_hat, x_tilde, masses, regions, batch, mu, offset, h, friction=None) -> float:
    """L(x_hat) (intact/solver.py:88-106)."""
    dev = device_system(masses, regions, None)
    aset = _batch_set(batch, dev.n)
    dev.set_friction(friction)
    try:
        return float(dev.energy(aset, to_dev(x_hat), to_dev(x_tilde), mu, offset, h)[0])
    finally:
        dev.set_friction(None)


def line_search(x_hat, p, energy_fn, safe_cap: float = 1.0) -> tuple[float, bool]:
    """Largest r in {cap, cap/2, ...} with strict decrease (intact/solver.py:159-175).
    Generic host control logic over an arbitrary energy callable."""
    base = energy_fn(x_hat)
    r = min(1.0, safe_cap)
    best_r, best_e = r, np.inf
    for _ in range(LINE_SEARCH_MAX_HALVINGS + 1):
        e = energy_fn(x_hat + r * p)
        if e < base:
            return r, False
        if e < best_e:
            best_r, best_e = r, e
        r *= 0.5
    return best_r, True


def solve_subproblem(x_tilde, x, x_hat0, masses, regions, active_set: ActiveSet, mu, offset, h, cg_tol=1e-4,
                     decay=0.9, dbc_mask=None, friction=None) -> SubproblemResult:
    """Newton loop (cap 64, exit on full step) plus one dual sweep
    (intact/solver.py:178-233), run by libibf on the device."""
    dev = device_system(masses, regions, dbc_mask)
    xt, xd, xh = to_dev(x_tilde), to_dev(x), to_dev(x_hat0)
    dev.set_friction(friction)
    try:
        nit, cgit, stalled, worst = dev.solve_subproblem(active_set, xt, xd, xh, mu, offset, h, cg_tol, decay)
    finally:
        dev.set_friction(None)
    return SubproblemResult(to_host(xh), nit, cgit, stalled, worst)
