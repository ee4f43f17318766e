"""Oracle: Alg. 1 outer loop (one implicit step with CCD-clamped passes).

Restates `intact/stepper.py` (paths relative to /root/reference/pkg/src),
including the code's parity traps noted in SURVEY.md §0.1: the beta
recursion is called with k-1 (:320), the CCD gap is 0.1*offset (:35, :316),
mu is re-initialised every step from a contact-free assembly (:265-268), and
admissions use the previous pass's blocking pairs (:303).
Test infrastructure only — see oracle/__init__.py.
"""

from __future__ import annotations

import time

import numpy as np

from .contact import ConstraintSet
from .geometry import step_limit
from .material import inversion_cap
from .newton import assemble, subproblem

OUTER_CAP = 1024                    # intact/stepper.py:29
STALL_ALPHA = 1e-4                  # :31
STALL_LIMIT = 50                    # :32
GAP_FRACTION = 0.1                  # :35


class Aborted(RuntimeError):
    """`StepAbortError` (intact/stepper.py:167-175)."""

    def __init__(self, records):
        super().__init__("outer loop hit the iteration cap before beta reached epsilon")
        self.records = records


def beta_next(beta, alpha, k, k_min):
    """`beta_update` (:178-183)."""
    return (1.0 - alpha) * beta if k + 1 >= k_min else beta


def max_diag_entry(x, masses, regions, h, memo):
    """Largest scalar diagonal of the contact-free system at x
    (`stiffness_diagonal_max`, :191-200)."""
    if len(masses) == 0:
        return 1.0
    _, H = assemble(x, x, masses, regions, None, 1.0, 1.0, h, memo=memo)
    d = H.diag()
    return float(d[:, (0, 1, 2), (0, 1, 2)].max())


def clamp(x, x_hat, alpha):
    """`clamp_state` (:229-239): convex step, coinciding components bit-kept."""
    if alpha >= 1.0:
        return x_hat.copy()
    mixed = (1.0 - alpha) * x + alpha * x_hat
    return np.where(x == x_hat, x, mixed)


class Scene:
    """Plain-array system: masses, regions, surface prims, DBC
    (`System`, :103-128; `BoundaryCondition`, :78-100).

    boundary: list of (vertex ids, trajectory or None); trajectory(k) returns
    the (len(ids),3) targets for step k, None pins the vertices in place.
    """

    def __init__(self, masses, regions, tris, edges, verts, boundary=()):
        self.masses, self.regions = masses, regions
        self.tris, self.edges, self.verts = tris, edges, verts
        self.boundary = list(boundary)
        mask = np.zeros(len(masses), dtype=bool)
        for ids, _ in self.boundary:
            mask[ids] = True
        self.dbc = mask
        self.memo = {}


def step(x_t, v_t, scene, aset, h, offset, epsilon=1e-3, k_min=1, decay=0.9,
         c_mu=0.1, cg_tol=1e-4, gravity=(0.0, 0.0, -9.81), step_index=0,
         outer_cap=OUTER_CAP, record_iterates=False, trace=None, mu_f=0.0, eps_v=1e-3, friction=None,
         friction_out=None):
    """One step (`step`, :242-371).  `friction` holds the terms frozen at the
    end of the previous step; with mu_f > 0 the new terms are appended to the
    list `friction_out` (`friction_precompute`, :361-370).

    Returns (x, v, records, mu, offset) with one record per pass:
    (alpha, beta, n_constraints, newton_iters, cg_iters, wall_ms).
    `trace`, if a list, receives per pass the exact inputs and outputs of
    the set-maintenance and CCD stages (for identical-input parity tests).
    """
    g = np.asarray(gravity, dtype=float)
    x_tilde = x_t + h * v_t + (h * h) * g
    mu = c_mu * max_diag_entry(x_t, scene.masses, scene.regions, h, scene.memo)
    x = x_t.copy()
    x_hat = x_t.copy()
    for ids, traj in scene.boundary:
        x_hat[ids] = x_t[ids] if traj is None else np.asarray(traj(step_index), dtype=float)
    beta, stall = 1.0, 0
    kinds = np.zeros(0, dtype=np.int64)
    quads = np.zeros((0, 4), dtype=np.int64)
    tois = np.zeros(0)
    records, iterates = [], []
    done = False
    for k in range(outer_cap):
        t0 = time.perf_counter()
        x_hat, nit, cgit, _, _ = subproblem(
            x_tilde, x, x_hat, scene.masses, scene.regions, aset, mu, offset, h,
            cg_tol=cg_tol, decay=decay, dbc=scene.dbc, memo=scene.memo, friction=friction)
        if trace is not None:
            rec = {"resident": (aset.kind.copy(), aset.quad.copy(), aset.gamma.copy()),
                   "blocking": (kinds.copy(), quads.copy(), tois.copy())}
        aset.update(kinds, quads, tois)
        cap = 1.0
        for model, _m, _l, tets, rows, _v in scene.regions:
            cap = min(cap, inversion_cap(model, x, x_hat - x, tets, rows))
        alpha, kinds, quads, tois = step_limit(
            x, x_hat, scene.tris, scene.edges, scene.verts, GAP_FRACTION * offset, cap=cap)
        if trace is not None:
            rec.update(updated=(aset.kind.copy(), aset.quad.copy()), x=x.copy(), x_hat=x_hat.copy(),
                       min_gap=GAP_FRACTION * offset, cap=cap, alpha=alpha,
                       new_blocking=(kinds.copy(), quads.copy(), tois.copy()))
            trace.append(rec)
        x = clamp(x, x_hat, alpha)
        beta = beta_next(beta, alpha, k - 1, k_min)
        records.append((alpha, beta, len(aset), nit, cgit, (time.perf_counter() - t0) * 1e3))
        if record_iterates:
            iterates.append(x_hat.copy())
        stall = stall + 1 if alpha < STALL_ALPHA else 0
        if stall >= STALL_LIMIT:
            mu, offset, stall = 2.0 * mu, 0.5 * offset, 0
        if beta <= epsilon:
            done = True
            break
    if not done:
        raise Aborted(records)
    v = (x - x_t) / h
    if friction_out is not None and mu_f > 0.0:
        from .friction import precompute
        friction_out.append(precompute(x, aset, mu, offset, h, mu_f, eps_v))
    if record_iterates:
        return x, v, records, mu, offset, iterates
    return x, v, records, mu, offset


def run(x, v, scene, n_steps, **params):
    """Advance n_steps with one persistent active set (`Simulation.run`, :400-407)."""
    aset = ConstraintSet()
    out = []
    for k in range(n_steps):
        x, v, rec, _, _ = step(x, v, scene, aset, step_index=k, **params)
        out.append(rec)
    return x, v, out, aset
