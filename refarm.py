"""CPU arm of the benchmark: the UNMODIFIED reference (`intact`, installed
into baseline/_ref by `pip install --no-deps --target baseline/_ref`, see
DESIGN.md §(d)) timed stage by stage through its own public functions.

Used only by bench.py (`--impl reference` and the `cpu_baseline` leg of the
GPU arm).  Nothing of this repo's engine runs inside a timed region here:
the device path only produces the input state (the press-window state the
GPU arm's timed frames start from), which is then handed to the reference
as numpy arrays and reference objects.

One Newton iteration of the reference's path (intact/stepper.py:242-371,
intact/solver.py:178-233) is split into the stages it calls:

  stiffness   stiffness_diagonal_max — one full assembly per frame (:191-200)
  refresh     ActiveSet.refresh_anchors + batch — once per outer pass
  assemble    solver.assemble with the constraint batch — per Newton iteration
  cg_iter     sparse.pcg_solve, per CG iteration (timed over a few)
  energy      solver.incremental_energy — per line-search evaluation
  ccd         ccd.max_step_size — once per outer pass
  update      ActiveSet.update + dual_update_sweep — once per outer pass

A frame of the reference then costs
  stiffness + passes x (refresh + ccd + update) + newton x assemble
  + cg x cg_iter + energy_evals x energy
with the per-frame operation counts of the GPU arm on the same frames (its
Newton / CG / pass counts, and the energy evaluations the reference's
sequential line search makes for those iterations, ibf_system_counts).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(ROOT, "baseline", "_ref")


def intact():
    """The installed reference package, or None when baseline/_ref is absent."""
    if not os.path.isdir(os.path.join(REF, "intact")):
        return None
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import intact as I
    import intact.ccd
    import intact.contact
    import intact.distance
    import intact.elasticity
    import intact.solver
    import intact.sparse
    import intact.stepper
    return I


def reference_system(I, system, regions_subset=None):
    """The reference's System for this repo's (drop-in) System."""
    E = I.elasticity
    regs = system.regions if regions_subset is None else [system.regions[k] for k in regions_subset]
    regions = [I.solver.ElasticRegion(E.Material(E.MaterialModel(r.material.model.value), r.material.young,
                                                 r.material.poisson), r.tets, r.shape_rows, r.volumes)
               for r in regs]
    bcs = [I.stepper.BoundaryCondition(bc.vertices, bc.kind, bc.trajectory) for bc in system.boundary]
    return I.stepper.System(system.masses, regions, system.surface_triangles, system.surface_edges,
                            system.surface_vertices, bcs)


def reference_active_set(I, state):
    """ActiveSet holding the exported device constraints (insertion order kept)."""
    kind, quad, lam, gamma, s, ad, ag, ax = state
    A = I.contact.ActiveSet()
    PK = I.distance.PairKind
    for k in range(len(kind)):
        A.add(I.contact.Constraint(PK(int(kind[k])), quad[k].copy(), float(lam[k]), float(gamma[k]), float(s[k]),
                                   float(ad[k]), ag[k].copy(), ax[k].copy()))
    return A


def time_stages(I, rsys, x, v, aset_state, params, step_index, cg_iters=3, log=None):
    """Wall time (s) of each reference stage at the state (x, v, active set).

    The Newton iterate is the reference's own: x_hat0 with the Dirichlet
    targets, one assembly, cg_iters CG iterations, the energy at the trial
    point, one CCD pass over that motion, then the set update and dual sweep.
    """
    S = I.solver
    h = params.h
    out = {}

    def tick(name, fn):
        t = time.perf_counter()
        r = fn()
        out[name] = time.perf_counter() - t
        if log:
            log(f"[reference] {name}: {out[name]:.2f} s")
        return r

    x = np.ascontiguousarray(x)
    x_tilde = x + h * v + (h * h) * np.asarray(params.gravity, dtype=float)
    mu = tick("stiffness", lambda: I.stepper.mu_init(
        I.stepper.stiffness_diagonal_max(x, rsys.masses, rsys.regions, h), params.stiffness_constant))
    x_hat = x.copy()
    I.stepper.apply_dbc(x_hat, rsys.boundary, x, step_index)
    aset = reference_active_set(I, aset_state) if aset_state is not None else I.contact.ActiveSet()
    out["constraints"] = len(aset)

    def refresh():
        aset.refresh_anchors(x)
        return aset.batch()

    batch = tick("refresh", refresh)
    grad, H = tick("assemble", lambda: S.assemble(x_hat, x_tilde, rsys.masses, rsys.regions, batch, mu,
                                                  params.offset, h, rsys.dbc_mask))
    # per CG iteration: the difference of a 1-iteration and a (1 + cg_iters)-
    # iteration solve, so the per-solve setup (the block-Jacobi inverses)
    # is not charged to the iterations
    t = time.perf_counter()
    _, info1 = I.sparse.pcg_solve(H, -grad, params.cg_tol, max_iters=1)
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    p, info = I.sparse.pcg_solve(H, -grad, params.cg_tol, max_iters=1 + cg_iters)
    t2 = time.perf_counter() - t
    k = max(info.iterations - info1.iterations, 1)
    out["cg_iter"] = max(t2 - t1, 0.0) / k
    out["cg_setup"] = max(t1 - out["cg_iter"], 0.0)
    out["cg_iters_timed"] = int(info.iterations)
    if log:
        log(f"[reference] cg_iter: {out['cg_iter']:.3f} s (+ {out['cg_setup']:.3f} s setup per solve)")
    trial = x_hat + p
    tick("energy", lambda: S.incremental_energy(trial, x_tilde, rsys.masses, rsys.regions, batch, mu,
                                                params.offset, h))
    alpha, blocking = tick("ccd", lambda: I.ccd.max_step_size(x, trial, rsys.surface_triangles,
                                                               rsys.surface_edges, rsys.surface_vertices,
                                                               I.stepper.CCD_GAP_FRACTION * params.offset))
    out["blocking"] = len(blocking.tois)

    def update():
        aset.dual_update_sweep(trial, params.offset, mu, params.decay)
        return aset.update(blocking)

    tick("update", update)
    return out


def frame_ms(stages, counts):
    """Reference ms per frame from stage times (s) and per-frame op counts."""
    parts = {
        "stiffness_ms": 1e3 * stages["stiffness"],
        "refresh_ms": 1e3 * stages["refresh"] * counts["passes"],
        "assemble_ms": 1e3 * stages["assemble"] * counts["newton"],
        "pcg_ms": 1e3 * (stages["cg_iter"] * counts["cg"] + stages["cg_setup"] * counts["newton"]),
        "energy_ms": 1e3 * stages["energy"] * counts["energy_evals"],
        "ccd_ms": 1e3 * stages["ccd"] * counts["passes"],
        "update_ms": 1e3 * stages["update"] * counts["passes"],
    }
    return float(sum(parts.values())), parts
