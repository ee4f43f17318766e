"""CPU baseline: the oracle's hot-path stages timed on bounded samples of a
scene — TEST/BENCH INFRASTRUCTURE ONLY (see oracle/__init__.py).

Used by bench.py's `cpu_baseline` leg (on the press-window state the GPU arm
just timed) and by `bench.py --impl reference` (on the scene's first frame,
without the GPU).  Nothing here is on the product path.

The reference is single-threaded numpy; a frame of the
C4 scene costs it hours (~90 s per elastic assembly, ~1.2 s per CG iteration,
~100 s per CCD pass at 2.3M tets / 1.6M surface triangles, measured in the
build container).  A frame is therefore not timed whole.  Instead each
sample times, at the scene's own state and resolution:

  elastic stages on a contiguous slice of one ball's tets:
    assemble   oracle.newton.assemble        (intact/solver.py:109-156)
    cg_iter    oracle.blocksparse.pcg, per CG iteration (intact/sparse.py:99-150)
    energy     oracle.newton.energy          (intact/solver.py:88-106)
  the CCD pass over that slice's surface     (intact/ccd.py:168-193)
  contact stages on the FULL active set (no scaling):
    contact assembly / energy terms, refresh_anchors, dual sweep, update
                                             (intact/contact.py:144-261)

and scales the slice stages to the whole scene by their own size measure
(tets, stored blocks, surface triangles).  ms/frame then multiplies the
stage times by per-frame operation counts (Newton iterations, CG iterations,
energy evaluations of the reference's sequential line search, outer passes)
— the one extrapolation, reported beside the measured stage times.
"""

from __future__ import annotations

import time

import numpy as np

from . import blocksparse, contact, geometry, newton


def oracle_regions(system, only=None):
    """Oracle region tuples of the system's ElasticRegions (all, or `only`)."""
    regs = system.regions if only is None else [system.regions[k] for k in only]
    return [(r.material.model.value, r.material.mu, r.material.lam, r.tets, r.shape_rows, r.volumes) for r in regs]


def ball_slices(system, n_slices):
    """(region index, lo, hi) tet ranges: the largest region (a ball) cut into
    n_slices contiguous slices."""
    k = int(np.argmax([len(r.tets) for r in system.regions]))
    m = len(system.regions[k].tets)
    edges = np.linspace(0, m, n_slices + 1).astype(np.int64)
    return [(k, int(edges[j]), int(edges[j + 1])) for j in range(n_slices)]


def _sub_system(system, k, lo, hi, *arrays):
    """The slice as a compact system: its tets renumbered over the vertices
    they use, the masses and the given (N,3) arrays restricted to those
    vertices, and the surface primitives lying entirely inside the slice."""
    r = system.regions[k]
    used, tets = np.unique(r.tets[lo:hi], return_inverse=True)
    tets = tets.reshape(-1, 4)
    remap = np.full(len(system.masses), -1, dtype=np.int64)
    remap[used] = np.arange(len(used))

    def prims(a):
        a = remap[a]
        return a[(a >= 0).all(axis=1)] if a.ndim == 2 else a[a >= 0]

    reg = (r.material.model.value, r.material.mu, r.material.lam, tets, r.shape_rows[lo:hi], r.volumes[lo:hi])
    surf = (prims(system.surface_triangles), prims(system.surface_edges), prims(system.surface_vertices))
    return reg, system.masses[used], surf, [np.ascontiguousarray(a[used]) for a in arrays]


def constraint_set(state):
    """oracle ConstraintSet holding an exported device active set (insertion order kept)."""
    kind, quad, lam, gamma, s, ad, ag, ax = state
    o = contact.ConstraintSet()
    if len(kind):
        o._append(np.asarray(kind, dtype=np.int64), np.asarray(quad, dtype=np.int64),
                  [contact.key_of(a, b) for a, b in zip(kind, quad)], lam=lam.copy(), gamma=gamma.copy(),
                  s=s.copy(), anchor_d=ad.copy(), anchor_grad=ag.copy(), anchor_x=ax.copy())
    return o


def time_sample(system, x, x_hat, x_tilde, mu, offset, h, slice_, aset_state=None, cg_iters=3,
                full_blocks=None, contacts=True):
    """Stage times (s) of one bounded sample, and the whole-scene stage times
    they scale to.  `slice_` = (region, lo, hi); `aset_state` = exported
    active set (None: no constraints); full_blocks = stored blocks (diagonal +
    strict upper) of the whole scene's matrix."""
    k, lo, hi = slice_
    reg, masses, (tris, edges, verts), (xs, xhs, xts) = _sub_system(system, k, lo, hi, x, x_hat, x_tilde)
    meas, scale = {}, {}
    tot_tets = sum(len(r.tets) for r in system.regions)

    def tick(name, fn):
        t = time.perf_counter()
        r = fn()
        meas[name] = time.perf_counter() - t
        return r

    g, H = tick("assemble", lambda: newton.assemble(xhs, xts, masses, [reg], None, mu, offset, h))
    scale["assemble"] = tot_tets / (hi - lo)
    # per CG iteration: a (1 + cg_iters)-iteration solve minus a 1-iteration
    # solve, so the per-solve setup (block-Jacobi inverses) is charged apart
    t = time.perf_counter()
    _, i1, _, _ = blocksparse.pcg(H, -g, 1e-30, max_iters=1)
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    _, i2, _, _ = blocksparse.pcg(H, -g, 1e-30, max_iters=1 + cg_iters)
    t2 = time.perf_counter() - t
    meas["cg_iter"] = max(t2 - t1, 0.0) / max(i2 - i1, 1)
    meas["cg_setup"] = max(t1 - meas["cg_iter"], 0.0)
    nb_sample = len(H.rows)
    # CG work is per stored block and per row; the slice's matrix has the
    # scene's blocks-per-row ratio, so it scales by the stored-block count
    scale["cg_iter"] = (full_blocks / nb_sample) if full_blocks else scale["assemble"]
    scale["cg_setup"] = len(system.masses) / len(masses)
    tick("energy", lambda: newton.energy(xhs, xts, masses, [reg], None, mu, offset, h))
    scale["energy"] = scale["assemble"]
    res = tick("ccd", lambda: geometry.step_limit(xs, xhs, tris, edges, verts, 0.1 * offset))
    scale["ccd"] = len(system.surface_triangles) / max(len(tris), 1)
    n_c = 0
    if contacts and aset_state is not None and len(aset_state[0]):
        cs = constraint_set(aset_state)
        n_c = len(cs)
        tick("refresh", lambda: cs.refresh_anchors(x))
        batch = cs.snapshot()
        tick("contact_assemble", lambda: newton.assemble(x_hat, x_tilde, system.masses, [], batch, mu, offset, h))
        tick("contact_energy", lambda: batch.energy(batch.values(x_hat, offset), mu))
        tick("dual", lambda: cs.dual_sweep(x_hat, offset, mu, 0.9))
        _, kinds, quads, tois = res
        tick("update", lambda: cs.update(kinds, quads, tois))
        for name in ("refresh", "contact_assemble", "contact_energy", "dual", "update"):
            scale[name] = 1.0
    full = {name: meas[name] * scale[name] for name in meas}
    info = {"region": k, "tets": hi - lo, "tets_total": tot_tets, "blocks": nb_sample, "tris": int(len(tris)),
            "constraints": n_c, "candidates_blocking": int(len(res[1]))}
    return meas, scale, full, info


def frame_ms(full, counts):
    """Reference ms/frame from whole-scene stage times (s) and per-frame op
    counts {newton, cg, energy, passes}."""
    g = lambda k: full.get(k, 0.0)
    parts = {
        "stiffness_ms": 1e3 * g("assemble"),      # stiffness_diagonal_max: one assembly per frame
        "assemble_ms": 1e3 * (g("assemble") + g("contact_assemble")) * counts["newton"],
        "pcg_ms": 1e3 * (g("cg_iter") * counts["cg"] + g("cg_setup") * counts["newton"]),
        "energy_ms": 1e3 * (g("energy") + g("contact_energy")) * counts["energy"],
        "ccd_ms": 1e3 * g("ccd") * counts["passes"],
        "active_set_ms": 1e3 * (g("refresh") + g("dual") + g("update")) * counts["passes"],
    }
    return float(sum(parts.values())), parts
