"""Oracle: AL subproblem (assembly, incremental energy, line search, Newton loop).

Restates `intact/solver.py` (paths relative to /root/reference/pkg/src).
Test infrastructure only — see oracle/__init__.py.

A region is a tuple (model, mu, lam, tets, shape_rows, volumes) — the data of
the reference's `ElasticRegion` with the material expanded to Lame pairs.
"""

from __future__ import annotations

import numpy as np

from .blocksparse import SymBlockMatrix, pcg, upper_triplets
from .material import def_grad, elem_grad, inversion_cap, total_energy, vertex_blocks

NEWTON_CAP = 64                     # intact/solver.py:31
LS_HALVINGS = 30                    # intact/solver.py:32


class NonFiniteEnergy(RuntimeError):
    """`NonFiniteEnergyError` (intact/solver.py:35-37)."""


def _scatter(out, ids, terms):
    """Accumulate (k,4,3) clique terms onto (n,3) rows (`scatter_terms`, :74-77)."""
    flat = (ids[:, :, None] * 3 + np.arange(3)).ravel()
    out += np.bincount(flat, weights=terms.ravel(), minlength=out.size).reshape(out.shape)


def _region_blocks(reg, F, memo):
    """PSD blocks; LIN is configuration independent and memoised per region
    (`region_hessian_blocks`, :50-62)."""
    model, mu, lam, tets, rows, vols = reg
    if model == "lin":
        key = id(tets)
        if key not in memo:
            memo[key] = vertex_blocks(model, mu, lam, F, rows, vols)
        return memo[key]
    return vertex_blocks(model, mu, lam, F, rows, vols)


def energy(x_hat, x_tilde, masses, regions, batch, mu, offset, h, friction=None):
    """Incremental potential L(x_hat) (`incremental_energy`, :88-106)."""
    d = x_hat - x_tilde
    total = 0.5 * float(np.sum(masses * np.sum(d * d, axis=1)))
    el = 0.0
    for model, m_, l_, tets, rows, vols in regions:
        el += total_energy(model, m_, l_, def_grad(x_hat, tets, rows), vols)
    total += h * h * el
    if batch is not None and len(batch):
        total += batch.energy(batch.values(x_hat, offset), mu)
    if friction is not None:
        total += friction.energy(x_hat)
    return total


def assemble(x_hat, x_tilde, masses, regions, batch, mu, offset, h, dbc=None, memo=None, friction=None):
    """(grad (n,3), SymBlockMatrix H) of the AL objective (`assemble`, :109-156)."""
    memo = {} if memo is None else memo
    n = len(x_hat)
    h2 = h * h
    g = masses[:, None] * (x_hat - x_tilde)
    R, C, B = [np.arange(n)], [np.arange(n)], [masses[:, None, None] * np.eye(3)]
    for reg in regions:
        model, m_, l_, tets, rows, vols = reg
        F = def_grad(x_hat, tets, rows)
        if not np.isfinite(total_energy(model, m_, l_, F, vols)):
            raise NonFiniteEnergy("elastic energy is not finite at the evaluation point")
        _scatter(g, tets, h2 * elem_grad(model, m_, l_, F, rows, vols))
        r, c, b = upper_triplets(tets, h2 * _region_blocks(reg, F, memo))
        R.append(r), C.append(c), B.append(b)
    if batch is not None and len(batch):
        cv = batch.values(x_hat, offset)
        _scatter(g, batch.quad, batch.grad_terms(cv, mu))
        r, c, b = upper_triplets(batch.quad, batch.hess_grids(mu))
        R.append(r), C.append(c), B.append(b)
    if friction is not None and len(friction):
        _scatter(g, friction.indices, friction.grad_terms(x_hat))
        r, c, b = upper_triplets(friction.indices, friction.hess_grids(x_hat))
        R.append(r), C.append(c), B.append(b)
    H = SymBlockMatrix(n, np.concatenate(R), np.concatenate(C), np.concatenate(B))
    if dbc is not None and dbc.any():
        H.mask(dbc, masses[:, None, None] * np.eye(3))
        g[dbc] = 0.0
    return g, H


def backtrack(x_hat, p, fn, cap=1.0):
    """Largest r in {cap, cap/2, ...} with fn(x + r p) < fn(x); after 30
    halvings return the lowest sample and stalled=True (`line_search`, :159-175)."""
    base = fn(x_hat)
    r = min(1.0, cap)
    best_r, best_e = r, np.inf
    for _ in range(LS_HALVINGS + 1):
        e = fn(x_hat + r * p)
        if e < base:
            return r, False
        if e < best_e:
            best_r, best_e = r, e
        r *= 0.5
    return best_r, True


def subproblem(x_tilde, x, x_hat0, masses, regions, aset, mu, offset, h,
               cg_tol=1e-4, decay=0.9, dbc=None, memo=None, friction=None):
    """Newton loop + one dual sweep (`solve_subproblem`, :178-233).

    Returns (x_hat, newton_iters, cg_iters, stalled, worst_violation).
    """
    memo = {} if memo is None else memo
    aset.refresh_anchors(x)
    batch = aset.snapshot()

    def fn(y):
        return energy(y, x_tilde, masses, regions, batch, mu, offset, h, friction)

    x_hat = x_hat0.copy()
    newton = cg_total = 0
    stalled = False
    for _ in range(NEWTON_CAP):
        g, H = assemble(x_hat, x_tilde, masses, regions, batch, mu, offset, h, dbc, memo, friction)
        if not np.any(g):
            break
        p, its, _, _ = pcg(H, -g, cg_tol)
        cg_total += its
        if float(np.sum(g * p)) >= 0.0:
            p = -np.einsum("nij,nj->ni", np.linalg.inv(H.diag()), g)
        cap = 1.0
        for model, _m, _l, tets, rows, _v in regions:
            cap = min(cap, inversion_cap(model, x_hat, p, tets, rows))
        r, st = backtrack(x_hat, p, fn, cap)
        x_hat = x_hat + r * p
        newton += 1
        stalled = stalled or st
        if r == 1.0:
            break
    else:
        stalled = True
    worst = aset.dual_sweep(x_hat, offset, mu, decay)
    return x_hat, newton, cg_total, stalled, worst
