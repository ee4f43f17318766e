"""Oracle: hyperelastic energies, stresses and PSD-projected element Hessians.

Restates `intact/elasticity.py` (paths relative to /root/reference/pkg/src).
Test infrastructure only — see oracle/__init__.py.

Models are keyed by the reference's `MaterialModel` string values
('snh', 'nh', 'cor', 'lin'); a material is the triple (model, mu, lam).
LAPACK-backed steps (SVD, 3x3 eigh, roots) use numpy exactly as the
reference does, so on the same host the outputs match bit-for-bit; across
hosts they are pinned only to the reference's own tolerances.
"""

from __future__ import annotations

import numpy as np

PAIRS = ((0, 1), (0, 2), (1, 2))     # MODE_PAIRS, intact/elasticity.py:24
DET_KEEP = 0.2                       # INVERSION_DET_FRACTION, :27
STEP_SCALE = 0.9                     # INVERSION_STEP_SCALE, :28


def lame(young, poisson):
    """(mu, lambda) — `lame_parameters` (intact/elasticity.py:38-42)."""
    return (young / (2.0 * (1.0 + poisson)),
            young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)))


def def_grad(x, tets, shape_rows):
    """F = sum_k x_k (x) A_k, summed k = 0..3 in order (intact/elasticity.py:66-68)."""
    xs = x[tets]
    F = xs[:, 0, :, None] * shape_rows[:, 0, None, :]
    for k in range(1, 4):
        F = F + xs[:, k, :, None] * shape_rows[:, k, None, :]
    return F


def cof(F):
    """Cofactor matrix, columns = crosses of F's columns (:75-80)."""
    c0, c1, c2 = F[..., :, 0], F[..., :, 1], F[..., :, 2]
    return np.stack([np.cross(c1, c2), np.cross(c2, c0), np.cross(c0, c1)], axis=-1)


def rv_svd(F):
    """Rotation-variant SVD: det U = det V = +1, reflection in sigma[2] (:83-97)."""
    U, s, Vt = np.linalg.svd(F)
    V = np.swapaxes(Vt, -1, -2)
    s = s.copy()
    for M in (U, V):
        neg = np.linalg.det(M) < 0.0
        M[neg, :, 2] *= -1.0
        s[neg, 2] *= -1.0
    return U, s, V


def _strain(F):
    eps = 0.5 * (F + np.swapaxes(F, -1, -2))
    for i in range(3):
        eps[..., i, i] -= 1.0
    return eps


def psi(model, mu, lam, F):
    """Energy density per rest volume (:108-132); NH is +inf for det F <= 0."""
    if model == "lin":
        eps = _strain(F)
        tr = np.trace(eps, axis1=-2, axis2=-1)
        return mu * (eps * eps).sum(axis=(-2, -1)) + 0.5 * lam * tr * tr
    if model == "cor":
        U, s, V = rv_svd(F)
        R = U @ np.swapaxes(V, -1, -2)
        dF = F - R
        tr = s.sum(axis=-1) - 3.0
        return mu * (dF * dF).sum(axis=(-2, -1)) + 0.5 * lam * tr * tr
    ic = (F * F).sum(axis=(-2, -1))
    J = np.linalg.det(F)
    if model == "snh":
        return 0.5 * mu * (ic - 3.0) - mu * (J - 1.0) + 0.5 * lam * (J - 1.0) ** 2
    pos = J > 0.0
    lj = np.log(J, where=pos, out=np.zeros_like(J))
    out = np.full(F.shape[:-2], np.inf)
    val = 0.5 * mu * (ic - 3.0) - mu * lj + 0.5 * lam * lj * lj
    out[pos] = val[pos]
    return out


def total_energy(model, mu, lam, F, volumes):
    """sum psi * V as `energy` (:135-137)."""
    return float(np.dot(psi(model, mu, lam, F), volumes))


def stress(model, mu, lam, F):
    """First Piola-Kirchhoff stress (:140-164)."""
    if model == "lin":
        eps = _strain(F)
        tr = np.trace(eps, axis1=-2, axis2=-1)
        P = 2.0 * mu * eps
        for i in range(3):
            P[..., i, i] += lam * tr
        return P
    if model == "cor":
        U, s, V = rv_svd(F)
        R = U @ np.swapaxes(V, -1, -2)
        return 2.0 * mu * (F - R) + lam * (s.sum(axis=-1) - 3.0)[..., None, None] * R
    J = np.linalg.det(F)
    C = cof(F)
    if model == "snh":
        return mu * F + (lam * (J - 1.0) - mu)[..., None, None] * C
    return mu * F + (lam * np.log(J) - mu)[..., None, None] * C / J[..., None, None]


def elem_grad(model, mu, lam, F, shape_rows, volumes):
    """dE/dx per element (M,4,3) — `element_gradients` (:167-170)."""
    P = stress(model, mu, lam, F)
    return volumes[:, None, None] * np.einsum("mab,mkb->mka", P, shape_rows)


def eigensystem(model, mu, lam, F):
    """(U, sigma, V, lam9, diag_vectors) — `eigen_system` (:188-249).

    lam9 = [3 scaling eigenvalues (eigh of the 3x3 A), 3 twist, 3 flip]
    in MODE_PAIRS order; diag_vectors row k is the k-th scaling direction.
    """
    M = F.shape[0]
    if model == "lin":
        U = np.broadcast_to(np.eye(3), (M, 3, 3)).copy()
        V = U.copy()
        s = np.ones((M, 3))
    else:
        U, s, V = rv_svd(F)
    s1, s2, s3 = s[:, 0], s[:, 1], s[:, 2]
    A = np.empty((M, 3, 3))
    twist = np.empty((M, 3))
    flip = np.empty((M, 3))
    if model in ("lin", "cor"):
        A[:] = 2.0 * mu * np.eye(3) + lam
        flip[:] = 2.0 * mu
        if model == "lin":
            twist[:] = 0.0
        else:
            num = 2.0 * lam * (s.sum(axis=1) - 3.0) - 4.0 * mu
            for k, (p, q) in enumerate(PAIRS):
                twist[:, k] = 2.0 * mu + num / np.maximum(s[:, p] + s[:, q], 1e-8)
    elif model == "snh":
        J = s1 * s2 * s3
        g = np.stack([s2 * s3, s1 * s3, s1 * s2], axis=1)
        kj = lam * (J - 1.0) - mu
        A[:] = lam * g[:, :, None] * g[:, None, :]
        for i in range(3):
            A[:, i, i] = mu + lam * g[:, i] ** 2
        for (i, j), sk in (((0, 1), s3), ((0, 2), s2), ((1, 2), s1)):
            A[:, i, j] += kj * sk
            A[:, j, i] += kj * sk
        other = np.stack([s3, s2, s1], axis=1)
        twist[:] = mu + kj[:, None] * other
        flip[:] = mu - kj[:, None] * other
    else:  # nh
        J = s1 * s2 * s3
        m = lam * np.log(np.abs(J)) - mu
        inv = 1.0 / s
        A[:] = lam * inv[:, :, None] * inv[:, None, :]
        for i in range(3):
            A[:, i, i] = mu + (lam - m) * inv[:, i] ** 2
        pp = np.stack([s1 * s2, s1 * s3, s2 * s3], axis=1)
        twist[:] = mu + m[:, None] * (1.0 / pp)
        flip[:] = mu - m[:, None] * (1.0 / pp)
    ev, vecs = np.linalg.eigh(A)
    lam9 = np.concatenate([ev, twist, flip], axis=1)
    return U, s, V, lam9, np.swapaxes(vecs, 1, 2)


def vertex_blocks(model, mu, lam, F, shape_rows, volumes, clamp=True):
    """PSD-projected per-element 12x12 Hessians as (M,4,4,3,3) vertex blocks via
    the sparse mode path — `psd_block_hessians` + `assemble_vertex_blocks`
    (:274-299)."""
    U, _, V, lam9, dv = eigensystem(model, mu, lam, F)
    if clamp:
        lam9 = np.maximum(lam9, 0.0)
    y = np.einsum("mba,mib->mia", V, shape_rows)
    Mij = np.einsum("mia,mjb->mijab", y, y)
    W = np.einsum("mk,mka,mkb->mab", lam9[:, :3], dv, dv)
    S = W[:, None, None] * Mij
    for k, (p, q) in enumerate(PAIRS):
        lt = 0.5 * lam9[:, 3 + k, None, None]
        lf = 0.5 * lam9[:, 6 + k, None, None]
        S[..., p, p] += (lt + lf) * Mij[..., q, q]
        S[..., q, q] += (lt + lf) * Mij[..., p, p]
        S[..., p, q] += (lf - lt) * Mij[..., q, p]
        S[..., q, p] += (lf - lt) * Mij[..., p, q]
    K = np.einsum("mra,mijab,msb->mijrs", U, S, U)
    return K * volumes[:, None, None, None, None]


def _first_positive_root(coeffs):
    """Smallest positive real root of a polynomial (:321-334)."""
    c = np.array(coeffs, dtype=np.float64)
    big = np.abs(c).max()
    if big == 0.0:
        return np.inf
    c = np.trim_zeros(c / big, "f")
    if len(c) <= 1:
        return np.inf
    z = np.roots(c)
    re = z[np.abs(z.imag) < 1e-10 * (1.0 + np.abs(z.real))].real
    re = re[re > 1e-12]
    return re.min() if len(re) else np.inf


def inversion_cap(model, x, p, tets, shape_rows):
    """Largest step along p keeping det F >= 0.2 det F(x) (:337-356); NH only."""
    if model != "nh":
        return 1.0
    A = def_grad(x, tets, shape_rows)
    B = def_grad(p, tets, shape_rows)
    da, db = np.linalg.det(A), np.linalg.det(B)
    c1 = (cof(A) * B).sum(axis=(-2, -1))
    c2 = (cof(B) * A).sum(axis=(-2, -1))
    c0 = (1.0 - DET_KEEP) * da
    alpha = 1.0
    for m in np.flatnonzero((np.abs(B) > 0.0).any(axis=(1, 2))):
        alpha = min(alpha, STEP_SCALE * _first_positive_root([db[m], c2[m], c1[m], c0[m]]))
    return max(alpha, 0.0)
