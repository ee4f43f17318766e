"""Oracle: augmented-Lagrangian contact constraints and the active set.

Restates `intact/contact.py` (paths relative to /root/reference/pkg/src) as
structure-of-arrays state instead of a dict of dataclasses — the same layout
the device active set uses — while keeping the reference's insertion order,
dedup keys, admission rule, pruning and multiplier/decay branches exactly.
Test infrastructure only — see oracle/__init__.py.
"""

from __future__ import annotations

import numpy as np

from .geometry import EE, VF, pair_eval

PRUNE_GAMMA = 0.01                  # GAMMA_PRUNE_THRESHOLD, intact/contact.py:20


def key_of(kind, quad):
    """(kind, sorted ids) — `constraint_key` (intact/contact.py:23-24)."""
    return (int(kind), tuple(sorted(int(i) for i in quad)))


def sum12(prod):
    """`float(np.sum(a))` of a (.., 4, 3) product array, i.e. numpy's pairwise
    sum with 8 accumulators over the 12 flattened entries."""
    q = prod.reshape(prod.shape[:-2] + (12,))
    acc = ((q[..., 0] + q[..., 1]) + (q[..., 2] + q[..., 3])) + \
        ((q[..., 4] + q[..., 5]) + (q[..., 6] + q[..., 7]))
    for k in range(8, 12):
        acc = acc + q[..., k]
    return acc


def earliest_admission(quads, tois):
    """Keep a new pair iff its TOI is the earliest among new pairs at one of
    its vertices — `admission_filter` (intact/contact.py:144-151)."""
    v = quads.ravel()
    t4 = np.repeat(tois, 4)
    uniq, inv = np.unique(v, return_inverse=True)
    first = np.full(len(uniq), np.inf)
    np.minimum.at(first, inv, t4)
    return (t4 == first[inv]).reshape(-1, 4).any(axis=1)


class ConstraintSet:
    """Insertion-ordered SoA active set (`ActiveSet`, intact/contact.py:154-261)."""

    def __init__(self, admit_all=False):
        self.admit_all = admit_all
        self.kind = np.zeros(0, dtype=np.int64)
        self.quad = np.zeros((0, 4), dtype=np.int64)
        self.lam = np.zeros(0)
        self.gamma = np.zeros(0)
        self.s = np.zeros(0)
        self.anchor_d = np.zeros(0)
        self.anchor_grad = np.zeros((0, 4, 3))
        self.anchor_x = np.zeros((0, 4, 3))
        self._keys: list = []

    def __len__(self):
        return len(self.kind)

    def keys(self):
        return list(self._keys)

    def _take(self, idx):
        for f in ("kind", "quad", "lam", "gamma", "s", "anchor_d", "anchor_grad", "anchor_x"):
            setattr(self, f, getattr(self, f)[idx])
        self._keys = [self._keys[i] for i in np.asarray(idx, dtype=np.int64)]

    def add(self, kind, quad, **state):
        """Append one constraint unless its key is resident (`add`, :172-177)."""
        k = key_of(kind, quad)
        if k in set(self._keys):
            return False
        self._append(np.array([kind]), np.asarray(quad, dtype=np.int64)[None], [k], **state)
        return True

    def _append(self, kinds, quads, keys, lam=None, gamma=None, s=None,
                anchor_d=None, anchor_grad=None, anchor_x=None):
        n = len(kinds)
        self.kind = np.concatenate([self.kind, kinds.astype(np.int64)])
        self.quad = np.concatenate([self.quad, quads.astype(np.int64)])
        self.lam = np.concatenate([self.lam, np.zeros(n) if lam is None else np.atleast_1d(lam)])
        self.gamma = np.concatenate([self.gamma, np.ones(n) if gamma is None else np.atleast_1d(gamma)])
        self.s = np.concatenate([self.s, np.zeros(n) if s is None else np.atleast_1d(s)])
        self.anchor_d = np.concatenate(
            [self.anchor_d, np.zeros(n) if anchor_d is None else np.atleast_1d(anchor_d)])
        self.anchor_grad = np.concatenate(
            [self.anchor_grad, np.zeros((n, 4, 3)) if anchor_grad is None
             else np.asarray(anchor_grad).reshape(n, 4, 3)])
        self.anchor_x = np.concatenate(
            [self.anchor_x, np.zeros((n, 4, 3)) if anchor_x is None
             else np.asarray(anchor_x).reshape(n, 4, 3)])
        self._keys += list(keys)

    def update(self, kinds, quads, tois):
        """Dedup vs resident keys, earliest-TOI admission among the new pairs,
        append in blocking order (first key wins), then prune gamma < 0.01.
        Returns (admitted, pruned) as the reference counts them
        (`ActiveSet.update`, intact/contact.py:179-205)."""
        resident = set(self._keys)
        admitted = 0
        if len(kinds):
            new = np.array([key_of(k, q) not in resident for k, q in zip(kinds, quads)], dtype=bool)
            if new.any():
                nq, nt, nk = quads[new], tois[new], kinds[new]
                keep = np.ones(len(nt), dtype=bool) if self.admit_all else earliest_admission(nq, nt)
                add_k, add_q, add_keys = [], [], []
                seen = set(resident)
                for k, q in zip(nk[keep], nq[keep]):
                    admitted += 1               # the reference counts duplicates too
                    key = key_of(k, q)
                    if key in seen:
                        continue
                    seen.add(key)
                    add_k.append(int(k))
                    add_q.append(np.asarray(q, dtype=np.int64))
                    add_keys.append(key)
                if add_k:
                    self._append(np.array(add_k), np.array(add_q), add_keys)
        stale = self.gamma < PRUNE_GAMMA
        n_stale = int(stale.sum())
        if n_stale:
            self._take(np.flatnonzero(~stale))
        return admitted, n_stale

    def refresh_anchors(self, x):
        """Re-linearise every constraint at x (`refresh_anchors`, :207-235).
        Degenerate evaluations keep the stale anchor, or install a null
        anchor (d = inf, grad = 0) when the constraint was never anchored
        (anchor_d <= 0).  Returns the degenerate count."""
        n_bad = 0
        for kind in (VF, EE):
            sel = np.flatnonzero(self.kind == kind)
            if len(sel) == 0:
                continue
            pts = x[self.quad[sel]]
            d, g, _, degen = pair_eval(kind, pts)
            good = sel[~degen]
            self.anchor_d[good] = d[~degen]
            self.anchor_grad[good] = g[~degen].reshape(-1, 4, 3)
            self.anchor_x[good] = pts[~degen]
            bad = sel[degen]
            n_bad += len(bad)
            fresh = bad[self.anchor_d[bad] <= 0.0]
            pts_bad = pts[degen][self.anchor_d[bad] <= 0.0]
            self.anchor_x[fresh] = pts_bad
            self.anchor_grad[fresh] = 0.0
            self.anchor_d[fresh] = np.inf
        return n_bad

    def snapshot(self):
        """Frozen arrays for one subproblem (`batch`, :237-249)."""
        if len(self) == 0:
            return None
        return Batch(self.kind.copy(), self.quad.copy(), self.lam.copy(), self.gamma.copy(),
                     self.anchor_d.copy(), self.anchor_grad.copy(), self.anchor_x.copy())

    def dual_sweep(self, x_hat, offset, mu, decay):
        """Multiplier/decay sweep (`dual_update_sweep` + `dual_update`,
        :91-106, :251-261): s = max(0, c - lam/mu); s == 0 -> lam -= mu c,
        gamma = 1; s > 0 -> lam = 0, gamma *= decay.  Returns max |c| over the
        s == 0 branch."""
        if len(self) == 0:
            return 0.0
        disp = x_hat[self.quad] - self.anchor_x
        c = (self.anchor_d + sum12(self.anchor_grad * disp)) - offset
        s = np.maximum(0.0, c - self.lam / mu)
        self.s = s
        on = s == 0.0
        self.lam = np.where(on, self.lam - mu * c, 0.0)
        self.gamma = np.where(on, 1.0, decay * self.gamma)
        return float(np.abs(c[on]).max()) if on.any() else 0.0


class Batch:
    """SoA view frozen at anchor-refresh time (`ConstraintBatch`, :109-141)."""

    def __init__(self, kind, quad, lam, gamma, anchor_d, anchor_grad, anchor_x):
        self.kind, self.quad, self.lam, self.gamma = kind, quad, lam, gamma
        self.anchor_d, self.anchor_grad, self.anchor_x = anchor_d, anchor_grad, anchor_x

    def __len__(self):
        return len(self.kind)

    def values(self, x_hat, offset):
        disp = x_hat[self.quad] - self.anchor_x
        return self.anchor_d + np.einsum("cia,cia->c", self.anchor_grad, disp) - offset

    def energy(self, c, mu):
        s = np.maximum(0.0, c - self.lam / mu)
        r = c - s
        return float(np.sum(self.gamma * (0.5 * mu * r * r - self.lam * r)))

    def grad_terms(self, c, mu):
        sh = c - self.lam / mu
        coef = mu * self.gamma * (sh - np.maximum(0.0, sh))
        return coef[:, None, None] * self.anchor_grad

    def hess_grids(self, mu):
        return np.einsum("c,cia,cjb->cijab", mu * self.gamma, self.anchor_grad, self.anchor_grad)
