"""Oracle: pair distances, additive CCD, LBVH broad phase, step limiting.

Restates `intact/distance.py`, `intact/bvh.py` and `intact/ccd.py` of the
reference (paths relative to /root/reference/pkg/src).  Test infrastructure
only — see oracle/__init__.py.

Arithmetic order is spelled out wherever numpy's own order decides the last
bit, so that TOIs and candidate sets are bit-identical to the reference as
run in the build container (pinned by tests/test_oracle_golden.py).
"""

from __future__ import annotations

import numpy as np

VF, EE = 0, 1                      # PairKind values, intact/distance.py:28-30
EE_PARALLEL_TOL = 1e-10            # intact/distance.py:18
DEGENERATE_DISTANCE = 1e-30        # intact/distance.py:21
DEGENERATE_RELATIVE = 1e-12        # intact/distance.py:25
S_ACCD = 0.1                       # intact/ccd.py:20
ACCD_MAX_ITERS = 100               # intact/ccd.py:21
BRUTE_FORCE_PAIRS = 1 << 14        # intact/ccd.py:101


def dot3(u, v):
    """`np.einsum('...k,...k->...')` on 3-vectors as numpy 2.3 evaluates it
    (intact/distance.py:43-44): (u0 v0 + u2 v2) + u1 v1, no fused multiply-add."""
    return (u[..., 0] * v[..., 0] + u[..., 2] * v[..., 2]) + u[..., 1] * v[..., 1]


def norm3(u):
    """`np.linalg.norm(u, axis=-1)` for 3-vectors: sequential sum of squares."""
    return np.sqrt((u[..., 0] * u[..., 0] + u[..., 1] * u[..., 1]) + u[..., 2] * u[..., 2])


def clamp01(t):
    """`np.clip(t, 0, 1)`: NaN propagates (intact/distance.py:104-105)."""
    return np.minimum(np.maximum(t, 0.0), 1.0)


def triangle_weights(p, a, b, c):
    """Barycentric weights of the closest point of triangle abc to p.

    Restates `point_triangle_weights` (intact/distance.py:47-101): seven
    Voronoi regions tested in the fixed priority order vertex a, vertex b,
    vertex c, edge ab, edge ac, edge bc, interior; the first match wins.
    """
    ab, ac = b - a, c - a
    ap, bp, cp = p - a, p - b, p - c
    d1, d2 = dot3(ab, ap), dot3(ac, ap)
    d3, d4 = dot3(ab, bp), dot3(ac, bp)
    d5, d6 = dot3(ab, cp), dot3(ac, cp)
    vc = d1 * d4 - d3 * d2
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4
    with np.errstate(divide="ignore", invalid="ignore"):
        t_ab = np.where(d1 != d3, d1 / (d1 - d3), 0.0)
        t_ac = np.where(d2 != d6, d2 / (d2 - d6), 0.0)
        num = d4 - d3
        den = (d4 - d3) + (d5 - d6)
        t_bc = np.where(den != 0.0, num / den, 0.0)
        tot = (va + vb) + vc
        bary_v = np.where(tot != 0.0, vb / tot, 1.0 / 3.0)
        bary_u = np.where(tot != 0.0, vc / tot, 1.0 / 3.0)
    one, zero = np.ones_like(d1), np.zeros_like(d1)
    regions = [
        ((d1 <= 0.0) & (d2 <= 0.0), (one, zero, zero)),
        ((d3 >= 0.0) & (d4 <= d3), (zero, one, zero)),
        ((d6 >= 0.0) & (d5 <= d6), (zero, zero, one)),
        ((vc <= 0.0) & (d1 >= 0.0) & (d3 <= 0.0), (1.0 - t_ab, t_ab, zero)),
        ((vb <= 0.0) & (d2 >= 0.0) & (d6 <= 0.0), (1.0 - t_ac, zero, t_ac)),
        ((va <= 0.0) & (d4 >= d3) & (d5 >= d6), (zero, 1.0 - t_bc, t_bc)),
    ]
    w = np.stack([(1.0 - bary_v) - bary_u, bary_v, bary_u], axis=-1)
    # apply in reverse priority so that earlier regions overwrite later ones
    for mask, vals in reversed(regions):
        w = np.where(mask[:, None], np.stack(vals, axis=-1), w)
    return w


def segment_params(p1, p2, q1, q2):
    """Closest-point parameters (s, t) of two segments.

    Restates `segment_segment_params` (intact/distance.py:108-150), including
    the near-parallel fallback over the four endpoint projections with
    first-index argmin tie breaking.
    """
    d1, d2, r = p2 - p1, q2 - q1, p1 - q1
    a, e, b = dot3(d1, d1), dot3(d2, d2), dot3(d1, d2)
    c, f = dot3(d1, r), dot3(d2, r)
    a_s = np.maximum(a, 1e-300)
    e_s = np.maximum(e, 1e-300)
    den = a * e - b * b
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(den > 0.0, clamp01((b * f - c * e) / np.maximum(den, 1e-300)), 0.0)
        t_raw = (b * s + f) / e_s
        t = clamp01(t_raw)
        s = np.where(t_raw < 0.0, clamp01(-c / a_s), s)
        s = np.where(t_raw > 1.0, clamp01((b - c) / a_s), s)
    cr = np.stack([d1[:, 1] * d2[:, 2] - d1[:, 2] * d2[:, 1],
                   d1[:, 2] * d2[:, 0] - d1[:, 0] * d2[:, 2],
                   d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0]], axis=-1)
    par = norm3(cr) < EE_PARALLEL_TOL * np.sqrt(a * e)
    if par.any():
        zero, one = np.zeros_like(a), np.ones_like(a)
        cs = np.stack([zero, one, clamp01(-c / a_s), clamp01((b - c) / a_s)], axis=-1)
        ct = np.stack([clamp01(f / e_s), clamp01((f + b) / e_s), zero, one], axis=-1)
        diff = (p1[:, None, :] + cs[:, :, None] * d1[:, None, :]) - (
            q1[:, None, :] + ct[:, :, None] * d2[:, None, :])
        sq = diff * diff
        dist2 = (sq[..., 0] + sq[..., 1]) + sq[..., 2]
        pick = dist2.argmin(axis=-1)
        rows = np.arange(len(a))
        s = np.where(par, cs[rows, pick], s)
        t = np.where(par, ct[rows, pick], t)
    return s, t


def _witness(kind, pts):
    """(diff, signed weights) of a pair; diff = witness A minus witness B."""
    if kind == VF:
        p, a, b, c = pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]
        w = triangle_weights(p, a, b, c)
        closest = (w[:, 0:1] * a + w[:, 1:2] * b) + w[:, 2:3] * c
        weights = np.concatenate([np.ones((len(p), 1)), -w], axis=1)
        return p - closest, weights
    p1, p2, q1, q2 = pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]
    s, t = segment_params(p1, p2, q1, q2)
    pa = p1 + s[:, None] * (p2 - p1)
    pb = q1 + t[:, None] * (q2 - q1)
    weights = np.stack([1.0 - s, s, -(1.0 - t), -t], axis=1)
    return pa - pb, weights


def pair_eval(kind, pts):
    """(d, grad (n,12), weights (n,4), degenerate) — `vf_eval`/`ee_eval` +
    `_finish` (intact/distance.py:153-189)."""
    pts = np.asarray(pts, dtype=np.float64)
    diff, weights = _witness(kind, pts)
    d = norm3(diff)
    scale = np.abs(pts).max(axis=(1, 2))
    degen = d <= np.maximum(DEGENERATE_DISTANCE, DEGENERATE_RELATIVE * scale)
    with np.errstate(divide="ignore", invalid="ignore"):
        unit = np.where(degen[:, None], 0.0, diff / np.maximum(d, 1e-300)[:, None])
    grad = (weights[:, :, None] * unit[:, None, :]).reshape(len(d), 12)
    return d, grad, weights, degen


def pair_dist(kind, pts):
    """Distances only — `pair_distances` (intact/distance.py:192-203)."""
    diff, _ = _witness(kind, pts)
    return norm3(diff)


# ----------------------------------------------------------------- ACCD

def _centered_motion(kind, disp):
    """Displacement minus the mean of the two sides' mean displacements
    (`_split_means`, intact/ccd.py:24-27 and :61)."""
    if kind == VF:
        ma = disp[:, 0]
        mb = ((disp[:, 1] + disp[:, 2]) + disp[:, 3]) / 3.0
    else:
        ma = (disp[:, 0] + disp[:, 1]) / 2.0
        mb = (disp[:, 2] + disp[:, 3]) / 2.0
    return disp - 0.5 * (ma + mb)[:, None, :]


def _motion_bound(kind, pm):
    """l_p of `_motion_bound` (intact/ccd.py:30-34)."""
    n = norm3(pm)
    if kind == VF:
        return n[:, 0] + np.maximum(np.maximum(n[:, 1], n[:, 2]), n[:, 3])
    return np.maximum(n[:, 0], n[:, 1]) + np.maximum(n[:, 2], n[:, 3])


def accd(kind, x0, x1, min_gap):
    """Conservative TOI per pair in [0, 1] — `accd_batch` (intact/ccd.py:37-91).

    Vectorised over pairs; each pair follows exactly the reference's scalar
    recurrence: x <- x + t_l pm, gap = d(x) - min_gap, stop when t > 0 and
    gap < 0.1 gap0, t <- t + t_l, t >= 1 -> 1, t_l = 0.9 gap / l_p, capped at
    100 advancements (reporting the committed t).
    """
    x0 = np.asarray(x0, dtype=np.float64)
    x1 = np.asarray(x1, dtype=np.float64)
    n = len(x0)
    toi = np.ones(n)
    if n == 0:
        return toi
    pm = _centered_motion(kind, x1 - x0)
    lp = _motion_bound(kind, pm)
    gap0 = pair_dist(kind, x0) - min_gap
    toi[gap0 <= 0.0] = 0.0
    live = np.flatnonzero((gap0 > 0.0) & (lp >= gap0))
    if len(live) == 0:
        return toi
    x = x0[live].copy()
    pm, lp = pm[live], lp[live]
    slack = S_ACCD * gap0[live]
    t = np.zeros(len(live))
    step = (1.0 - S_ACCD) * gap0[live] / lp
    for _ in range(ACCD_MAX_ITERS):
        x = x + step[:, None, None] * pm
        gap = pair_dist(kind, x) - min_gap
        hit = (t > 0.0) & (gap < slack)
        toi[live[hit]] = t[hit]
        t = t + step
        done = hit | (~hit & (t >= 1.0))
        toi[live[~hit & (t >= 1.0)]] = 1.0
        keep = ~done
        live, x, pm, lp, slack, gap, t = (
            live[keep], x[keep], pm[keep], lp[keep], slack[keep], gap[keep], t[keep])
        if len(live) == 0:
            return toi
        step = 0.9 * gap / lp
    toi[live] = t
    return toi


# ------------------------------------------------------------------ LBVH

def _spread21(v):
    """Spread the low 21 bits to every third bit (intact/bvh.py:14-22)."""
    v = v.astype(np.uint64)
    for shift, mask in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF),
                        (8, 0x100F00F00F00F00F), (4, 0x10C30C30C30C30C3),
                        (2, 0x1249249249249249)):
        v = (v | (v << np.uint64(shift))) & np.uint64(mask)
    return v


def morton63(points):
    """63-bit Morton codes of points normalised to their bounding box
    (intact/bvh.py:25-40)."""
    lo = points.min(axis=0)
    span = points.max(axis=0) - lo
    span[span == 0.0] = 1.0
    q = np.clip(((points - lo) / span) * (2**21 - 1), 0, 2**21 - 1).astype(np.uint64)
    code = (_spread21(q[:, 0]) << np.uint64(2)) | (_spread21(q[:, 1]) << np.uint64(1)) \
        | _spread21(q[:, 2])
    return code.astype(np.int64)


class BoxTree:
    """Post-ordered LBVH with frontier queries (intact/bvh.py:54-154).

    Build order, split rule and query order follow the reference so that
    candidate lists come out in the reference's order, not just as the same
    set.
    """

    def __init__(self, lo, hi):
        m = len(lo)
        self.m = m
        if m == 0:
            self.root = -1
            return
        codes = morton63(0.5 * (np.asarray(lo) + np.asarray(hi)))
        order = np.argsort(codes, kind="stable")
        codes = codes[order]
        n_nodes = 2 * m - 1
        self.left = np.full(n_nodes, -1, dtype=np.int64)
        self.right = np.full(n_nodes, -1, dtype=np.int64)
        self.prim = np.full(n_nodes, -1, dtype=np.int64)
        height = np.zeros(n_nodes, dtype=np.int64)
        nxt = 0
        done: list[int] = []
        todo: list[tuple[int, int, int]] = [(0, m, -1)]
        while todo:
            a, b, mid = todo.pop()
            if b - a == 1:
                self.prim[nxt] = order[a]
                done.append(nxt)
                nxt += 1
            elif mid < 0:
                mid = self._split(codes, a, b)
                if not a < mid < b:
                    mid = (a + b) // 2
                todo += [(a, b, mid), (mid, b, -1), (a, mid, -1)]
            else:
                r = done.pop()
                l_ = done.pop()
                self.left[nxt], self.right[nxt] = l_, r
                height[nxt] = 1 + max(height[l_], height[r])
                done.append(nxt)
                nxt += 1
        self.root = done.pop()
        by_h = np.argsort(height, kind="stable")
        cut = np.searchsorted(height[by_h], np.arange(height.max() + 2))
        self.levels = [by_h[cut[i]:cut[i + 1]] for i in range(height.max() + 1)]
        self.lo = np.empty((n_nodes, 3))
        self.hi = np.empty((n_nodes, 3))
        leaves = self.levels[0]
        self.lo[leaves] = lo[self.prim[leaves]]
        self.hi[leaves] = hi[self.prim[leaves]]
        for ids in self.levels[1:]:
            self.lo[ids] = np.minimum(self.lo[self.left[ids]], self.lo[self.right[ids]])
            self.hi[ids] = np.maximum(self.hi[self.left[ids]], self.hi[self.right[ids]])

    @staticmethod
    def _split(codes, lo, hi):
        """Highest-differing-bit split (intact/bvh.py:43-51)."""
        first, last = int(codes[lo]), int(codes[hi - 1])
        if first == last:
            return (lo + hi) // 2
        bit = 1 << ((first ^ last).bit_length() - 1)
        target = np.int64((first & ~((bit << 1) - 1)) | bit)
        return lo + int(np.searchsorted(codes[lo:hi], target, side="left"))

    def query(self, qlo, qhi):
        """All (query, primitive) overlaps in frontier order."""
        if self.m == 0 or len(qlo) == 0:
            return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64)
        oq, op = [], []
        q = np.arange(len(qlo), dtype=np.int64)
        node = np.full(len(qlo), self.root, dtype=np.int64)
        while len(q):
            hit = np.all(qlo[q] <= self.hi[node], axis=1) & np.all(qhi[q] >= self.lo[node], axis=1)
            q, node = q[hit], node[hit]
            leaf = self.prim[node] >= 0
            if leaf.any():
                oq.append(q[leaf])
                op.append(self.prim[node[leaf]])
            inner_q, inner_n = q[~leaf], node[~leaf]
            q = np.concatenate([inner_q, inner_q])
            node = np.concatenate([self.left[inner_n], self.right[inner_n]])
        if not oq:
            return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64)
        return np.concatenate(oq), np.concatenate(op)


def _dense_overlaps(alo, ahi, blo, bhi):
    """Row-major (i, j) box overlaps (intact/ccd.py:104-110)."""
    hit = (alo[:, None] <= bhi[None]).all(axis=2) & (blo[None] <= ahi[:, None]).all(axis=2)
    return np.nonzero(hit)


def swept_prim_boxes(x0, x1, prims, pad):
    """Swept (start ∪ end) boxes of primitives, inflated by pad
    (intact/bvh.py:172-174 applied as in intact/ccd.py:115-133)."""
    a, b = x0[prims], x1[prims]
    if a.ndim == 2:            # points
        return np.minimum(a, b) - pad, np.maximum(a, b) + pad
    return (np.minimum(a.min(axis=1), b.min(axis=1)) - pad,
            np.maximum(a.max(axis=1), b.max(axis=1)) + pad)


def candidates(x0, x1, tris, edges, verts, min_gap):
    """Broad phase (vf (n,4), ee (m,4)) — `candidate_pairs` (intact/ccd.py:113-145).

    Pads: triangles +min_gap, vertices 0, edges 0.5*min_gap each; EE keeps
    a < b; pairs sharing a vertex are dropped.
    """
    tlo, thi = swept_prim_boxes(x0, x1, tris, min_gap)
    vlo, vhi = swept_prim_boxes(x0, x1, verts, 0.0)
    if len(verts) * len(tris) <= BRUTE_FORCE_PAIRS:
        qi, ti = _dense_overlaps(vlo, vhi, tlo, thi)
    else:
        qi, ti = BoxTree(tlo, thi).query(vlo, vhi)
    v_ids, tri_ids = verts[qi], tris[ti]
    shared = (tri_ids == v_ids[:, None]).any(axis=1)
    vf = np.concatenate([v_ids[~shared, None], tri_ids[~shared]], axis=1)

    elo, ehi = swept_prim_boxes(x0, x1, edges, 0.5 * min_gap)
    if len(edges) * len(edges) <= BRUTE_FORCE_PAIRS:
        ai, bi = _dense_overlaps(elo, ehi, elo, ehi)
    else:
        ai, bi = BoxTree(elo, ehi).query(elo, ehi)
    keep = ai < bi
    ea, eb = edges[ai[keep]], edges[bi[keep]]
    shared = ((ea[:, 0:1] == eb) | (ea[:, 1:2] == eb)).any(axis=1)
    ee = np.concatenate([ea[~shared], eb[~shared]], axis=1)
    return vf.astype(np.int64).reshape(-1, 4), ee.astype(np.int64).reshape(-1, 4)


def step_limit(x, x_hat, tris, edges, verts, min_gap, cap=1.0):
    """(alpha, kinds, quads, tois) — `max_step_size` (intact/ccd.py:168-193)."""
    vf, ee = candidates(x, x_hat, tris, edges, verts, min_gap)
    t_vf = accd(VF, x[vf], x_hat[vf], min_gap)
    t_ee = accd(EE, x[ee], x_hat[ee], min_gap)
    alpha = float(cap)
    if len(t_vf):
        alpha = min(alpha, float(t_vf.min()))
    if len(t_ee):
        alpha = min(alpha, float(t_ee.min()))
    bv, be = t_vf < 1.0, t_ee < 1.0
    kinds = np.concatenate([np.full(bv.sum(), VF, dtype=np.int64),
                            np.full(be.sum(), EE, dtype=np.int64)])
    quads = np.concatenate([vf[bv], ee[be]], axis=0).reshape(-1, 4)
    tois = np.concatenate([t_vf[bv], t_ee[be]])
    return alpha, kinds, quads, tois
