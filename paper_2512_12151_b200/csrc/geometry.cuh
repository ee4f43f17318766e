// Pair distances and additive CCD on the device, bit-identical to the
// reference's numpy evaluation (intact/distance.py, intact/ccd.py).
//
// Every multiply/add/sub goes through __dmul_rn/__dadd_rn/__dsub_rn so the
// compiler can never contract them into FMAs, whatever -fmad says; division
// and sqrt are IEEE round-to-nearest in CUDA double precision, like numpy.
// Reduction orders follow what numpy 2.3 does on the build host (probed, see
// oracle/__init__.py): 3-term dot = (u0 v0 + u2 v2) + u1 v1, norms and small
// sums sequential, mean of 3 = ((a+b)+c)/3.
#pragma once

#include <math.h>

namespace ibf {
namespace geo {

struct V3 {
  double x, y, z;
};

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return {sub(a.x, b.x), sub(a.y, b.y), sub(a.z, b.z)}; }
__device__ __forceinline__ V3 vadd(V3 a, V3 b) { return {add(a.x, b.x), add(a.y, b.y), add(a.z, b.z)}; }
__device__ __forceinline__ V3 vscale(double s, V3 a) { return {mul(s, a.x), mul(s, a.y), mul(s, a.z)}; }
// einsum('...k,...k->...') order on the build host
__device__ __forceinline__ double dot3(V3 u, V3 v) { return add(add(mul(u.x, v.x), mul(u.z, v.z)), mul(u.y, v.y)); }
// np.linalg.norm(axis=-1): sequential sum of squares
__device__ __forceinline__ double norm3(V3 u) { return sqrt(add(add(mul(u.x, u.x), mul(u.y, u.y)), mul(u.z, u.z))); }

// np.maximum / np.minimum: NaN propagates (first NaN operand wins)
__device__ __forceinline__ double np_max(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}
__device__ __forceinline__ double np_min(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a <= b ? a : b;
}
__device__ __forceinline__ double clip01(double t) { return np_min(np_max(t, 0.0), 1.0); }

__device__ __forceinline__ V3 ld3(const double* p) { return {p[0], p[1], p[2]}; }

// point_triangle_weights (intact/distance.py:47-101): first matching region wins.
__device__ __forceinline__ void triangle_weights(V3 p, V3 a, V3 b, V3 c, double w[3]) {
  const V3 ab = vsub(b, a), ac = vsub(c, a);
  const V3 ap = vsub(p, a);
  const double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  const V3 bp = vsub(p, b);
  const double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  const V3 cp = vsub(p, c);
  const double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  const double vc = sub(mul(d1, d4), mul(d3, d2));
  const double vb = sub(mul(d5, d2), mul(d1, d6));
  const double va = sub(mul(d3, d6), mul(d5, d4));
  if (d1 <= 0.0 && d2 <= 0.0) { w[0] = 1.0; w[1] = 0.0; w[2] = 0.0; return; }
  if (d3 >= 0.0 && d4 <= d3) { w[0] = 0.0; w[1] = 1.0; w[2] = 0.0; return; }
  if (d6 >= 0.0 && d5 <= d6) { w[0] = 0.0; w[1] = 0.0; w[2] = 1.0; return; }
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    const double v = (d1 != d3) ? d1 / sub(d1, d3) : 0.0;
    w[0] = sub(1.0, v); w[1] = v; w[2] = 0.0; return;
  }
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    const double v = (d2 != d6) ? d2 / sub(d2, d6) : 0.0;
    w[0] = sub(1.0, v); w[1] = 0.0; w[2] = v; return;
  }
  if (va <= 0.0 && d4 >= d3 && d5 >= d6) {
    const double num = sub(d4, d3);
    const double den = add(sub(d4, d3), sub(d5, d6));
    const double v = (den != 0.0) ? num / den : 0.0;
    w[0] = 0.0; w[1] = sub(1.0, v); w[2] = v; return;
  }
  const double tot = add(add(va, vb), vc);
  const double v = (tot != 0.0) ? vb / tot : 1.0 / 3.0;
  const double u = (tot != 0.0) ? vc / tot : 1.0 / 3.0;
  w[0] = sub(sub(1.0, v), u); w[1] = v; w[2] = u;
}

// segment_segment_params (intact/distance.py:108-150), near-parallel fallback
// included, argmin ties to the first candidate.
__device__ __forceinline__ void segment_params(V3 p1, V3 p2, V3 q1, V3 q2, double& s, double& t) {
  const V3 d1 = vsub(p2, p1), d2 = vsub(q2, q1), r = vsub(p1, q1);
  const double a = dot3(d1, d1), e = dot3(d2, d2), b = dot3(d1, d2);
  const double c = dot3(d1, r), f = dot3(d2, r);
  const double a_s = np_max(a, 1e-300), e_s = np_max(e, 1e-300);
  const double den = sub(mul(a, e), mul(b, b));
  s = (den > 0.0) ? clip01(sub(mul(b, f), mul(c, e)) / np_max(den, 1e-300)) : 0.0;
  const double t_raw = add(mul(b, s), f) / e_s;
  t = clip01(t_raw);
  if (t_raw < 0.0) s = clip01(-c / a_s);
  if (t_raw > 1.0) s = clip01(sub(b, c) / a_s);
  const V3 cr = {sub(mul(d1.y, d2.z), mul(d1.z, d2.y)), sub(mul(d1.z, d2.x), mul(d1.x, d2.z)),
                 sub(mul(d1.x, d2.y), mul(d1.y, d2.x))};
  if (norm3(cr) < mul(1e-10, sqrt(mul(a, e)))) {
    const double cs[4] = {0.0, 1.0, clip01(-c / a_s), clip01(sub(b, c) / a_s)};
    const double ct[4] = {clip01(f / e_s), clip01(add(f, b) / e_s), 0.0, 1.0};
    double best_d = 0.0;
    int best = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const V3 pa = vadd(p1, vscale(cs[k], d1));
      const V3 pb = vadd(q1, vscale(ct[k], d2));
      const V3 df = vsub(pa, pb);
      const double d2s = add(add(mul(df.x, df.x), mul(df.y, df.y)), mul(df.z, df.z));
      if (k == 0) {
        best_d = d2s;
      } else if (best_d == best_d && (d2s != d2s || d2s < best_d)) {
        best = k;
        best_d = d2s;
      }
    }
    s = cs[best];
    t = ct[best];
  }
}

// Witness difference (side A minus side B) and signed weights of a pair.
__device__ __forceinline__ V3 witness(int kind, const V3 P[4], double wts[4]) {
  if (kind == 0) {
    double w[3];
    triangle_weights(P[0], P[1], P[2], P[3], w);
    const V3 cl = {add(add(mul(w[0], P[1].x), mul(w[1], P[2].x)), mul(w[2], P[3].x)),
                   add(add(mul(w[0], P[1].y), mul(w[1], P[2].y)), mul(w[2], P[3].y)),
                   add(add(mul(w[0], P[1].z), mul(w[1], P[2].z)), mul(w[2], P[3].z))};
    wts[0] = 1.0; wts[1] = -w[0]; wts[2] = -w[1]; wts[3] = -w[2];
    return vsub(P[0], cl);
  }
  double s, t;
  segment_params(P[0], P[1], P[2], P[3], s, t);
  const V3 pa = vadd(P[0], vscale(s, vsub(P[1], P[0])));
  const V3 pb = vadd(P[2], vscale(t, vsub(P[3], P[2])));
  wts[0] = sub(1.0, s); wts[1] = s; wts[2] = -sub(1.0, t); wts[3] = -t;
  return vsub(pa, pb);
}

__device__ __forceinline__ double pair_dist(int kind, const V3 P[4]) {
  double wts[4];
  return norm3(witness(kind, P, wts));
}

// vf_eval / ee_eval + _finish (intact/distance.py:153-189)
__device__ __forceinline__ double pair_eval(int kind, const V3 P[4], double grad[12], double wts[4],
                                            bool& degenerate) {
  const V3 df = witness(kind, P, wts);
  const double d = norm3(df);
  double scale = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    scale = np_max(scale, fabs(P[k].x));
    scale = np_max(scale, fabs(P[k].y));
    scale = np_max(scale, fabs(P[k].z));
  }
  degenerate = d <= np_max(1e-30, mul(1e-12, scale));
  V3 u = {0.0, 0.0, 0.0};
  if (!degenerate) {
    const double dd = np_max(d, 1e-300);
    u = {df.x / dd, df.y / dd, df.z / dd};
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    grad[3 * k + 0] = mul(wts[k], u.x);
    grad[3 * k + 1] = mul(wts[k], u.y);
    grad[3 * k + 2] = mul(wts[k], u.z);
  }
  return d;
}

// Centered relative motion and its bound l_p (intact/ccd.py:24-34, :59-62).
__device__ __forceinline__ double accd_setup(int kind, const V3 X0[4], const V3 X1[4], V3 pm[4]) {
  V3 p[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) p[k] = vsub(X1[k], X0[k]);
  V3 ma, mb;
  if (kind == 0) {
    ma = p[0];
    const V3 s3 = vadd(vadd(p[1], p[2]), p[3]);
    mb = {s3.x / 3.0, s3.y / 3.0, s3.z / 3.0};
  } else {
    const V3 sa = vadd(p[0], p[1]), sb = vadd(p[2], p[3]);
    ma = {sa.x / 2.0, sa.y / 2.0, sa.z / 2.0};
    mb = {sb.x / 2.0, sb.y / 2.0, sb.z / 2.0};
  }
  const V3 m = vscale(0.5, vadd(ma, mb));
  double n[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    pm[k] = vsub(p[k], m);
    n[k] = norm3(pm[k]);
  }
  if (kind == 0) return add(n[0], np_max(np_max(n[1], n[2]), n[3]));
  return add(np_max(n[0], n[1]), np_max(n[2], n[3]));
}

// Classification of a candidate before advancement: 0 -> TOI 0, 1 -> TOI 1,
// 2 -> needs the iteration (intact/ccd.py:64-68).
__device__ __forceinline__ int accd_class(int kind, const V3 X0[4], const V3 X1[4], double min_gap) {
  V3 pm[4];
  const double lp = accd_setup(kind, X0, X1, pm);
  const double gap0 = sub(pair_dist(kind, X0), min_gap);
  if (gap0 <= 0.0) return 0;
  if (gap0 > 0.0 && lp >= gap0) return 2;
  return 1;
}

// Conservative TOI of one pair, the scalar recurrence of accd_batch
// (intact/ccd.py:37-91).
__device__ __forceinline__ double accd_toi(int kind, const V3 X0[4], const V3 X1[4], double min_gap) {
  V3 pm[4];
  const double lp = accd_setup(kind, X0, X1, pm);
  const double gap0 = sub(pair_dist(kind, X0), min_gap);
  if (gap0 <= 0.0) return 0.0;
  if (!(gap0 > 0.0 && lp >= gap0)) return 1.0;
  V3 X[4] = {X0[0], X0[1], X0[2], X0[3]};
  const double slack = mul(0.1, gap0);
  double t = 0.0;
  double tl = mul(0.9, gap0) / lp;
  for (int it = 0; it < 100; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) X[k] = vadd(X[k], vscale(tl, pm[k]));
    const double gap = sub(pair_dist(kind, X), min_gap);
    if (t > 0.0 && gap < slack) return t;
    t = add(t, tl);
    if (t >= 1.0) return 1.0;
    tl = mul(0.9, gap) / lp;
  }
  return t;
}

}  // namespace geo
}  // namespace ibf
