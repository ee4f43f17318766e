// Per-tetrahedron elasticity math in FP64 registers: deformation gradient,
// rotation-variant 3x3 SVD, energy density, PK1 stress and the analytic
// 9-mode eigensystem feeding the PSD 12x12 vertex-block Hessian.
//
// Follows intact/elasticity.py (paths relative to /root/reference/pkg/src):
// svd_rotation_variant :83-97, energy_density :108-132, pk1 :140-164,
// eigen_system :188-249, assemble_vertex_blocks :286-299.  LAPACK is replaced
// by a one-sided Jacobi SVD and a cyclic Jacobi 3x3 eigensolver; parity with
// the reference is to FP64 rounding (the block Hessian is basis invariant).
#pragma once

#include <math.h>

namespace ibf {
namespace el {

struct M3 {
  double m[3][3];
};

__device__ __forceinline__ double det3(const M3& F) {
  return F.m[0][0] * (F.m[1][1] * F.m[2][2] - F.m[1][2] * F.m[2][1]) -
         F.m[0][1] * (F.m[1][0] * F.m[2][2] - F.m[1][2] * F.m[2][0]) +
         F.m[0][2] * (F.m[1][0] * F.m[2][1] - F.m[1][1] * F.m[2][0]);
}

// cofactor (intact/elasticity.py:75-80): column k = cross of the other two columns
__device__ __forceinline__ M3 cofactor(const M3& F) {
  M3 C;
  // col0 = c1 x c2, col1 = c2 x c0, col2 = c0 x c1  (c_j = column j)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int a = (k + 1) % 3, b = (k + 2) % 3;
    C.m[0][k] = F.m[1][a] * F.m[2][b] - F.m[2][a] * F.m[1][b];
    C.m[1][k] = F.m[2][a] * F.m[0][b] - F.m[0][a] * F.m[2][b];
    C.m[2][k] = F.m[0][a] * F.m[1][b] - F.m[1][a] * F.m[0][b];
  }
  return C;
}

// F = sum_k x_k (x) A_k, summed in k order (intact/elasticity.py:66-68)
__device__ __forceinline__ M3 def_grad(const double X[4][3], const double A[4][3]) {
  M3 F;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double v = X[0][a] * A[0][b];
      v = v + X[1][a] * A[1][b];
      v = v + X[2][a] * A[2][b];
      v = v + X[3][a] * A[3][b];
      F.m[a][b] = v;
    }
  return F;
}

// Rotation-variant SVD F = U diag(s) V^T with det U = det V = +1,
// s0 >= s1 >= |s2|, reflection folded into s2 (intact/elasticity.py:83-97).
// One-sided (Hestenes) Jacobi on the columns of F V.
__device__ __forceinline__ void svd_rv(const M3& F, M3& U, double s[3], M3& V) {
  double B[3][3], W[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      B[i][j] = F.m[i][j];
      W[i][j] = (i == j) ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 12; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int pair = 0; pair < 3; ++pair) {
      const int p = pair == 2 ? 1 : 0;
      const int q = pair == 0 ? 1 : 2;
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        al += B[i][p] * B[i][p];
        be += B[i][q] * B[i][q];
        ga += B[i][p] * B[i][q];
      }
      if (fabs(ga) > 1e-15 * sqrt(al * be) && ga != 0.0) {
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double sn = c * t;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double bp = B[i][p], bq = B[i][q];
          B[i][p] = c * bp - sn * bq;
          B[i][q] = sn * bp + c * bq;
          const double wp = W[i][p], wq = W[i][q];
          W[i][p] = c * wp - sn * wq;
          W[i][q] = sn * wp + c * wq;
        }
      }
    }
    if (!rotated) break;
  }
  double nrm[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) nrm[j] = sqrt(B[0][j] * B[0][j] + B[1][j] * B[1][j] + B[2][j] * B[2][j]);
  // sort columns by descending norm (3-element network), keeping B, W aligned
  int o[3] = {0, 1, 2};
  if (nrm[o[0]] < nrm[o[1]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
  if (nrm[o[1]] < nrm[o[2]]) { int t = o[1]; o[1] = o[2]; o[2] = t; }
  if (nrm[o[0]] < nrm[o[1]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
  double Bs[3][3];
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      Bs[i][j] = B[i][o[j]];
      V.m[i][j] = W[i][o[j]];
    }
  // proper rotation V: flip the third column if det V < 0 (B follows: B = F V)
  if (det3(V) < 0.0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      V.m[i][2] = -V.m[i][2];
      Bs[i][2] = -Bs[i][2];
    }
  }
  const double s0 = sqrt(Bs[0][0] * Bs[0][0] + Bs[1][0] * Bs[1][0] + Bs[2][0] * Bs[2][0]);
  const double s1 = sqrt(Bs[0][1] * Bs[0][1] + Bs[1][1] * Bs[1][1] + Bs[2][1] * Bs[2][1]);
  double u0[3], u1[3], u2[3];
  if (s0 > 0.0) {
    for (int i = 0; i < 3; ++i) u0[i] = Bs[i][0] / s0;
  } else {
    u0[0] = 1.0; u0[1] = 0.0; u0[2] = 0.0;
  }
  if (s1 > 1e-300 * (1.0 + s0) && s1 > 0.0) {
    for (int i = 0; i < 3; ++i) u1[i] = Bs[i][1] / s1;
    // re-orthogonalise against u0 (tiny cleanup for clustered singular values)
    const double d = u0[0] * u1[0] + u0[1] * u1[1] + u0[2] * u1[2];
    for (int i = 0; i < 3; ++i) u1[i] -= d * u0[i];
    const double n1 = sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
    for (int i = 0; i < 3; ++i) u1[i] /= n1;
  } else {
    // any unit vector orthogonal to u0
    const int k = (fabs(u0[0]) <= fabs(u0[1]) && fabs(u0[0]) <= fabs(u0[2])) ? 0 : (fabs(u0[1]) <= fabs(u0[2]) ? 1 : 2);
    double e[3] = {0.0, 0.0, 0.0};
    e[k] = 1.0;
    u1[0] = u0[1] * e[2] - u0[2] * e[1];
    u1[1] = u0[2] * e[0] - u0[0] * e[2];
    u1[2] = u0[0] * e[1] - u0[1] * e[0];
    const double n1 = sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
    for (int i = 0; i < 3; ++i) u1[i] /= n1;
  }
  u2[0] = u0[1] * u1[2] - u0[2] * u1[1];
  u2[1] = u0[2] * u1[0] - u0[0] * u1[2];
  u2[2] = u0[0] * u1[1] - u0[1] * u1[0];
  s[0] = s0;
  s[1] = s1;
  s[2] = u2[0] * Bs[0][2] + u2[1] * Bs[1][2] + u2[2] * Bs[2][2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    U.m[i][0] = u0[i];
    U.m[i][1] = u1[i];
    U.m[i][2] = u2[i];
  }
}

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3: A = Q diag(ev) Q^T,
// Q columns are eigenvectors.
__device__ __forceinline__ void eig_sym3(const double Ain[3][3], double ev[3], double Q[3][3]) {
  double A[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      A[i][j] = Ain[i][j];
      Q[i][j] = (i == j) ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 16; ++sweep) {
    const double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
    const double dia = fabs(A[0][0]) + fabs(A[1][1]) + fabs(A[2][2]);
    if (off <= 1e-17 * dia || off == 0.0) break;
#pragma unroll
    for (int pair = 0; pair < 3; ++pair) {
      const int p = pair == 2 ? 1 : 0;
      const int q = pair == 0 ? 1 : 2;
      const double apq = A[p][q];
      if (apq == 0.0) continue;
      const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
      const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0);
      const double sn = t * c;
      // A <- J^T A J with J the (p,q) rotation
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double akp = A[k][p], akq = A[k][q];
        A[k][p] = c * akp - sn * akq;
        A[k][q] = sn * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double apk = A[p][k], aqk = A[q][k];
        A[p][k] = c * apk - sn * aqk;
        A[q][k] = sn * apk + c * aqk;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double qkp = Q[k][p], qkq = Q[k][q];
        Q[k][p] = c * qkp - sn * qkq;
        Q[k][q] = sn * qkp + c * qkq;
      }
    }
  }
  ev[0] = A[0][0];
  ev[1] = A[1][1];
  ev[2] = A[2][2];
}

enum { SNH = 0, NH = 1, COR = 2, LIN = 3 };

// Energy density per rest volume; NH is +inf for det F <= 0 (:108-132).
__device__ __forceinline__ double psi(int model, double mu, double lam, const M3& F) {
  if (model == LIN) {
    double e2 = 0.0, tr = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double eij = 0.5 * (F.m[i][j] + F.m[j][i]) - (i == j ? 1.0 : 0.0);
        e2 += eij * eij;
        if (i == j) tr += eij;
      }
    return mu * e2 + 0.5 * lam * tr * tr;
  }
  if (model == COR) {
    M3 U, V;
    double s[3];
    svd_rv(F, U, s, V);
    double d2 = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double r = U.m[i][0] * V.m[j][0] + U.m[i][1] * V.m[j][1] + U.m[i][2] * V.m[j][2];
        const double d = F.m[i][j] - r;
        d2 += d * d;
      }
    const double tr = (s[0] + s[1] + s[2]) - 3.0;
    return mu * d2 + 0.5 * lam * tr * tr;
  }
  double ic = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) ic += F.m[i][j] * F.m[i][j];
  const double J = det3(F);
  if (model == SNH) return 0.5 * mu * (ic - 3.0) - mu * (J - 1.0) + 0.5 * lam * (J - 1.0) * (J - 1.0);
  if (!(J > 0.0)) return INFINITY;
  const double lj = log(J);
  return 0.5 * mu * (ic - 3.0) - mu * lj + 0.5 * lam * lj * lj;
}

// First Piola-Kirchhoff stress (:140-164). For COR the SVD is passed in.
__device__ __forceinline__ M3 pk1(int model, double mu, double lam, const M3& F, const M3& U,
                                  const double s[3], const M3& V) {
  M3 P;
  if (model == LIN) {
    const double tr = (F.m[0][0] - 1.0) + (F.m[1][1] - 1.0) + (F.m[2][2] - 1.0);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        P.m[i][j] = 2.0 * mu * (0.5 * (F.m[i][j] + F.m[j][i]) - (i == j ? 1.0 : 0.0)) + (i == j ? lam * tr : 0.0);
    return P;
  }
  if (model == COR) {
    const double tr = (s[0] + s[1] + s[2]) - 3.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double r = U.m[i][0] * V.m[j][0] + U.m[i][1] * V.m[j][1] + U.m[i][2] * V.m[j][2];
        P.m[i][j] = 2.0 * mu * (F.m[i][j] - r) + lam * tr * r;
      }
    return P;
  }
  const double J = det3(F);
  const M3 C = cofactor(F);
  const double k = (model == SNH) ? (lam * (J - 1.0) - mu) : (lam * log(J) - mu) / J;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) P.m[i][j] = mu * F.m[i][j] + k * C.m[i][j];
  return P;
}

// Clamped scaling-mode kernel W = sum_k max(l_k,0) e_k e_k^T and clamped
// twist/flip eigenvalues (eigen_system :188-249 + _clamped :270-271).
__device__ __forceinline__ void mode_weights(int model, double mu, double lam, const double s[3],
                                             double W[3][3], double twist[3], double flip[3]) {
  double A[3][3];
  bool psd_known = false;
  if (model == LIN || model == COR) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) A[i][j] = (i == j ? 2.0 * mu : 0.0) + lam;
    psd_known = true;  // eigenvalues 2mu, 2mu, 2mu + 3 lam >= 0
    for (int k = 0; k < 3; ++k) flip[k] = 2.0 * mu;
    if (model == LIN) {
      for (int k = 0; k < 3; ++k) twist[k] = 0.0;
    } else {
      const double num = 2.0 * lam * ((s[0] + s[1] + s[2]) - 3.0) - 4.0 * mu;
      twist[0] = 2.0 * mu + num / fmax(s[0] + s[1], 1e-8);
      twist[1] = 2.0 * mu + num / fmax(s[0] + s[2], 1e-8);
      twist[2] = 2.0 * mu + num / fmax(s[1] + s[2], 1e-8);
    }
  } else if (model == SNH) {
    const double J = s[0] * s[1] * s[2];
    const double g[3] = {s[1] * s[2], s[0] * s[2], s[0] * s[1]};
    const double kj = lam * (J - 1.0) - mu;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) A[i][j] = (i == j) ? mu + lam * g[i] * g[i] : lam * g[i] * g[j];
    A[0][1] += kj * s[2]; A[1][0] += kj * s[2];
    A[0][2] += kj * s[1]; A[2][0] += kj * s[1];
    A[1][2] += kj * s[0]; A[2][1] += kj * s[0];
    const double other[3] = {s[2], s[1], s[0]};
    for (int k = 0; k < 3; ++k) {
      twist[k] = mu + kj * other[k];
      flip[k] = mu - kj * other[k];
    }
  } else {  // NH
    const double J = s[0] * s[1] * s[2];
    const double m = lam * log(fabs(J)) - mu;
    const double inv[3] = {1.0 / s[0], 1.0 / s[1], 1.0 / s[2]};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) A[i][j] = (i == j) ? mu + (lam - m) * inv[i] * inv[i] : lam * inv[i] * inv[j];
    const double pp[3] = {s[0] * s[1], s[0] * s[2], s[1] * s[2]};
    for (int k = 0; k < 3; ++k) {
      twist[k] = mu + m / pp[k];
      flip[k] = mu - m / pp[k];
    }
  }
  for (int k = 0; k < 3; ++k) {
    twist[k] = fmax(twist[k], 0.0);
    flip[k] = fmax(flip[k], 0.0);
  }
  if (psd_known) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) W[i][j] = A[i][j];
    return;
  }
  double ev[3], Q[3][3];
  eig_sym3(A, ev, Q);
  if (ev[0] >= 0.0 && ev[1] >= 0.0 && ev[2] >= 0.0) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) W[i][j] = A[i][j];
    return;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      W[i][j] = fmax(ev[0], 0.0) * Q[i][0] * Q[j][0] + fmax(ev[1], 0.0) * Q[i][1] * Q[j][1] +
                fmax(ev[2], 0.0) * Q[i][2] * Q[j][2];
}

// One PSD 3x3 vertex block K_ij (assemble_vertex_blocks :286-299) times scale.
// y_i = V^T A_i; M = y_i y_j^T; S = W o M (+ twist/flip pair terms); K = U S U^T.
__device__ __forceinline__ void vertex_block(const double yi[3], const double yj[3], const double W[3][3],
                                             const double twist[3], const double flip[3], const M3& U,
                                             double scale, double K[9]) {
  double Mm[3][3], S[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      Mm[a][b] = yi[a] * yj[b];
      S[a][b] = W[a][b] * Mm[a][b];
    }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int p = k == 2 ? 1 : 0;
    const int q = k == 0 ? 1 : 2;
    const double lt = 0.5 * twist[k], lf = 0.5 * flip[k];
    S[p][p] += (lt + lf) * Mm[q][q];
    S[q][q] += (lt + lf) * Mm[p][p];
    S[p][q] += (lf - lt) * Mm[q][p];
    S[q][p] += (lf - lt) * Mm[p][q];
  }
  double T[3][3];  // T = U S
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int b = 0; b < 3; ++b) T[r][b] = U.m[r][0] * S[0][b] + U.m[r][1] * S[1][b] + U.m[r][2] * S[2][b];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      K[3 * r + c] = scale * (T[r][0] * U.m[c][0] + T[r][1] * U.m[c][1] + T[r][2] * U.m[c][2]);
}

}  // namespace el
}  // namespace ibf
