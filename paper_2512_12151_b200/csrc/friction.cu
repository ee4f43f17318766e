// Semi-implicit smoothed Coulomb friction on the device.
//
// Replaces (paths relative to /root/reference/pkg/src):
//   friction_precompute          intact/friction.py:103-151
//   FrictionTerms energy / gradient_terms / hessian_grids
//                                intact/friction.py:56-100
//   f0 / f0_over_y / f0_second   intact/friction.py:26-42
//   tangent_basis                intact/friction.py:45-53
//
// Terms are frozen at the end of an accepted step (one per constraint with a
// positive normal force, in active-set order) and enter the next step's
// assembly, energy and SpMV matrix-free: per term, a slip u = T^T (sum w x -
// ref), a 3-vector force T f0'(|u|)/|u| u coeff and a 3x3 PSD world Hessian,
// scattered through a vertex -> term incidence (fixed order, no atomics).
#include <cub/cub.cuh>

#include <algorithm>

#include "geometry.cuh"
#include "system.cuh"

namespace ibf {

__device__ __forceinline__ double fr_f0(double y, double eps) {
  return y >= eps ? y : -(y * y * y) / (3.0 * eps * eps) + y * y / eps + eps / 3.0;
}
__device__ __forceinline__ double fr_f0_over_y(double y, double eps) {
  if (y >= eps) return y > 0.0 ? 1.0 / fmax(y, 1e-300) : 0.0;
  return (2.0 * eps - y) / (eps * eps);
}
__device__ __forceinline__ double fr_f0_second(double y, double eps) {
  return y >= eps ? 0.0 : 2.0 * (eps - y) / (eps * eps);
}

// friction_precompute per constraint: keep flag + the term in slot c
__global__ void k_fr_terms(int64_t n, const int* __restrict__ kind, const int* __restrict__ quad,
                           const double* __restrict__ lam, const double* __restrict__ x, double mu, double offset,
                           double mu_f, int* __restrict__ keep, double* __restrict__ tw, double* __restrict__ tfr,
                           double* __restrict__ tcoeff, double* __restrict__ tref) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    geo::V3 P[4];
    int q[4];
    for (int k = 0; k < 4; ++k) {
      q[k] = quad[4 * c + k];
      P[k] = geo::ld3(x + 3 * (int64_t)q[k]);
    }
    double g[12], w[4];
    bool degen;
    const double d = geo::pair_eval(kind[c], P, g, w, degen);
    int ok = 0;
    if (!degen) {
      const double shifted = (d - offset) - lam[c] / mu;
      const double sl = fmax(0.0, shifted);
      const double force = fmax(0.0, -mu * (shifted - sl));
      if (force != 0.0) {
        ok = 1;
        int m = 0;
        for (int k = 1; k < 4; ++k)
          if (fabs(w[k]) > fabs(w[m])) m = k;   // np.argmax: first maximum
        double nx = g[3 * m] / w[m], ny = g[3 * m + 1] / w[m], nz = g[3 * m + 2] / w[m];
        const double nn = sqrt(nx * nx + ny * ny + nz * nz);
        nx /= nn; ny /= nn; nz /= nn;
        // tangent_basis: helper axis = first smallest |n| component
        const double an[3] = {fabs(nx), fabs(ny), fabs(nz)};
        const int a = (an[0] <= an[1] && an[0] <= an[2]) ? 0 : (an[1] <= an[2] ? 1 : 2);
        const double e[3] = {a == 0 ? 1.0 : 0.0, a == 1 ? 1.0 : 0.0, a == 2 ? 1.0 : 0.0};
        double t1x = ny * e[2] - nz * e[1], t1y = nz * e[0] - nx * e[2], t1z = nx * e[1] - ny * e[0];
        const double tn = sqrt(t1x * t1x + t1y * t1y + t1z * t1z);
        t1x /= tn; t1y /= tn; t1z /= tn;
        const double t2x = ny * t1z - nz * t1y, t2y = nz * t1x - nx * t1z, t2z = nx * t1y - ny * t1x;
        double* F = tfr + 6 * c;   // (3,2) row-major: [t1x t2x; t1y t2y; t1z t2z]
        F[0] = t1x; F[1] = t2x; F[2] = t1y; F[3] = t2y; F[4] = t1z; F[5] = t2z;
        for (int k = 0; k < 4; ++k) tw[4 * c + k] = w[k];
        tcoeff[c] = mu_f * force;
        double rx = 0.0, ry = 0.0, rz = 0.0;
        for (int k = 0; k < 4; ++k) {
          rx += w[k] * P[k].x;
          ry += w[k] * P[k].y;
          rz += w[k] * P[k].z;
        }
        tref[3 * c] = rx; tref[3 * c + 1] = ry; tref[3 * c + 2] = rz;
      }
    }
    keep[c] = ok;
  }
}

__global__ void k_fr_compact(int64_t n, const int* __restrict__ keep, const int* __restrict__ pos,
                             const int* __restrict__ quad, const double* __restrict__ tw,
                             const double* __restrict__ tfr, const double* __restrict__ tcoeff,
                             const double* __restrict__ tref, int* __restrict__ oquad, double* __restrict__ ow,
                             double* __restrict__ ofr, double* __restrict__ ocoeff, double* __restrict__ oref) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[c]) continue;
    const int64_t k = pos[c];
    for (int e = 0; e < 4; ++e) {
      oquad[4 * k + e] = quad[4 * c + e];
      ow[4 * k + e] = tw[4 * c + e];
    }
    for (int e = 0; e < 6; ++e) ofr[6 * k + e] = tfr[6 * c + e];
    ocoeff[k] = tcoeff[c];
    for (int e = 0; e < 3; ++e) oref[3 * k + e] = tref[3 * c + e];
  }
}

// slip of term k at y (= x_hat + r p when p is given)
__device__ __forceinline__ void fr_slip(const int* quad, const double* w, const double* fr, const double* ref,
                                        int64_t k, const double* xh, const double* p, double r, double u[2]) {
  double rel[3] = {0.0, 0.0, 0.0};
  for (int j = 0; j < 4; ++j) {
    const int64_t v = quad[4 * k + j];
    const double wj = w[4 * k + j];
    for (int c = 0; c < 3; ++c) {
      const double xc = p ? __dadd_rn(xh[3 * v + c], __dmul_rn(r, p[3 * v + c])) : xh[3 * v + c];
      rel[c] += wj * xc;
    }
  }
  for (int c = 0; c < 3; ++c) rel[c] -= ref[3 * k + c];
  const double* F = fr + 6 * k;
  u[0] = F[0] * rel[0] + F[2] * rel[1] + F[4] * rel[2];
  u[1] = F[1] * rel[0] + F[3] * rel[1] + F[5] * rel[2];
}

// per term at x_hat: world force (gradient direction) and world Hessian
__global__ void k_fr_prepare(int64_t n, const int* __restrict__ quad, const double* __restrict__ w,
                             const double* __restrict__ fr, const double* __restrict__ coeff,
                             const double* __restrict__ ref, double eps, const double* __restrict__ xh,
                             double* __restrict__ gw, double* __restrict__ hw) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double u[2];
    fr_slip(quad, w, fr, ref, k, xh, nullptr, 0.0, u);
    const double y = sqrt(u[0] * u[0] + u[1] * u[1]);
    const double g1 = fr_f0_over_y(y, eps), g2 = fr_f0_second(y, eps);
    const double cf = coeff[k];
    const double* F = fr + 6 * k;
    const double f0 = cf * g1 * u[0], f1 = cf * g1 * u[1];
    for (int c = 0; c < 3; ++c) gw[3 * k + c] = F[2 * c] * f0 + F[2 * c + 1] * f1;
    // h_u = g2 uhat + g1 (I - uhat), isotropic g1 I at vanishing slip
    double h00, h01, h11;
    if (y < 1e-12 * fmax(eps, 1e-300)) {
      h00 = h11 = g1;
      h01 = 0.0;
    } else {
      const double y2 = fmax(y * y, 1e-300);
      const double a = u[0] * u[0] / y2, b = u[0] * u[1] / y2, d = u[1] * u[1] / y2;
      h00 = g2 * a + g1 * (1.0 - a);
      h01 = g2 * b - g1 * b;
      h11 = g2 * d + g1 * (1.0 - d);
    }
    // Hw = coeff F h_u F^T
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        const double a0 = F[2 * i], a1 = F[2 * i + 1], b0 = F[2 * j], b1 = F[2 * j + 1];
        hw[9 * k + 3 * i + j] = cf * ((a0 * h00 + a1 * h01) * b0 + (a0 * h01 + a1 * h11) * b1);
      }
  }
}

__global__ void k_fr_incidence_keys(int64_t n, const int* __restrict__ quad, int* __restrict__ keys,
                                    int* __restrict__ vals, int* __restrict__ count) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 4 * n; e += (int64_t)gridDim.x * blockDim.x) {
    keys[e] = quad[e];
    vals[e] = (int)e;
    atomicAdd(count + quad[e], 1);
  }
}

static int fr_grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(div_up(n, 256), 148LL * 8)); }

static int fr_scan(ibf_friction* f, const int* in, int* out, int64_t n, cudaStream_t s) {
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, (int)n, s);
  IBF_TRY(f->cub_tmp.reserve(need + 16));
  size_t have = f->cub_tmp.cap;
  IBF_CUDA(cub::DeviceScan::ExclusiveSum(f->cub_tmp.p, have, in, out, (int)n, s));
  return IBF_OK;
}

int friction_build_incidence(ibf_friction* f, int64_t n_verts, cudaStream_t s) {
  if (f->vf_nverts == n_verts) return IBF_OK;
  const int64_t ne = 4 * f->n;
  IBF_TRY(f->vf_ptr.reserve(n_verts + 1));
  IBF_TRY(f->v_count.reserve(n_verts + 1));
  IBF_TRY(f->vf_src.reserve(std::max<int64_t>(ne, 1)));
  IBF_TRY(f->keys.reserve(std::max<int64_t>(ne, 1)));
  IBF_TRY(f->keys2.reserve(std::max<int64_t>(ne, 1)));
  IBF_TRY(f->vals.reserve(std::max<int64_t>(ne, 1)));
  IBF_CUDA(cudaMemsetAsync(f->v_count.p, 0, (n_verts + 1) * sizeof(int), s));
  if (ne) {
    k_fr_incidence_keys<<<fr_grid(ne), 256, 0, s>>>(f->n, f->quad.p, f->keys.p, f->vals.p, f->v_count.p);
    IBF_LAUNCH_CHECK();
    int bits = 1;
    while ((1LL << bits) < n_verts) ++bits;
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, f->keys.p, f->keys2.p, f->vals.p, f->vf_src.p, (int)ne, 0, bits,
                                    s);
    IBF_TRY(f->cub_tmp.reserve(need + 16));
    size_t have = f->cub_tmp.cap;
    IBF_CUDA(cub::DeviceRadixSort::SortPairs(f->cub_tmp.p, have, f->keys.p, f->keys2.p, f->vals.p, f->vf_src.p,
                                             (int)ne, 0, bits, s));
  }
  IBF_TRY(fr_scan(f, f->v_count.p, f->vf_ptr.p, n_verts + 1, s));
  f->vf_nverts = n_verts;
  return IBF_OK;
}

int friction_prepare(ibf_friction* f, const double* x_hat, cudaStream_t s) {
  if (!f->n) return IBF_OK;
  IBF_TRY(f->gw.reserve(3 * f->n));
  IBF_TRY(f->hw.reserve(9 * f->n));
  IBF_TRY(f->tvec.reserve(3 * f->n));
  k_fr_prepare<<<fr_grid(f->n), 256, 0, s>>>(f->n, f->quad.p, f->w.p, f->frames.p, f->coeff.p, f->ref.p, f->eps,
                                             x_hat, f->gw.p, f->hw.p);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

FrictionView friction_view(ibf_friction* f) {
  FrictionView v;
  v.n = (int)f->n;
  v.quad = f->quad.p;
  v.w = f->w.p;
  v.hw = f->hw.p;
  v.vf_ptr = f->vf_ptr.p;
  v.vf_src = f->vf_src.p;
  v.t = f->tvec.p;
  return v;
}

static int fr_reserve(ibf_friction* f, int64_t n) {
  const size_t m = (size_t)std::max<int64_t>(n, 1);
  IBF_TRY(f->quad.reserve(4 * m));
  IBF_TRY(f->w.reserve(4 * m));
  IBF_TRY(f->frames.reserve(6 * m));
  IBF_TRY(f->coeff.reserve(m));
  IBF_TRY(f->ref.reserve(3 * m));
  return IBF_OK;
}

}  // namespace ibf

using namespace ibf;

extern "C" int ibf_friction_create(ibf_friction** out) {
  if (!out) {
    set_error("ibf_friction_create: null out");
    return IBF_ERR_BAD_ARG;
  }
  *out = new ibf_friction();
  return IBF_OK;
}

extern "C" void ibf_friction_destroy(ibf_friction* f) { delete f; }

extern "C" int64_t ibf_friction_size(const ibf_friction* f) { return f ? f->n : 0; }

extern "C" int ibf_friction_precompute(ibf_friction* f, const ibf_contacts* c, const double* x, double mu,
                                       double offset, double h, double mu_f, double eps_v, int64_t* n_terms,
                                       ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  f->n = 0;
  f->vf_nverts = -1;
  f->eps = h * eps_v;
  *n_terms = 0;
  const int64_t n = c ? c->n : 0;
  if (mu_f <= 0.0 || n == 0) return IBF_OK;
  IBF_TRY(f->flags.reserve(n + 1));
  IBF_TRY(f->pos.reserve(n + 1));
  IBF_TRY(f->t_w.reserve(4 * n));
  IBF_TRY(f->t_frames.reserve(6 * n));
  IBF_TRY(f->t_coeff.reserve(n));
  IBF_TRY(f->t_ref.reserve(3 * n));
  k_fr_terms<<<fr_grid(n), 256, 0, s>>>(n, c->kind.p, c->quad.p, c->lam.p, x, mu, offset, mu_f, f->flags.p,
                                        f->t_w.p, f->t_frames.p, f->t_coeff.p, f->t_ref.p);
  IBF_LAUNCH_CHECK();
  IBF_CUDA(cudaMemsetAsync(f->flags.p + n, 0, sizeof(int), s));
  IBF_TRY(fr_scan(f, f->flags.p, f->pos.p, n + 1, s));
  IBF_TRY(f->host.reserve(16));
  int* hk = (int*)f->host.p;
  IBF_CUDA(cudaMemcpyAsync(hk, f->pos.p + n, sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  const int64_t k = hk[0];
  IBF_TRY(fr_reserve(f, k));
  if (k) {
    k_fr_compact<<<fr_grid(n), 256, 0, s>>>(n, f->flags.p, f->pos.p, c->quad.p, f->t_w.p, f->t_frames.p,
                                            f->t_coeff.p, f->t_ref.p, f->quad.p, f->w.p, f->frames.p, f->coeff.p,
                                            f->ref.p);
    IBF_LAUNCH_CHECK();
  }
  f->n = k;
  *n_terms = k;
  return IBF_OK;
}

extern "C" int ibf_friction_import(ibf_friction* f, int64_t n, const int64_t* quad, const double* w,
                                   const double* frames, const double* coeff, const double* ref, double eps,
                                   ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  if (n < 0) {
    set_error("ibf_friction_import: negative size");
    return IBF_ERR_BAD_ARG;
  }
  IBF_TRY(fr_reserve(f, n));
  std::vector<int> q(4 * n);
  for (int64_t k = 0; k < 4 * n; ++k) q[k] = (int)quad[k];
  if (n) {
    IBF_CUDA(cudaMemcpyAsync(f->quad.p, q.data(), 4 * n * sizeof(int), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(f->w.p, w, 4 * n * sizeof(double), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(f->frames.p, frames, 6 * n * sizeof(double), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(f->coeff.p, coeff, n * sizeof(double), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(f->ref.p, ref, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  IBF_CUDA(cudaStreamSynchronize(s));
  f->n = n;
  f->eps = eps;
  f->vf_nverts = -1;
  return IBF_OK;
}

extern "C" int ibf_friction_export(const ibf_friction* f, int64_t* quad, double* w, double* frames, double* coeff,
                                   double* ref, double* eps, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  const int64_t n = f->n;
  *eps = f->eps;
  if (!n) return IBF_OK;
  std::vector<int> q(4 * n);
  IBF_CUDA(cudaMemcpyAsync(q.data(), f->quad.p, 4 * n * sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(w, f->w.p, 4 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(frames, f->frames.p, 6 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(coeff, f->coeff.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(ref, f->ref.p, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  for (int64_t k = 0; k < 4 * n; ++k) quad[k] = q[k];
  return IBF_OK;
}

extern "C" int ibf_system_set_friction(ibf_system* s, ibf_friction* f) {
  s->friction = f;
  return IBF_OK;
}
