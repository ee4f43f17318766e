// Augmented-Lagrangian contact constraints on the device: the active set as
// insertion-ordered SoA, anchor refresh, AL coefficients, dual sweep, and the
// set maintenance of ActiveSet.update.
//
// Replaces (paths relative to /root/reference/pkg/src):
//   ActiveSet.update / admission_filter / constraint_key
//                              intact/contact.py:179-205, :144-151, :23-24
//   ActiveSet.refresh_anchors  intact/contact.py:207-235
//   ConstraintBatch values / gradient_terms / hessian_grids
//                              intact/contact.py:124-141
//   dual_update_sweep / dual_update / slack_update
//                              intact/contact.py:251-261, :91-106, :67-69
//
// Dedup keys are (kind, sorted quad).  Membership is answered through a CSR
// over a hash of the full key (buckets hold ~1 constraint), with exact key
// comparison inside a bucket, so the result does not depend on the hash;
// first-occurrence among new pairs picks the smallest blocking index, i.e.
// the reference's dict insertion order.  Pruning is a stable compaction, so the resident order is
// the reference's insertion order.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "geometry.cuh"
#include "system.cuh"

namespace ibf {

__device__ __forceinline__ void sort4(int v[4]) {
#define IBF_CSWAP(a, b)      \
  if (v[a] > v[b]) {         \
    const int t_ = v[a];     \
    v[a] = v[b];             \
    v[b] = t_;               \
  }
  IBF_CSWAP(0, 1) IBF_CSWAP(2, 3) IBF_CSWAP(0, 2) IBF_CSWAP(1, 3) IBF_CSWAP(1, 2)
#undef IBF_CSWAP
}

__device__ __forceinline__ void load_key(const int* quad, const int* kind, int64_t j, int key[5]) {
  int v[4] = {quad[4 * j], quad[4 * j + 1], quad[4 * j + 2], quad[4 * j + 3]};
  sort4(v);
  key[0] = kind[j];
  key[1] = v[0];
  key[2] = v[1];
  key[3] = v[2];
  key[4] = v[3];
}

// Membership buckets: constraints are bucketed by a hash of their full key
// (kind, sorted quad) into a power-of-two table.  (Bucketing by the smallest
// vertex degenerates when a pinned plate's few vertices are the smallest id
// of every pair against it: buckets of 10^4 entries, quadratic scans.)
__device__ __forceinline__ unsigned key_bucket(const int k[5], unsigned mask) {
  unsigned long long h = 0x9E3779B97F4A7C15ull;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    h ^= (unsigned long long)(unsigned)k[i] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h *= 0xBF58476D1CE4E5B9ull;
  }
  h ^= h >> 31;
  return (unsigned)h & mask;
}

__global__ void k_count_bucket(int64_t n, const int* __restrict__ quad, const int* __restrict__ kind,
                               const int* __restrict__ sel, unsigned mask, int* __restrict__ count) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    if (sel && !sel[j]) continue;
    int k[5];
    load_key(quad, kind, j, k);
    atomicAdd(count + key_bucket(k, mask), 1);
  }
}
__global__ void k_fill_bucket(int64_t n, const int* __restrict__ quad, const int* __restrict__ kind,
                              const int* __restrict__ sel, unsigned mask, const int* __restrict__ ptr,
                              int* __restrict__ cursor, int* __restrict__ list) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    if (sel && !sel[j]) continue;
    int k[5];
    load_key(quad, kind, j, k);
    const unsigned b = key_bucket(k, mask);
    list[ptr[b] + atomicAdd(cursor + b, 1)] = (int)j;
  }
}

// new[j] = key(blocking j) not resident
__global__ void k_new_flags(int64_t nb, const int* __restrict__ bkind, const int* __restrict__ bquad,
                            const int* __restrict__ rkind, const int* __restrict__ rquad, unsigned mask,
                            const int* __restrict__ rptr, const int* __restrict__ rlist, int* __restrict__ is_new) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
    int kj[5];
    load_key(bquad, bkind, j, kj);
    const unsigned bk = key_bucket(kj, mask);
    bool found = false;
    for (int e = rptr[bk]; e < rptr[bk + 1] && !found; ++e) {
      int kr[5];
      load_key(rquad, rkind, rlist[e], kr);
      found = kr[0] == kj[0] && kr[1] == kj[1] && kr[2] == kj[2] && kr[3] == kj[3] && kr[4] == kj[4];
    }
    is_new[j] = found ? 0 : 1;
  }
}

// admission_filter (intact/contact.py:144-151): per-vertex earliest TOI among new pairs
__global__ void k_earliest(int64_t nb, const int* __restrict__ bquad, const double* __restrict__ tois,
                           const int* __restrict__ is_new, double* __restrict__ earliest) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
    if (!is_new[j]) continue;
    for (int k = 0; k < 4; ++k) atomic_min_nonneg(earliest + bquad[4 * j + k], tois[j]);
  }
}
__global__ void k_admit(int64_t nb, const int* __restrict__ bquad, const double* __restrict__ tois,
                        const int* __restrict__ is_new, const double* __restrict__ earliest, int admit_all,
                        int* __restrict__ keep) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
    int k = 0;
    if (is_new[j]) {
      if (admit_all) {
        k = 1;
      } else {
        for (int e = 0; e < 4; ++e) k |= (tois[j] == earliest[bquad[4 * j + e]]) ? 1 : 0;
      }
    }
    keep[j] = k;
  }
}
__global__ void k_reset_earliest(int64_t nb, const int* __restrict__ bquad, double* __restrict__ earliest) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < 4; ++k) earliest[bquad[4 * j + k]] = INFINITY;
}
// first occurrence of each key among kept pairs (smallest blocking index)
__global__ void k_first(int64_t nb, const int* __restrict__ bkind, const int* __restrict__ bquad,
                        const int* __restrict__ keep, unsigned mask, const int* __restrict__ kptr,
                        const int* __restrict__ klist, int* __restrict__ append) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[j]) {
      append[j] = 0;
      continue;
    }
    int kj[5];
    load_key(bquad, bkind, j, kj);
    const unsigned bk = key_bucket(kj, mask);
    bool first = true;
    for (int e = kptr[bk]; e < kptr[bk + 1] && first; ++e) {
      const int o = klist[e];
      if (o >= j) continue;
      int ko[5];
      load_key(bquad, bkind, o, ko);
      first = !(ko[0] == kj[0] && ko[1] == kj[1] && ko[2] == kj[2] && ko[3] == kj[3] && ko[4] == kj[4]);
    }
    append[j] = first ? 1 : 0;
  }
}
__global__ void k_append(int64_t nb, int64_t base, const int* __restrict__ bkind, const int* __restrict__ bquad,
                         const int* __restrict__ append, const int* __restrict__ pos, int* __restrict__ kind,
                         int* __restrict__ quad, double* __restrict__ lam, double* __restrict__ gamma,
                         double* __restrict__ s, double* __restrict__ ad, double* __restrict__ ag,
                         double* __restrict__ ax) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
    if (!append[j]) continue;
    const int64_t c = base + pos[j];
    kind[c] = bkind[j];
    for (int k = 0; k < 4; ++k) quad[4 * c + k] = bquad[4 * j + k];
    lam[c] = 0.0;
    gamma[c] = 1.0;
    s[c] = 0.0;
    ad[c] = 0.0;
    for (int k = 0; k < 12; ++k) {
      ag[12 * c + k] = 0.0;
      ax[12 * c + k] = 0.0;
    }
  }
}

__global__ void k_keep_gamma(int64_t n, const double* __restrict__ gamma, int* __restrict__ keep) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    keep[c] = gamma[c] < 0.01 ? 0 : 1;   // GAMMA_PRUNE_THRESHOLD, intact/contact.py:20
}

template <typename T, int W>
__global__ void k_compact(int64_t n, const int* __restrict__ keep, const int* __restrict__ pos,
                          const T* __restrict__ src, T* __restrict__ dst) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[c]) continue;
    const int64_t d = pos[c];
    for (int k = 0; k < W; ++k) dst[W * d + k] = src[W * c + k];
  }
}

// refresh_anchors (intact/contact.py:207-235)
__global__ void k_refresh(int64_t n, const int* __restrict__ kind, const int* __restrict__ quad,
                          const double* __restrict__ x, double* __restrict__ ad, double* __restrict__ ag,
                          double* __restrict__ ax, int* __restrict__ n_degen) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    geo::V3 P[4];
    for (int k = 0; k < 4; ++k) P[k] = geo::ld3(x + 3 * (int64_t)quad[4 * c + k]);
    double g[12], w[4];
    bool degen;
    const double d = geo::pair_eval(kind[c], P, g, w, degen);
    if (degen) {
      atomicAdd(n_degen, 1);
      if (ad[c] <= 0.0) {  // never anchored: null anchor exerting no force
        for (int k = 0; k < 4; ++k) {
          ax[12 * c + 3 * k] = P[k].x;
          ax[12 * c + 3 * k + 1] = P[k].y;
          ax[12 * c + 3 * k + 2] = P[k].z;
        }
        for (int k = 0; k < 12; ++k) ag[12 * c + k] = 0.0;
        ad[c] = INFINITY;
      }
      continue;
    }
    ad[c] = d;
    for (int k = 0; k < 12; ++k) ag[12 * c + k] = g[k];
    for (int k = 0; k < 4; ++k) {
      ax[12 * c + 3 * k] = P[k].x;
      ax[12 * c + 3 * k + 1] = P[k].y;
      ax[12 * c + 3 * k + 2] = P[k].z;
    }
  }
}

// per-constraint AL coefficients at x_hat (ConstraintBatch, intact/contact.py:124-141)
__global__ void k_prepare(int64_t n, const int* __restrict__ quad, const double* __restrict__ ad,
                          const double* __restrict__ ag, const double* __restrict__ ax,
                          const double* __restrict__ lam, const double* __restrict__ gamma,
                          const double* __restrict__ x_hat, double mu, double offset, double* __restrict__ cval,
                          double* __restrict__ coef_g, double* __restrict__ coef_h) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    double dot = 0.0;
    for (int k = 0; k < 4; ++k) {
      const int64_t v = quad[4 * c + k];
      for (int e = 0; e < 3; ++e) dot += ag[12 * c + 3 * k + e] * (x_hat[3 * v + e] - ax[12 * c + 3 * k + e]);
    }
    const double cv = ad[c] + dot - offset;
    const double sh = cv - lam[c] / mu;
    const double mg = mu * gamma[c];
    cval[c] = cv;
    coef_g[c] = mg * (sh - fmax(0.0, sh));
    coef_h[c] = mg;
  }
}

// dual_update_sweep (intact/contact.py:251-261); the 12-term sum follows
// numpy's pairwise order so the s == 0 branch decisions match bit for bit.
__global__ void k_dual(int64_t n, const int* __restrict__ quad, const double* __restrict__ ad,
                       const double* __restrict__ ag, const double* __restrict__ ax, const double* __restrict__ x_hat,
                       double offset, double mu, double decay, double* __restrict__ lam, double* __restrict__ gamma,
                       double* __restrict__ s, double* __restrict__ worst) {
  __shared__ double red[8];
  double wmax = 0.0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    double q[12];
    for (int k = 0; k < 4; ++k) {
      const int64_t v = quad[4 * c + k];
      for (int e = 0; e < 3; ++e)
        q[3 * k + e] = geo::mul(ag[12 * c + 3 * k + e], geo::sub(x_hat[3 * v + e], ax[12 * c + 3 * k + e]));
    }
    using geo::add;
    double acc = add(add(add(q[0], q[1]), add(q[2], q[3])), add(add(q[4], q[5]), add(q[6], q[7])));
    for (int k = 8; k < 12; ++k) acc = add(acc, q[k]);
    const double cv = geo::sub(add(ad[c], acc), offset);
    const double sl = geo::np_max(0.0, geo::sub(cv, lam[c] / mu));
    s[c] = sl;
    if (sl == 0.0) {
      lam[c] = geo::sub(lam[c], geo::mul(mu, cv));
      gamma[c] = 1.0;
      wmax = fmax(wmax, fabs(cv));
    } else {
      lam[c] = 0.0;
      gamma[c] = geo::mul(decay, gamma[c]);
    }
  }
  wmax = block_max(wmax, red);
  if (threadIdx.x == 0) atomic_max_nonneg(worst, wmax);
}

__global__ void k_incidence_keys(int64_t n, const int* __restrict__ quad, int* __restrict__ keys,
                                 int* __restrict__ vals, int* __restrict__ count) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 4 * n; e += (int64_t)gridDim.x * blockDim.x) {
    keys[e] = quad[e];
    vals[e] = (int)e;  // c*4 + slot
    atomicAdd(count + quad[e], 1);
  }
}

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(div_up(n, 256), 148LL * 8)); }

static int exclusive_scan(ibf_contacts* c, const int* in, int* out, int64_t n, cudaStream_t s) {
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, (int)n, s);
  IBF_TRY(c->cub_tmp.reserve(need + 16));
  size_t have = c->cub_tmp.cap;
  IBF_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, have, in, out, (int)n, s));
  return IBF_OK;
}

// CSR of the selected rows' keys over a hash table of 2^k >= 2 n buckets
static int key_csr(ibf_contacts* c, int64_t n, const int* quad, const int* kind, const int* sel, DevBuf<int>& count,
                   DevBuf<int>& ptr, DevBuf<int>& list, unsigned* mask_out, cudaStream_t s) {
  int64_t nbk = 1;
  while (nbk < 2 * std::max<int64_t>(n, 1)) nbk <<= 1;
  const unsigned mask = (unsigned)(nbk - 1);
  *mask_out = mask;
  IBF_TRY(count.reserve(nbk + 1));
  IBF_TRY(ptr.reserve(nbk + 1));
  IBF_TRY(list.reserve(std::max<int64_t>(n, 1)));
  IBF_CUDA(cudaMemsetAsync(count.p, 0, (nbk + 1) * sizeof(int), s));
  if (n) {
    k_count_bucket<<<grid_for(n), 256, 0, s>>>(n, quad, kind, sel, mask, count.p);
    IBF_LAUNCH_CHECK();
  }
  IBF_TRY(exclusive_scan(c, count.p, ptr.p, nbk + 1, s));
  IBF_CUDA(cudaMemsetAsync(count.p, 0, (nbk + 1) * sizeof(int), s));
  if (n) {
    k_fill_bucket<<<grid_for(n), 256, 0, s>>>(n, quad, kind, sel, mask, ptr.p, count.p, list.p);
    IBF_LAUNCH_CHECK();
  }
  return IBF_OK;
}

static int reserve_soa(ibf_contacts* c, int64_t want, cudaStream_t s) {
  const int64_t used = c->n;
  IBF_TRY(c->kind.grow_keep(want, used, s));
  IBF_TRY(c->quad.grow_keep(4 * want, 4 * used, s));
  IBF_TRY(c->lam.grow_keep(want, used, s));
  IBF_TRY(c->gamma.grow_keep(want, used, s));
  IBF_TRY(c->s.grow_keep(want, used, s));
  IBF_TRY(c->anchor_d.grow_keep(want, used, s));
  IBF_TRY(c->anchor_grad.grow_keep(12 * want, 12 * used, s));
  IBF_TRY(c->anchor_x.grow_keep(12 * want, 12 * used, s));
  return IBF_OK;
}

// Stable compaction of one SoA field through the handle's scratch buffer
// (compacted into scratch, copied back): no allocation per prune, and the
// field keeps its capacity.
template <typename T, int W>
static int compact_field(ibf_contacts* c, DevBuf<T>& field, int64_t n, int64_t n_new, cudaStream_t s) {
  const size_t bytes = (size_t)W * std::max<int64_t>(n_new, 1) * sizeof(T);
  IBF_TRY(c->compact_tmp.reserve(div_up((int64_t)W * n * sizeof(T), 8) + 1));
  T* tmp = reinterpret_cast<T*>(c->compact_tmp.p);
  k_compact<T, W><<<grid_for(n), 256, 0, s>>>(n, c->flags.p, c->pos.p, field.p, tmp);
  IBF_LAUNCH_CHECK();
  if (n_new) IBF_CUDA(cudaMemcpyAsync(field.p, tmp, bytes, cudaMemcpyDeviceToDevice, s));
  return IBF_OK;
}

// ActiveSet.update on device arrays (blocking kinds/quads int32, tois)
int contacts_update_dev(ibf_contacts* c, int64_t nb, const int* bkind, const int* bquad, const double* btoi,
                        int64_t* admitted, int64_t* pruned, cudaStream_t s) {
  int* hostc = nullptr;
  IBF_TRY(c->host.reserve(64));
  hostc = (int*)c->host.p;
  int64_t n_admit = 0;
  Trace tr("contacts_update");
  tr.mark("enter", s, nb);
  if (nb > 0) {
    IBF_TRY(c->flags.reserve(nb + 1));
    IBF_TRY(c->pos.reserve(nb + 1));
    IBF_TRY(c->iscratch.reserve(2 * (nb + 1)));
    int* is_new = c->iscratch.p;
    int* keep = c->iscratch.p + (nb + 1);
    // resident CSR by min vertex
    unsigned rmask = 0, kmask = 0;
    IBF_TRY(key_csr(c, c->n, c->quad.p, c->kind.p, nullptr, c->v_count, c->v_ptr, c->v_list, &rmask, s));
    tr.mark("resident_csr", s, c->n);
    k_new_flags<<<grid_for(nb), 256, 0, s>>>(nb, bkind, bquad, c->kind.p, c->quad.p, rmask, c->v_ptr.p,
                                             c->v_list.p, is_new);
    IBF_LAUNCH_CHECK();
    tr.mark("new_flags", s);
    if (!c->admit_all) {
      k_earliest<<<grid_for(nb), 256, 0, s>>>(nb, bquad, btoi, is_new, c->earliest.p);
      IBF_LAUNCH_CHECK();
    }
    k_admit<<<grid_for(nb), 256, 0, s>>>(nb, bquad, btoi, is_new, c->earliest.p, c->admit_all, keep);
    IBF_LAUNCH_CHECK();
    if (!c->admit_all) {
      k_reset_earliest<<<grid_for(nb), 256, 0, s>>>(nb, bquad, c->earliest.p);
      IBF_LAUNCH_CHECK();
    }
    tr.mark("admit", s);
    // first occurrence among kept pairs
    IBF_TRY(key_csr(c, nb, bquad, bkind, keep, c->k_count, c->k_ptr, c->k_list, &kmask, s));
    tr.mark("kept_csr", s);
    k_first<<<grid_for(nb), 256, 0, s>>>(nb, bkind, bquad, keep, kmask, c->k_ptr.p, c->k_list.p, c->flags.p);
    IBF_LAUNCH_CHECK();
    IBF_CUDA(cudaMemsetAsync(c->flags.p + nb, 0, sizeof(int), s));
    IBF_TRY(exclusive_scan(c, c->flags.p, c->pos.p, nb + 1, s));
    // counts: number kept (reference counts duplicates), number appended
    IBF_CUDA(cudaMemsetAsync(keep + nb, 0, sizeof(int), s));
    IBF_TRY(exclusive_scan(c, keep, is_new, nb + 1, s));  // is_new reused as scan output
    IBF_CUDA(cudaMemcpyAsync(hostc, is_new + nb, sizeof(int), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaMemcpyAsync(hostc + 1, c->pos.p + nb, sizeof(int), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaStreamSynchronize(s));
    n_admit = hostc[0];
    const int64_t n_app = hostc[1];
    tr.mark("first_scan", s, n_app);
    if (n_app) {
      IBF_TRY(reserve_soa(c, c->n + n_app, s));
      k_append<<<grid_for(nb), 256, 0, s>>>(nb, c->n, bkind, bquad, c->flags.p, c->pos.p, c->kind.p, c->quad.p,
                                            c->lam.p, c->gamma.p, c->s.p, c->anchor_d.p, c->anchor_grad.p,
                                            c->anchor_x.p);
      IBF_LAUNCH_CHECK();
      c->n += n_app;
    }
  }
  tr.mark("append", s);
  // prune gamma < 0.01, stable
  int64_t n_pruned = 0;
  if (c->n) {
    const int64_t n = c->n;
    IBF_TRY(c->flags.reserve(n + 1));
    IBF_TRY(c->pos.reserve(n + 1));
    k_keep_gamma<<<grid_for(n), 256, 0, s>>>(n, c->gamma.p, c->flags.p);
    IBF_LAUNCH_CHECK();
    IBF_CUDA(cudaMemsetAsync(c->flags.p + n, 0, sizeof(int), s));
    IBF_TRY(exclusive_scan(c, c->flags.p, c->pos.p, n + 1, s));
    IBF_CUDA(cudaMemcpyAsync(hostc + 2, c->pos.p + n, sizeof(int), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaStreamSynchronize(s));
    const int64_t n_keep = hostc[2];
    n_pruned = n - n_keep;
    if (n_pruned) {
      IBF_TRY((compact_field<int, 1>(c, c->kind, n, n_keep, s)));
      IBF_TRY((compact_field<int, 4>(c, c->quad, n, n_keep, s)));
      IBF_TRY((compact_field<double, 1>(c, c->lam, n, n_keep, s)));
      IBF_TRY((compact_field<double, 1>(c, c->gamma, n, n_keep, s)));
      IBF_TRY((compact_field<double, 1>(c, c->s, n, n_keep, s)));
      IBF_TRY((compact_field<double, 1>(c, c->anchor_d, n, n_keep, s)));
      IBF_TRY((compact_field<double, 12>(c, c->anchor_grad, n, n_keep, s)));
      IBF_TRY((compact_field<double, 12>(c, c->anchor_x, n, n_keep, s)));
      c->n = n_keep;
    }
  }
  tr.mark("prune", s, n_pruned);
  tr.mark("exit", s);
  c->vc_nverts = -1;  // incidence must be rebuilt
  *admitted = n_admit;
  *pruned = n_pruned;
  return IBF_OK;
}

int contact_build_incidence(ibf_contacts* c, int64_t n_verts, cudaStream_t s) {
  const int64_t n = c->n;
  const int64_t ne = 4 * n;
  IBF_TRY(c->vc_ptr.reserve(n_verts + 1));
  IBF_TRY(c->vc_src.reserve(std::max<int64_t>(ne, 1)));
  IBF_TRY(c->sort_keys.reserve(std::max<int64_t>(ne, 1)));
  IBF_TRY(c->sort_vals.reserve(std::max<int64_t>(ne, 1)));
  IBF_TRY(c->sort_keys2.reserve(std::max<int64_t>(ne, 1)));
  IBF_TRY(c->v_count.reserve(n_verts + 1));
  IBF_TRY(c->tdot.reserve(std::max<int64_t>(n, 1)));
  IBF_TRY(c->coef_h.reserve(std::max<int64_t>(n, 1)));
  IBF_TRY(c->coef_g.reserve(std::max<int64_t>(n, 1)));
  IBF_TRY(c->cval.reserve(std::max<int64_t>(n, 1)));
  IBF_CUDA(cudaMemsetAsync(c->v_count.p, 0, (n_verts + 1) * sizeof(int), s));
  if (ne) {
    k_incidence_keys<<<grid_for(ne), 256, 0, s>>>(n, c->quad.p, c->sort_keys.p, c->sort_vals.p, c->v_count.p);
    IBF_LAUNCH_CHECK();
    int bits = 1;
    while ((1LL << bits) < n_verts) ++bits;
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, c->sort_keys.p, c->sort_keys2.p, c->sort_vals.p, c->vc_src.p,
                                    (int)ne, 0, bits, s);
    IBF_TRY(c->cub_tmp.reserve(need + 16));
    size_t have = c->cub_tmp.cap;
    IBF_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, have, c->sort_keys.p, c->sort_keys2.p, c->sort_vals.p,
                                             c->vc_src.p, (int)ne, 0, bits, s));
  }
  IBF_TRY(exclusive_scan(c, c->v_count.p, c->vc_ptr.p, n_verts + 1, s));
  c->vc_nverts = n_verts;
  c->trec_nverts = -1;
  return IBF_OK;
}

int contact_prepare(ibf_contacts* c, const double* x_hat, double mu, double offset, cudaStream_t s) {
  if (!c->n) return IBF_OK;
  k_prepare<<<grid_for(c->n), 256, 0, s>>>(c->n, c->quad.p, c->anchor_d.p, c->anchor_grad.p, c->anchor_x.p,
                                           c->lam.p, c->gamma.p, x_hat, mu, offset, c->cval.p, c->coef_g.p,
                                           c->coef_h.p);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

// Per-row term records for the PCG (k_pcg's warp-cooperative term pass):
// the incidences of every unmasked row, in vc order, as 32-byte records
// {g_c[slot] (3 doubles), c}, with masked (Dirichlet) rows given none — a
// pinned plate vertex can sit in 10^4 constraints, which a warp sharing its
// incidence range would otherwise walk.
__global__ void k_term_counts(int64_t n, const int* __restrict__ vc_ptr, const uint8_t* __restrict__ mask,
                              int* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = (mask && mask[i]) ? 0 : vc_ptr[i + 1] - vc_ptr[i];
}
__global__ void k_term_records(int64_t n, const int* __restrict__ vc_ptr, const int* __restrict__ vc_src,
                               const int* __restrict__ ip_ptr, const double* __restrict__ grad,
                               double4* __restrict__ rec) {
  // one warp per row: its lanes copy the row's records
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int o = ip_ptr[i], m = ip_ptr[i + 1] - o, e0 = vc_ptr[i];
    for (int k = lane; k < m; k += 32) {
      const int src = vc_src[e0 + k];
      const double* g = grad + 12 * (size_t)(src >> 2) + 3 * (src & 3);
      // meta: constraint (bits 0-31), slot (32-33), the row's lane in its 32-row slice (34-38)
      const long long meta = (long long)(src >> 2) | ((long long)(src & 3) << 32) | ((long long)(i & 31) << 34);
      rec[o + k] = make_double4(g[0], g[1], g[2], __longlong_as_double(meta));
    }
  }
}

int contact_pack_terms(ibf_contacts* c, int64_t n_verts, const uint8_t* mask, cudaStream_t s) {
  if (!c->n) return IBF_OK;
  IBF_TRY(c->ip_ptr.reserve(n_verts + 1));
  IBF_TRY(c->v_count.reserve(n_verts + 1));
  k_term_counts<<<grid_for(n_verts), 256, 0, s>>>(n_verts, c->vc_ptr.p, mask, c->v_count.p);
  IBF_LAUNCH_CHECK();
  IBF_CUDA(cudaMemsetAsync(c->v_count.p + n_verts, 0, sizeof(int), s));
  IBF_TRY(exclusive_scan(c, c->v_count.p, c->ip_ptr.p, n_verts + 1, s));
  IBF_TRY(c->trec.reserve(std::max<int64_t>(4 * c->n, 1)));
  k_term_records<<<(int)std::max<int64_t>(1, std::min<int64_t>(div_up(32 * n_verts, 256), 148LL * 16)), 256, 0, s>>>(
      n_verts, c->vc_ptr.p, c->vc_src.p, c->ip_ptr.p, c->anchor_grad.p, c->trec.p);
  IBF_LAUNCH_CHECK();
  c->trec_nverts = n_verts;
  return IBF_OK;
}

ContactView contact_view(ibf_contacts* c) {
  ContactView v;
  v.n = (int)c->n;
  v.quad = c->quad.p;
  v.grad = c->anchor_grad.p;
  v.coef = c->coef_h.p;
  v.vc_ptr = c->vc_ptr.p;
  v.vc_src = c->vc_src.p;
  v.t = c->tdot.p;
  if (c->trec_nverts >= 0) {
    v.ip_ptr = c->ip_ptr.p;
    v.rec = c->trec.p;
  }
  return v;
}

int contacts_refresh(ibf_contacts* c, const double* x, int* degen_dev, cudaStream_t s) {
  if (!c->n) return IBF_OK;
  k_refresh<<<grid_for(c->n), 256, 0, s>>>(c->n, c->kind.p, c->quad.p, x, c->anchor_d.p, c->anchor_grad.p,
                                           c->anchor_x.p, degen_dev);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

int contacts_dual(ibf_contacts* c, const double* x_hat, double offset, double mu, double decay, double* worst_dev,
                  cudaStream_t s) {
  IBF_CUDA(cudaMemsetAsync(worst_dev, 0, sizeof(double), s));
  if (!c->n) return IBF_OK;
  k_dual<<<grid_for(c->n), 256, 0, s>>>(c->n, c->quad.p, c->anchor_d.p, c->anchor_grad.p, c->anchor_x.p, x_hat,
                                        offset, mu, decay, c->lam.p, c->gamma.p, c->s.p, worst_dev);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

}  // namespace ibf

using namespace ibf;

extern "C" int ibf_contacts_create(int64_t n_verts, int admit_all, ibf_contacts** out) {
  if (n_verts < 0 || !out) {
    set_error("ibf_contacts_create: bad arguments");
    return IBF_ERR_BAD_ARG;
  }
  ibf_contacts* c = new ibf_contacts();
  c->admit_all = admit_all;
  c->n_verts = n_verts;
  int st = c->earliest.reserve(std::max<int64_t>(n_verts, 1));
  if (st == IBF_OK) st = reserve_soa(c, 1024, 0);
  if (st == IBF_OK) {
    std::vector<double> inf(std::max<int64_t>(n_verts, 1), INFINITY);
    st = c->earliest.upload(inf.data(), inf.size());
  }
  if (st == IBF_OK && cudaDeviceSynchronize() != cudaSuccess) st = IBF_ERR_CUDA;
  if (st != IBF_OK) {
    delete c;
    return st;
  }
  *out = c;
  return IBF_OK;
}

extern "C" void ibf_contacts_destroy(ibf_contacts* c) { delete c; }
extern "C" int64_t ibf_contacts_size(const ibf_contacts* c) { return c ? c->n : 0; }

extern "C" int ibf_contacts_update_host(ibf_contacts* c, int64_t n, const int64_t* kinds, const int64_t* quads,
                                        const double* tois, int64_t* admitted, int64_t* pruned, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  std::vector<int> k32(n), q32(4 * n);
  for (int64_t j = 0; j < n; ++j) {
    k32[j] = (int)kinds[j];
    for (int e = 0; e < 4; ++e) {
      if (quads[4 * j + e] < 0 || quads[4 * j + e] >= c->n_verts) {
        set_error("ibf_contacts_update_host: vertex index out of range");
        return IBF_ERR_BAD_ARG;
      }
      q32[4 * j + e] = (int)quads[4 * j + e];
    }
  }
  IBF_TRY(c->tmp_kind.upload(k32.data(), k32.size(), s));
  IBF_TRY(c->tmp_quad.upload(q32.data(), q32.size(), s));
  IBF_TRY(c->tmp_tois.upload(tois, (size_t)n, s));
  return contacts_update_dev(c, n, c->tmp_kind.p, c->tmp_quad.p, c->tmp_tois.p, admitted, pruned, s);
}

extern "C" int ibf_contacts_refresh_anchors(ibf_contacts* c, const double* x, int64_t* n_degenerate, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  IBF_TRY(c->iscratch.reserve(2));
  IBF_CUDA(cudaMemsetAsync(c->iscratch.p, 0, sizeof(int), s));
  IBF_TRY(contacts_refresh(c, x, c->iscratch.p, s));
  int h = 0;
  IBF_CUDA(cudaMemcpyAsync(&h, c->iscratch.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  *n_degenerate = h;
  return IBF_OK;
}

extern "C" int ibf_contacts_dual_sweep(ibf_contacts* c, const double* x_hat, double offset, double mu, double decay,
                                       double* worst_host, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  IBF_TRY(c->dscratch.reserve(2));
  IBF_TRY(contacts_dual(c, x_hat, offset, mu, decay, c->dscratch.p, s));
  IBF_CUDA(cudaMemcpyAsync(worst_host, c->dscratch.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  return IBF_OK;
}

extern "C" int ibf_contacts_export(const ibf_contacts* cc, int64_t* kind, int64_t* quad, double* lam, double* gamma,
                                   double* s_, double* anchor_d, double* anchor_grad, double* anchor_x,
                                   ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  ibf_contacts* c = const_cast<ibf_contacts*>(cc);
  cudaStream_t s = (cudaStream_t)st;
  const int64_t n = c->n;
  if (!n) return IBF_OK;
  std::vector<int> k32(n), q32(4 * n);
  IBF_CUDA(cudaMemcpyAsync(k32.data(), c->kind.p, n * sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(q32.data(), c->quad.p, 4 * n * sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(lam, c->lam.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(gamma, c->gamma.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(s_, c->s.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(anchor_d, c->anchor_d.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(anchor_grad, c->anchor_grad.p, 12 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(anchor_x, c->anchor_x.p, 12 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  for (int64_t j = 0; j < n; ++j) {
    kind[j] = k32[j];
    for (int e = 0; e < 4; ++e) quad[4 * j + e] = q32[4 * j + e];
  }
  return IBF_OK;
}

extern "C" int ibf_contacts_import(ibf_contacts* c, int64_t n, const int64_t* kind, const int64_t* quad,
                                   const double* lam, const double* gamma, const double* s_, const double* anchor_d,
                                   const double* anchor_grad, const double* anchor_x, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  std::vector<int> k32(n), q32(4 * n);
  for (int64_t j = 0; j < n; ++j) {
    k32[j] = (int)kind[j];
    for (int e = 0; e < 4; ++e) {
      if (quad[4 * j + e] < 0 || quad[4 * j + e] >= c->n_verts) {
        set_error("ibf_contacts_import: vertex index out of range");
        return IBF_ERR_BAD_ARG;
      }
      q32[4 * j + e] = (int)quad[4 * j + e];
    }
  }
  c->n = 0;
  IBF_TRY(reserve_soa(c, std::max<int64_t>(n, 1), s));
  if (n) {
    IBF_CUDA(cudaMemcpyAsync(c->kind.p, k32.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(c->quad.p, q32.data(), 4 * n * sizeof(int), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(c->lam.p, lam, n * sizeof(double), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(c->gamma.p, gamma, n * sizeof(double), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(c->s.p, s_, n * sizeof(double), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(c->anchor_d.p, anchor_d, n * sizeof(double), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(c->anchor_grad.p, anchor_grad, 12 * n * sizeof(double), cudaMemcpyHostToDevice, s));
    IBF_CUDA(cudaMemcpyAsync(c->anchor_x.p, anchor_x, 12 * n * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  IBF_CUDA(cudaStreamSynchronize(s));
  c->n = n;
  c->vc_nverts = -1;
  return IBF_OK;
}
