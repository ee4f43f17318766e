// Symmetric 3x3-block SpMV and the device-resident block-Jacobi PCG.
//
// Replaces BlockSparseMatrix.matvec and pcg_solve (intact/sparse.py:64-73,
// :99-150; paths relative to /root/reference/pkg/src).
//
// Storage is the reference's information content — diagonal + strict-upper
// 3x3 blocks only — laid out as sliced ELL (internal.cuh, `qel`).  One
// thread owns one row (all three components): it streams its upper blocks
// (slot-major, so the 32 lanes of a warp read 256 contiguous bytes per
// entry), gathers p at their columns, then applies the lower triangle
// through the row's transpose list (block, source row), then the matrix-free
// contact term.  Every row is a fixed-order gather: no atomics, results are
// bit-reproducible run to run.  A block's second (transposed) read hits L2:
// the grid sweeps rows in ascending order with a bounded window of rows in
// flight, and a row's lower blocks were streamed at most (n+1)^2 rows earlier
// on lattice meshes (ncu: DRAM bytes 1.06x the algorithmic SpMV bytes).
//
// The whole PCG (all iterations, the reference's stopping rule, best-iterate
// tracking, the 250-iteration restart, pAp <= 0 bail-out) runs in ONE
// persistent cooperative kernel with two grid barriers per iteration:
//
//   A  p_k = z + beta p_{k-1} (formed on the fly wherever p is gathered, so
//      there is no separate direction-update pass), q = H p_k, pAp partials
//   B  alpha = rz / pAp; x += alpha p; r -= alpha q; z = P^-1 r; |r|^2, rz
//
// Each thread keeps q and p_k of its own rows in shared memory between A and
// B (same row mapping in both phases), and its rows' residual for the whole
// solve, so none of them makes a round trip through HBM.  All reductions are
// fixed-order (per-CTA tree, then one warp over the CTA partials), so every
// CTA derives bit-identical scalars.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <type_traits>
#include <vector>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace ibf {

#ifndef IBF_PCG_THREADS
#define IBF_PCG_THREADS 256
#endif
#ifndef IBF_PCG_MINB
#define IBF_PCG_MINB 4
#endif
// rows stop at their first padded slot / lower entry (1) or walk the slice's full width (0)
#ifndef IBF_SELL_STOP
#define IBF_SELL_STOP 1
#endif
#ifndef IBF_SPMV_UNROLL
#define IBF_SPMV_UNROLL 2
#endif
// Dynamic chunk scheduling of phase A (IBF_PCG_DYNAMIC=1): measured equal to
// the static split (86.3 vs 86.4 us per iteration).  The per-CTA spread of
// phase A (44-77 us) persists with it: a chunk is one row per thread, and a
// row's dependent-load latency (~20 us under load) is the scheduling grain.
#ifndef IBF_PCG_DYNAMIC
#define IBF_PCG_DYNAMIC 0
#endif
constexpr int PCG_THREADS = IBF_PCG_THREADS;
// Shared-memory budget per CTA for keeping each thread's rows' residual on
// chip for the whole solve (it is only ever touched by its row's owner):
// 16 KB per CTA at C4 size, 86.6 vs 90.4 us per CG iteration.  Carrying q
// and p across the A/B barrier as well (IBF_PCG_CARRY_QP=1, ~48 KB per CTA)
// is 2x slower: that SMEM comes out of the unified L1 the SpMV gathers live
// in.  An interleaved (z, p) record layout for the gathers was also slower
// (94 vs 88 us: the two half-record writes per iteration cost more than the
// fused gather saves).
#ifndef IBF_PCG_SMEM_KB
#define IBF_PCG_SMEM_KB 20
#endif
constexpr int PCG_SMEM_BYTES = IBF_PCG_SMEM_KB * 1024;
// phase B's barrier split around the x update
#ifndef IBF_PCG_SPLIT_BAR
#define IBF_PCG_SPLIT_BAR 1
#endif
// small systems: lanes per row in phase A
#ifndef IBF_PCG_LANES
#define IBF_PCG_LANES 4
#endif
#ifndef IBF_PCG_LANES_MAX_N
#define IBF_PCG_LANES_MAX_N 16384
#endif
// contact dots by linearity from per-row z products (no dot phase; see warp_zdot)
#ifndef IBF_PCG_ZDOT
#define IBF_PCG_ZDOT 0
#endif
// with the materialised direction, the term dots run in phase P before its barrier (1) or after it,
// behind the ready counter (0): measured equal (203.7 vs 202.6 us per CG iteration at 331k contacts)
#ifndef IBF_PCG_PMAT_DOTS
#define IBF_PCG_PMAT_DOTS 0
#endif
// materialise p_k behind a third grid barrier (1) or form it on the fly where gathered (0)
#ifndef IBF_PCG_PMAT
#define IBF_PCG_PMAT 1
#endif
// contact_dot_rec issues its 4 z gathers unconditionally, mask applied after (1;
// measured equal, 225.3 vs 226.2 us per CG iteration, with a 28-byte spill), or
// behind the mask (0)
#ifndef IBF_PCG_DOT_UNCOND
#define IBF_PCG_DOT_UNCOND 0
#endif
// contact dots g.p_k = g.z_k + beta g.p_{k-1} (z gathers only; contact_dot_rec)
#ifndef IBF_PCG_DOT_REC
#define IBF_PCG_DOT_REC 1
#endif
// matrix-free term dots behind a ready counter instead of a grid barrier
#ifndef IBF_PCG_READY
#define IBF_PCG_READY 1
#endif

// ---------------------------------------------------------------- gathers

// Diagnostic builds for the DRAM-traffic breakdown (never the product):
// IBF_DIAG_NO_GATHER replaces the SpMV's vector gathers by constants,
// IBF_DIAG_NO_LOWER skips the transposed (lower) entries.
#ifndef IBF_DIAG_NO_GATHER
#define IBF_DIAG_NO_GATHER 0
#endif
#ifndef IBF_DIAG_NO_LOWER
#define IBF_DIAG_NO_LOWER 0
#endif

// p at vertex j: a plain vector ...
struct PlainGather {
  const double* __restrict__ p;
  __device__ __forceinline__ void get(int j, double& x0, double& x1, double& x2) const {
    if (IBF_DIAG_NO_GATHER) {
      x0 = x1 = x2 = 1e-3 * (double)(j & 7);
      return;
    }
    const double* P = p + 3 * (size_t)j;
    x0 = P[0];
    x1 = P[1];
    x2 = P[2];
  }
};

// ... or the new CG direction z + beta p_old formed on the fly (first:
// p = z; intact/sparse.py:148), one fused multiply-add, so every reader
// forms the bits the owner stores.  (-DIBF_CG_DIR_NUMPY rounds the product
// separately as numpy does; neither is bit-identical to the oracle's CG,
// whose Jacobi inverse and dot orders differ anyway.  The golden box-on-slab
// trajectory sits on exact admission ties, intact/contact.py:151, and its
// key sets match with the fused form, parity.)
#ifdef IBF_CG_DIR_NUMPY
__device__ __forceinline__ double cg_dir(double beta, double p, double z) { return __dadd_rn(z, __dmul_rn(beta, p)); }
#else
__device__ __forceinline__ double cg_dir(double beta, double p, double z) { return __fma_rn(beta, p, z); }
#endif

struct DirGather {
  const double* __restrict__ z;
  const double* __restrict__ pold;
  double beta;
  bool first;
  __device__ __forceinline__ void get(int j, double& x0, double& x1, double& x2) const {
    if (IBF_DIAG_NO_GATHER) {
      x0 = x1 = x2 = 1e-3 * (double)(j & 7);
      return;
    }
    const double* Z = z + 3 * (size_t)j;
    if (first) {
      x0 = Z[0];
      x1 = Z[1];
      x2 = Z[2];
    } else {
      const double* P = pold + 3 * (size_t)j;
      const double z0 = Z[0], z1 = Z[1], z2 = Z[2];
      const double p0 = P[0], p1 = P[1], p2 = P[2];
      x0 = cg_dir(beta, p0, z0);
      x1 = cg_dir(beta, p1, z1);
      x2 = cg_dir(beta, p2, z2);
    }
  }
};

// ---------------------------------------------------------------- SpMV pieces

// t_c = coef_c * sum_slot g_c[slot] . p[v(slot)], masked columns excluded.
// Ready counter for the term dots (k_pcg): each CTA that computes term dots
// adds 1 to a global counter once all its dots are stored, and a row that
// touches terms waits once, just before its term loop, until the counter
// reaches this iteration's target — a barrier only for the rows that need
// it, at the end of their SpMV work, instead of a grid barrier before it.
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
  unsigned x;
  while (true) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
    if ((int)(x - target) >= 0) break;
    __nanosleep(32);
  }
}

template <class Gather>
__device__ __forceinline__ void contact_dot(const Operator& op, const Gather& gp, int c) {
  const ContactView& cv = op.contact;
  const int* q = cv.quad + 4 * c;
  const double* g = cv.grad + 12 * c;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int v = q[k];
    if (op.mask && op.mask[v]) continue;
    double x0, x1, x2;
    gp.get(v, x0, x1, x2);
    acc += g[3 * k] * x0 + g[3 * k + 1] * x1 + g[3 * k + 2] * x2;
  }
  cv.t[c] = cv.coef[c] * acc;
}

// The CG direction's dot by linearity, g_c . p_k = g_c . z_k + beta_k (g_c . p_{k-1})
// (IBF_PCG_DOT_REC): only z is gathered at the 4 vertices, not z and p_{k-1};
// tprev[c] carries g_c . p_{k-1} from the previous iteration (first
// iteration and after a restart: p_k = z_k).
__device__ __forceinline__ void contact_dot_rec(const Operator& op, const DirGather& gd, int c, double* tprev) {
  const ContactView& cv = op.contact;
#if !IBF_PCG_DOT_UNCOND
  const int* qq = cv.quad + 4 * c;
  const double* gg = cv.grad + 12 * c;
  double acc0 = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int vv = qq[k];
    if (op.mask && op.mask[vv]) continue;
    const double* Z = gd.z + 3 * (size_t)vv;
    acc0 += gg[3 * k] * Z[0] + gg[3 * k + 1] * Z[1] + gg[3 * k + 2] * Z[2];
  }
  const double dot0 = gd.first ? acc0 : __fma_rn(gd.beta, tprev[c], acc0);
  tprev[c] = dot0;
  cv.t[c] = cv.coef[c] * dot0;
#else
  const int4 q = *reinterpret_cast<const int4*>(cv.quad + 4 * (size_t)c);
  const int v[4] = {q.x, q.y, q.z, q.w};
  const double* g = cv.grad + 12 * (size_t)c;
  // the z gathers are issued unconditionally and masked slots dropped after
  // (z is finite everywhere): the chain is quad -> (mask, z), not quad ->
  // mask -> z
  double z[4][3];
  bool m[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double* Z = gd.z + 3 * (size_t)v[k];
    z[k][0] = Z[0];
    z[k][1] = Z[1];
    z[k][2] = Z[2];
    m[k] = op.mask && op.mask[v[k]];
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (!m[k]) acc += g[3 * k] * z[k][0] + g[3 * k + 1] * z[k][1] + g[3 * k + 2] * z[k][2];
  const double dot = gd.first ? acc : __fma_rn(gd.beta, tprev[c], acc);
  tprev[c] = dot;
  cv.t[c] = cv.coef[c] * dot;
#endif
}

// friction term k: t_k = Hw_k sum_j w_j p_j over unmasked j
template <class Gather>
__device__ __forceinline__ void friction_dot(const Operator& op, const Gather& gp, int k) {
  const FrictionView& fv = op.friction;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int v = fv.quad[4 * k + j];
    if (op.mask && op.mask[v]) continue;
    double x0, x1, x2;
    gp.get(v, x0, x1, x2);
    const double w = fv.w[4 * k + j];
    a0 += w * x0;
    a1 += w * x1;
    a2 += w * x2;
  }
  const double* H = fv.hw + 9 * (size_t)k;
  double* t = fv.t + 3 * (size_t)k;
  t[0] = H[0] * a0 + H[1] * a1 + H[2] * a2;
  t[1] = H[3] * a0 + H[4] * a1 + H[5] * a2;
  t[2] = H[6] * a0 + H[7] * a1 + H[8] * a2;
}

// the matrix-free terms' per-term dots (contact and friction) over this thread's share
template <class Gather>
__device__ __forceinline__ void term_dots(const Operator& op, const Gather& gp, bool contacts = true,
                                          double* tprev = nullptr) {
  const int S = gridDim.x * blockDim.x;
  if (contacts) {
    if constexpr (std::is_same<Gather, DirGather>::value) {
      if (tprev) {
        // two constraints per step, all their loads issued before any use:
        // the dot phase is a chain quad -> z gathers per constraint, and the
        // ready counter holds every row with terms until it ends
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < op.contact.n; c += S) contact_dot_rec(op, gp, c, tprev);
        contacts = false;
      }
    }
    if (contacts)
      for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < op.contact.n; c += S) contact_dot(op, gp, c);
  }
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < op.friction.n; k += S) friction_dot(op, gp, k);
}

// Where row_product reads the terms' dots: after a grid barrier ...
struct StoredTerms {
  __device__ __forceinline__ void ready() const {}
  __device__ __forceinline__ double contact(const ContactView& cv, int c) const { return cv.t[c]; }
  __device__ __forceinline__ void friction(const FrictionView& fv, int k, double t[3]) const {
    const double* T = fv.t + 3 * (size_t)k;
    t[0] = T[0];
    t[1] = T[1];
    t[2] = T[2];
  }
};
// ... or after this row's wait on the ready counter (L2 reads: another SM
// wrote them after this one's L1 may have cached the previous iteration's)
struct CountedTerms {
  const unsigned* counter;
  unsigned target;
  __device__ __forceinline__ void ready() const { wait_count(counter, target); }
  __device__ __forceinline__ double contact(const ContactView& cv, int c) const { return __ldcg(cv.t + c); }
  __device__ __forceinline__ void friction(const FrictionView& fv, int k, double t[3]) const {
    const double* T = fv.t + 3 * (size_t)k;
    t[0] = __ldcg(T);
    t[1] = __ldcg(T + 1);
    t[2] = __ldcg(T + 2);
  }
};

// one upper block: a_r += (b[3r] x0 + b[3r+1] x1) + b[3r+2] x2
__device__ __forceinline__ void acc_upper(const double b[9], double x0, double x1, double x2, double& a0, double& a1,
                                          double& a2) {
  a0 += b[0] * x0 + b[1] * x1 + b[2] * x2;
  a1 += b[3] * x0 + b[4] * x1 + b[5] * x2;
  a2 += b[6] * x0 + b[7] * x1 + b[8] * x2;
}
// one transposed block: a_c += (b[c] x0 + b[3+c] x1) + b[6+c] x2
__device__ __forceinline__ void acc_lower(const double b[9], double x0, double x1, double x2, double& a0, double& a1,
                                          double& a2) {
  a0 += b[0] * x0 + b[3] * x1 + b[6] * x2;
  a1 += b[1] * x0 + b[4] * x1 + b[7] * x2;
  a2 += b[2] * x0 + b[5] * x1 + b[8] * x2;
}

// y_i = (H p)_i for row i: upper slots, transposed lower entries, contact.
// Block values and the pattern are read-only for the whole solve
// (non-coherent loads); p is rewritten between phases of the persistent
// kernel, so it is loaded coherently.  Per component the sum runs over the
// row's blocks in storage order.  Two slots are in flight per iteration
// (18 matrix entries, 2 indices, 6 p entries): the product is latency-bound
// otherwise.
template <class Gather, class Terms = StoredTerms, bool CONTACT = true>
__device__ __forceinline__ void row_product(const Operator& op, const Gather& gp, int pos, int i, double y[3],
                                            const Terms& terms = Terms()) {
  // storage by position (row_at maps positions to rows: internal.cuh); row i
  // for the contact incidences.  Padding slots are zero blocks whose column
  // is the position's own row, so they add exact zeros.
  const int s = pos >> SELL_SHIFT, lane = pos & (SELL_C - 1);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  {
    const int q0 = __ldg(op.slice_ptr + s), w = (__ldg(op.slice_ptr + s + 1) - q0) >> SELL_SHIFT;
    const double* V = op.val + 9 * (size_t)q0 + QEL_LS * lane;
    const int* C = op.col + q0 + lane;
    int k = 0;
    if (IBF_SPMV_UNROLL >= 2) {
      // column indices are loaded one slot pair ahead, so the p gathers of a
      // pair never wait on an index load (the chain per pair is one level)
      int n0 = w > 0 ? __ldg(C) : 0, n1 = w > 1 ? __ldg(C + SELL_C) : 0;
      for (; k + 2 <= w; k += 2) {
        const int j0 = n0, j1 = n1;
        // IBF_SELL_STOP: a padded slot (col == own row past the diagonal
        // slot) ends the row: its lane issues no more loads for the slice
        if (IBF_SELL_STOP && k > 0 && j0 == i) {
          k = w;
          break;
        }
        if (k + 2 < w) n0 = __ldg(C + SELL_C * (k + 2));
        if (k + 3 < w) n1 = __ldg(C + SELL_C * (k + 3));
        const double* B = V + 9 * SELL_C * (size_t)k;
        double b[9], c[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) {
          b[e] = __ldg(B + QEL_ES * e);
          c[e] = __ldg(B + 9 * SELL_C + QEL_ES * e);
        }
        double x0, x1, x2, y0, y1, y2;
        gp.get(j0, x0, x1, x2);
        gp.get(j1, y0, y1, y2);
        acc_upper(b, x0, x1, x2, a0, a1, a2);
        acc_upper(c, y0, y1, y2, a0, a1, a2);
      }
    }
    for (; k < w; ++k) {
      const int j = __ldg(C + SELL_C * k);
      if (IBF_SELL_STOP && k > 0 && j == i) break;
      const double* B = V + 9 * SELL_C * (size_t)k;
      double b[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) b[e] = __ldg(B + QEL_ES * e);
      double x0, x1, x2;
      gp.get(j, x0, x1, x2);
      acc_upper(b, x0, x1, x2, a0, a1, a2);
    }
  }
  if (!IBF_DIAG_NO_LOWER) {
    const int l0 = __ldg(op.low_ptr + s), w = (__ldg(op.low_ptr + s + 1) - l0) >> SELL_SHIFT;
    const int2* L = op.low + l0 + lane;
    int t = 0;
    if (IBF_SPMV_UNROLL >= 2) {
      int2 n0 = w > 0 ? __ldg(L) : make_int2(0, 0), n1 = w > 1 ? __ldg(L + SELL_C) : make_int2(0, 0);
      for (; t + 2 <= w; t += 2) {
        const int2 e0 = n0, e1 = n1;
        if (IBF_SELL_STOP && e0.x == op.zero_q) {
          t = w;
          break;
        }
        if (t + 2 < w) n0 = __ldg(L + SELL_C * (t + 2));
        if (t + 3 < w) n1 = __ldg(L + SELL_C * (t + 3));
        const double* B0 = op.val + qel(e0.x, 0);
        const double* B1 = op.val + qel(e1.x, 0);
        double b[9], c[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) {
          b[e] = __ldg(B0 + QEL_ES * e);
          c[e] = __ldg(B1 + QEL_ES * e);
        }
        double x0, x1, x2, y0, y1, y2;
        gp.get(e0.y, x0, x1, x2);
        gp.get(e1.y, y0, y1, y2);
        acc_lower(b, x0, x1, x2, a0, a1, a2);
        acc_lower(c, y0, y1, y2, a0, a1, a2);
      }
    }
    for (; t < w; ++t) {
      const int2 le = __ldg(L + SELL_C * t);
      if (IBF_SELL_STOP && le.x == op.zero_q) break;
      const double* B = op.val + qel(le.x, 0);
      double b[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) b[e] = __ldg(B + QEL_ES * e);
      double x0, x1, x2;
      gp.get(le.y, x0, x1, x2);
      acc_lower(b, x0, x1, x2, a0, a1, a2);
    }
  }
  if (CONTACT && op.contact.n && !(op.mask && op.mask[i])) {
    const ContactView& cv = op.contact;
    const int e0 = cv.vc_ptr[i], e1 = cv.vc_ptr[i + 1];
    if (e0 < e1) terms.ready();
    for (int e = e0; e < e1; ++e) {
      const int src = cv.vc_src[e];
      const int c = src >> 2, slot = src & 3;
      const double t = terms.contact(cv, c);
      const double* g = cv.grad + 12 * c + 3 * slot;
      a0 += t * g[0];
      a1 += t * g[1];
      a2 += t * g[2];
    }
  }
  if (op.friction.n && !(op.mask && op.mask[i])) {
    const FrictionView& fv = op.friction;
    if (fv.vf_ptr[i] < fv.vf_ptr[i + 1]) terms.ready();
    for (int e = fv.vf_ptr[i]; e < fv.vf_ptr[i + 1]; ++e) {
      const int src = fv.vf_src[e];
      const double w = fv.w[src];
      double t[3];
      terms.friction(fv, src >> 2, t);
      a0 += w * t[0];
      a1 += w * t[1];
      a2 += w * t[2];
    }
  }
  y[0] = a0;
  y[1] = a1;
  y[2] = a2;
}

// Contact terms of the warp's 32 consecutive rows r0 .. r0+31 (all lanes
// call this, converged): the rows' term records are one contiguous range of
// ContactView::rec, so the lanes walk it together, TERM_CHUNK records at a
// time, each forming t_c g_c[slot] into shared memory; then each row adds
// its own records' products in record order.  Rows take 0-50 terms (p50 3,
// p99 17 on the squishy press), so one row per lane kept ~1/6 of the lanes
// busy through the term loop (the slowest row of a warp sets its length).
constexpr int TERM_CHUNK = 32;
template <class Terms>
__device__ __forceinline__ void warp_terms(const ContactView& cv, const Terms& terms, int r0, int n, double* buf,
                                           double& a0, double& a1, double& a2) {
  const int lane = threadIdx.x & 31;
  const int rl = min(r0 + 32, n);
  const int E0 = __ldg(cv.ip_ptr + r0), E1 = __ldg(cv.ip_ptr + rl);
  if (E0 == E1) return;
  terms.ready();
  const int i = r0 + lane;
  const int s0 = i < rl ? __ldg(cv.ip_ptr + i) : 0, s1 = i < rl ? __ldg(cv.ip_ptr + i + 1) : 0;
  for (int base = E0; base < E1; base += TERM_CHUNK) {
    const int m = min(TERM_CHUNK, E1 - base);
    for (int k = lane; k < m; k += 32) {
      const double2* rp = reinterpret_cast<const double2*>(cv.rec + base + k);
      const double2 ra = __ldg(rp), rb = __ldg(rp + 1);
      const double4 r = make_double4(ra.x, ra.y, rb.x, rb.y);
      const double t = terms.contact(cv, (int)(__double_as_longlong(r.w) & 0xffffffffll));
      buf[k] = t * r.x;
      buf[TERM_CHUNK + k] = t * r.y;
      buf[2 * TERM_CHUNK + k] = t * r.z;
    }
    __syncwarp();
    const int lo = max(s0, base), hi = min(s1, base + m);
    for (int e = lo - base; e < hi - base; ++e) {
      a0 += buf[e];
      a1 += buf[TERM_CHUNK + e];
      a2 += buf[2 * TERM_CHUNK + e];
    }
    __syncwarp();
  }
}

// Contact dots without a dot phase (k_pcg "zdot" mode).  By linearity
// g_c . p_k = sum_slots g_c[slot] . z_k[v_slot] + beta_k (g_c . p_{k-1}):
// where a row's z is formed (init, phase B, restart) its warp writes
// g_c[slot] . z_i into zdot[4c + slot] for each of the row's records, and in
// phase A each record sums its constraint's 4 zdot entries in slot order and
// adds beta times its own copy of the previous dot (pdot[4c + slot]; the
// copies of one constraint are formed from identical inputs, so they stay
// bit-identical).  Masked slots have no records and keep zdot = 0, as the
// masked gathers of contact_dot contribute nothing.  No CTA waits for
// another's term dots inside phase A, and the z / p gathers of the dot
// phase (quad -> vertex -> value chains) are gone.
__device__ __forceinline__ double4 ld_rec(const double4* p) {
  const double2* rp = reinterpret_cast<const double2*>(p);
  const double2 ra = __ldg(rp), rb = __ldg(rp + 1);
  return make_double4(ra.x, ra.y, rb.x, rb.y);
}
__device__ __forceinline__ void warp_zdot(const ContactView& cv, int r0, int n, const double z[3], double* zs,
                                          double* zdot) {
  const int lane = threadIdx.x & 31;
  const int rl = min(r0 + 32, n);
  const int E0 = __ldg(cv.ip_ptr + r0), E1 = __ldg(cv.ip_ptr + rl);
  if (E0 == E1) return;
  zs[lane] = z[0];
  zs[32 + lane] = z[1];
  zs[64 + lane] = z[2];
  __syncwarp();
  for (int e = E0 + lane; e < E1; e += 32) {
    const double4 r = ld_rec(cv.rec + e);
    const long long m = __double_as_longlong(r.w);
    const int c = (int)(m & 0xffffffffll), slot = (int)((m >> 32) & 3), ol = (int)((m >> 34) & 31);
    zdot[4 * (size_t)c + slot] = r.x * zs[ol] + r.y * zs[32 + ol] + r.z * zs[64 + ol];
  }
  __syncwarp();
}
__device__ __forceinline__ void warp_terms_z(const ContactView& cv, int r0, int n, double* buf, bool first,
                                             double beta, const double* zdot, double* pdot, double& a0, double& a1,
                                             double& a2) {
  const int lane = threadIdx.x & 31;
  const int rl = min(r0 + 32, n);
  const int E0 = __ldg(cv.ip_ptr + r0), E1 = __ldg(cv.ip_ptr + rl);
  if (E0 == E1) return;
  const int i = r0 + lane;
  const int s0 = i < rl ? __ldg(cv.ip_ptr + i) : 0, s1 = i < rl ? __ldg(cv.ip_ptr + i + 1) : 0;
  for (int base = E0; base < E1; base += TERM_CHUNK) {
    const int m = min(TERM_CHUNK, E1 - base);
    for (int k = lane; k < m; k += 32) {
      const double4 r = ld_rec(cv.rec + base + k);
      const long long mt = __double_as_longlong(r.w);
      const int c = (int)(mt & 0xffffffffll), slot = (int)((mt >> 32) & 3);
      const double2* Zd = reinterpret_cast<const double2*>(zdot + 4 * (size_t)c);
      const double2 z01 = Zd[0], z23 = Zd[1];
      const double zsum = ((z01.x + z01.y) + z23.x) + z23.y;
      double* pd = pdot + 4 * (size_t)c + slot;
      const double dot = first ? zsum : __fma_rn(beta, *pd, zsum);
      *pd = dot;
      const double t = __ldg(cv.coef + c) * dot;
      buf[k] = t * r.x;
      buf[TERM_CHUNK + k] = t * r.y;
      buf[2 * TERM_CHUNK + k] = t * r.z;
    }
    __syncwarp();
    const int lo = max(s0, base), hi = min(s1, base + m);
    for (int e = lo - base; e < hi - base; ++e) {
      a0 += buf[e];
      a1 += buf[TERM_CHUNK + e];
      a2 += buf[2 * TERM_CHUNK + e];
    }
    __syncwarp();
  }
}

// Row i's product split over L lanes of one warp (lane sub takes slots,
// lower entries and term incidences sub, sub + L, ...); the caller sums the
// L partial results with shuffles in a fixed order.  For small systems, where
// a CG iteration is the latency of one row's chain of block loads.
template <class Gather, class Terms = StoredTerms>
__device__ __forceinline__ void row_product_lanes(const Operator& op, const Gather& gp, int pos, int i, double y[3],
                                                  int sub, int L, const Terms& terms = Terms()) {
  const int s = pos >> SELL_SHIFT, lane = pos & (SELL_C - 1);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  {
    const int q0 = __ldg(op.slice_ptr + s), w = (__ldg(op.slice_ptr + s + 1) - q0) >> SELL_SHIFT;
    const double* V = op.val + 9 * (size_t)q0 + QEL_LS * lane;
    const int* C = op.col + q0 + lane;
    for (int k = sub; k < w; k += L) {
      const int j = __ldg(C + SELL_C * k);
      const double* B = V + 9 * SELL_C * (size_t)k;
      double b[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) b[e] = __ldg(B + QEL_ES * e);
      double x0, x1, x2;
      gp.get(j, x0, x1, x2);
      acc_upper(b, x0, x1, x2, a0, a1, a2);
    }
  }
  {
    const int l0 = __ldg(op.low_ptr + s), w = (__ldg(op.low_ptr + s + 1) - l0) >> SELL_SHIFT;
    const int2* Lw = op.low + l0 + lane;
    for (int t = sub; t < w; t += L) {
      const int2 le = __ldg(Lw + SELL_C * t);
      const double* B = op.val + qel(le.x, 0);
      double b[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) b[e] = __ldg(B + QEL_ES * e);
      double x0, x1, x2;
      gp.get(le.y, x0, x1, x2);
      acc_lower(b, x0, x1, x2, a0, a1, a2);
    }
  }
  if (op.contact.n && !(op.mask && op.mask[i])) {
    const ContactView& cv = op.contact;
    const int e0 = cv.vc_ptr[i], e1 = cv.vc_ptr[i + 1];
    if (e0 + sub < e1) terms.ready();
    for (int e = e0 + sub; e < e1; e += L) {
      const int src = cv.vc_src[e];
      const int c = src >> 2, slot = src & 3;
      const double t = terms.contact(cv, c);
      const double* g = cv.grad + 12 * c + 3 * slot;
      a0 += t * g[0];
      a1 += t * g[1];
      a2 += t * g[2];
    }
  }
  if (op.friction.n && !(op.mask && op.mask[i])) {
    const FrictionView& fv = op.friction;
    if (fv.vf_ptr[i] + sub < fv.vf_ptr[i + 1]) terms.ready();
    for (int e = fv.vf_ptr[i] + sub; e < fv.vf_ptr[i + 1]; e += L) {
      const int src = fv.vf_src[e];
      const double w = fv.w[src];
      double t[3];
      terms.friction(fv, src >> 2, t);
      a0 += w * t[0];
      a1 += w * t[1];
      a2 += w * t[2];
    }
  }
  y[0] = a0;
  y[1] = a1;
  y[2] = a2;
}

__global__ void k_contact_dot(Operator op, const double* __restrict__ p) {
  term_dots(op, PlainGather{p});
}

__global__ void __launch_bounds__(256, 2) k_spmv(Operator op, const double* __restrict__ p, double* __restrict__ y) {
  const PlainGather gp{p};
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < op.n; pos += gridDim.x * blockDim.x) {
    const int i = row_at(op, pos);
    double v[3];
    row_product(op, gp, pos, i, v);
    y[3 * (size_t)i] = v[0];
    y[3 * (size_t)i + 1] = v[1];
    y[3 * (size_t)i + 2] = v[2];
  }
}

// ------------------------------------------------ TMA-staged upper stream
// Each warp owns one 32-row slice at a time.  Its upper slots are one
// contiguous range (w x 2304 bytes, 16-byte aligned), so lane 0 streams them
// into the warp's shared-memory stages with 1D bulk async copies
// (cp.async.bulk ... mbarrier::complete_tx), two slots per stage, two stages:
// the copy engine moves the next pair while the lanes consume the current
// one from SMEM (conflict-free: entry e of slot k for lane l at
// stage[(k*9 + e)*32 + l]).  The p gathers and the transposed part stay LDG.
constexpr int TMA_WARPS = 4;                   // 128 threads, 36.9 KB of stages
constexpr int TMA_STAGE_DOUBLES = 2 * 288;     // two slots of a slice

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(TMA_WARPS * 32, 1) k_spmv_tma(Operator op, const double* __restrict__ p,
                                                              double* __restrict__ y) {
  __shared__ __align__(128) double stage[TMA_WARPS][2][TMA_STAGE_DOUBLES];
  __shared__ __align__(8) unsigned long long bar[TMA_WARPS][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    mbar_init(&bar[warp][0], 1);
    mbar_init(&bar[warp][1], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  unsigned phase[2] = {0, 0};
  const PlainGather gp{p};
  const int n_slices = (op.n + 31) >> 5;
  for (int sl = blockIdx.x * TMA_WARPS + warp; sl < n_slices; sl += gridDim.x * TMA_WARPS) {
    const int pos = 32 * sl + lane;
    const int i = pos < op.n ? row_at(op, pos) : 0;
    const int q0 = __ldg(op.slice_ptr + sl), w = (__ldg(op.slice_ptr + sl + 1) - q0) >> 5;
    const double* V = op.val + 9 * (size_t)q0;
    const int* C = op.col + q0 + lane;
    const int npairs = (w + 1) >> 1;
    auto issue = [&](int pr, int st) {
      if (lane == 0) {
        const int slots = min(2, w - 2 * pr);
        const unsigned bytes = (unsigned)(slots * 288 * sizeof(double));
        mbar_expect_tx(&bar[warp][st], bytes);
        bulk_g2s(stage[warp][st], V + 576 * (size_t)pr, bytes, &bar[warp][st]);
      }
    };
    if (npairs > 0) issue(0, 0);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int pr = 0; pr < npairs; ++pr) {
      const int st = pr & 1;
      // every lane has finished reading stage st^1 (pair pr-1) before it is refilled
      __syncwarp();
      if (pr + 1 < npairs) issue(pr + 1, st ^ 1);
      const int k = 2 * pr;
      const int j0 = __ldg(C + 32 * k);
      const int j1 = (k + 1 < w) ? __ldg(C + 32 * k + 32) : i;
      double x0, x1, x2, z0 = 0.0, z1 = 0.0, z2 = 0.0;
      gp.get(j0, x0, x1, x2);
      if (k + 1 < w) gp.get(j1, z0, z1, z2);
      mbar_wait(&bar[warp][st], phase[st]);
      phase[st] ^= 1;
      const double* S0 = stage[warp][st] + QEL_LS * lane;
      double b[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) b[e] = S0[QEL_ES * e];
      acc_upper(b, x0, x1, x2, a0, a1, a2);
      if (k + 1 < w) {
#pragma unroll
        for (int e = 0; e < 9; ++e) b[e] = S0[288 + QEL_ES * e];
        acc_upper(b, z0, z1, z2, a0, a1, a2);
      }
    }
    __syncwarp();
    if (pos < op.n) {
      // transposed part and contact/friction as in row_product
      const int l0 = __ldg(op.low_ptr + sl), lw = (__ldg(op.low_ptr + sl + 1) - l0) >> 5;
      const int2* L = op.low + l0 + lane;
      for (int t = 0; t < lw; ++t) {
        const int2 le = __ldg(L + 32 * t);
        const double* B = op.val + qel(le.x, 0);
        double b[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) b[e] = __ldg(B + QEL_ES * e);
        double x0, x1, x2;
        gp.get(le.y, x0, x1, x2);
        acc_lower(b, x0, x1, x2, a0, a1, a2);
      }
      y[3 * (size_t)i] = a0;
      y[3 * (size_t)i + 1] = a1;
      y[3 * (size_t)i + 2] = a2;
    }
  }
}

int spmv(const Operator& op, const double* x, double* y, cudaStream_t s) {
  if (op.n == 0) return IBF_OK;
  static int tma = -1;
  if (tma < 0) tma = getenv("IBF_SPMV_TMA") ? atoi(getenv("IBF_SPMV_TMA")) : 0;
  if (tma && SELL_C == 32 && !op.contact.n && !op.friction.n) {
    // experimental (measured): TMA-staged upper stream
    const int grid = (int)std::min<int64_t>(div_up(op.n, 32 * TMA_WARPS), (int64_t)tma * sm_count());
    k_spmv_tma<<<grid, 32 * TMA_WARPS, 0, s>>>(op, x, y);
    IBF_LAUNCH_CHECK();
    return IBF_OK;
  }
  if (op.contact.n || op.friction.n) {
    k_contact_dot<<<(int)div_up(std::max(op.contact.n, op.friction.n), 256), 256, 0, s>>>(op, x);
    IBF_LAUNCH_CHECK();
  }
  // two CTAs per SM sweep the rows in ascending order: a small in-flight
  // window keeps each block's transposed re-read an L2 hit
  const int grid = (int)std::min<int64_t>(div_up(op.n, 256), 2LL * sm_count());
  k_spmv<<<grid, 256, 0, s>>>(op, x, y);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

// ----------------------------------------------------------- 3x3 inverses

__global__ void k_invert_diag(int n, const double* __restrict__ val, const int* __restrict__ diag_q,
                              double* __restrict__ pinv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double A[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const int q = diag_q[i];
    if (q >= 0)
      for (int k = 0; k < 9; ++k) A[k] = val[qel(q, k)];
    inv3_sym6(A, pinv + PINV_STRIDE * (size_t)i);
  }
}

int invert_diag_blocks(int n, const double* val, const int* diag_q, double* pinv, cudaStream_t s) {
  if (n == 0) return IBF_OK;
  k_invert_diag<<<(int)div_up(n, 256), 256, 0, s>>>(n, val, diag_q, pinv);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

// ------------------------------------------------------- persistent PCG

struct PcgArgs {
  Operator op;
  const double* rhs;
  double* x_out;
  double* r;
  double* z;
  double* p[2];     // CG directions, alternating
  double* hp;       // H p (global fallback when the rows do not fit in smem)
  double* X;        // 3 iterate buffers of 3n
  double* part;     // 4 * gridDim partial sums
  double* info;     // (iterations, converged, rel_res)
  double tol;
  int64_t max_iters;
  unsigned long long* prof;  // IBF_PCG_PROFILE builds: per-CTA phase nanoseconds (G,6)
  int* counter;         // dynamic phase A: chunk counters (2, alternating iterations)
  double* part_chunk;   // dynamic phase A: per-chunk p.q partials
  int n_chunks;         // dynamic phase A: chunks of blockDim rows (0: static mapping)
  int rows_per_thread;  // ceil(n / (grid * block))
  int smem_rows;        // rows_per_thread if the carry lives in shared memory, else 0
  int carry_qp;         // with smem_rows: 1 carries r, q and p; 0 carries r only
  unsigned* ready;      // term-dot ready counter, or null: grid barrier after the dots
  unsigned* bar;        // split-barrier arrival counter (phase B), or null: grid barrier
  int lanes;            // lanes per row in phase A (1: one thread per row)
  unsigned n_home;      // CTAs that compute term dots (each adds 1 per iteration)
  double* zdot;         // zdot mode (contacts without a dot phase): (C,4) g_c[slot] . z
  double* pdot;         // (C,4) each record's copy of g_c . p_{k-1}
  int zmode;
  int pmat;             // materialised direction this solve (IBF_PCG_PMAT and enough contact terms)
  double* tprev;        // (C) g_c . p_{k-1} for the linear-recursion dots, or null
  int wdyn;             // warp-granular dynamic phase A (IBF_PCG_WARPDYN)
  int n_units, n_groups;
  int* wcounter;        // (2) slice counters, alternating iterations
  int* gcount;          // (n_groups) finished slices per group
  double* part_unit;    // (n_units) per-slice p.q partials
  double* part_group;   // (n_groups) per-group sums
};

// all CTAs compute the same fixed-order total of part[slot*G .. slot*G+G)
__device__ __forceinline__ double grid_total(const double* part, int slot, double* sh) {
  const int G = gridDim.x;
  if (threadIdx.x < 32) {
    const double v = warp_sum_array(part + (size_t)slot * G, G);
    if (threadIdx.x == 0) sh[0] = v;
  }
  __syncthreads();
  const double v = sh[0];
  __syncthreads();
  return v;
}

// publish this CTA's partials of `k` sums into part[slot_j * G + b]
__device__ __forceinline__ void put_partials(double* part, int slot, double v, double* red) {
  v = block_sum(v, red);
  if (threadIdx.x == 0) part[(size_t)slot * gridDim.x + blockIdx.x] = v;
}

#ifndef IBF_PCG_PROFILE
#define IBF_PCG_PROFILE 0
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// phase timers of a profiling build: [0] term dots + barrier, [1] A work,
// [2] A barrier + reduction, [3] B work, [4] B barrier + reduction, [5] iterations
#define PCG_PT(slot)                                   \
  if (IBF_PCG_PROFILE && threadIdx.x == 0) {           \
    const unsigned long long t_ = gtimer();            \
    prof[slot] += t_ - t_last;                         \
    t_last = t_;                                       \
  }

__global__ void __launch_bounds__(PCG_THREADS, IBF_PCG_MINB) k_pcg(PcgArgs a) {
  unsigned long long prof[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long t_last = IBF_PCG_PROFILE ? gtimer() : 0;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double dyn[];
  __shared__ double red[32];
  __shared__ double bc[1];
  __shared__ double term_buf[(PCG_THREADS / 32) * 3 * TERM_CHUNK];
  double* wbuf = term_buf + (threadIdx.x >> 5) * 3 * TERM_CHUNK;
  const bool zmode = IBF_PCG_ZDOT && a.zmode != 0;
  double dummy[3] = {0.0, 0.0, 0.0};
  const Operator& op = a.op;
  const int n = op.n;
  const int S = gridDim.x * blockDim.x;          // rows per sweep
  const int R = a.rows_per_thread;
  const bool in_smem = a.smem_rows > 0;
  const bool qp_smem = in_smem && a.carry_qp;
  // per-thread row slots: row(k) = blockIdx.x*blockDim.x + threadIdx.x + k*S
  double* sq = dyn;                                  // (R, 3, blockDim) H p
  double* sp = dyn + 3 * (size_t)R * blockDim.x;     // (R, 3, blockDim) p
  double* sr = dyn + (a.carry_qp ? 6 : 0) * (size_t)R * blockDim.x;   // (R, 3, blockDim) residual
  auto slot = [&](int k, int c) { return ((size_t)k * 3 + c) * blockDim.x + threadIdx.x; };
  // the residual is only ever touched by its row's owner: keep it on chip
  auto r_ref = [&](int k, int i, int c) -> double& { return in_smem ? sr[slot(k, c)] : a.r[3 * (size_t)i + c]; };
  // Row of this thread in sweep k.  Full sweeps give each CTA a contiguous
  // block of blockDim rows; the last, partial sweep is dealt out by 32-row
  // slices round-robin over the CTAs (slice = warp * G + CTA), so every CTA
  // (and SM) gets the same share of it instead of the low CTAs taking it all
  // (a ~10 % per-SM imbalance at C4 size otherwise).
  auto row_of = [&](int k) {
    if (k < R - 1) return k * S + blockIdx.x * blockDim.x + threadIdx.x;
    const int slice = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    return (R - 1) * S + 32 * slice + (threadIdx.x & 31);
  };
  auto Xb = [&](int k) { return a.X + (size_t)k * 3 * n; };

  // ---- r = b, z = P^-1 r, x = 0
  double acc_b = 0.0, acc_rz = 0.0;
  for (int k = 0; k < R; ++k) {
    const int pos = row_of(k);
    if (zmode) {
      if (__all_sync(0xffffffffu, pos >= n)) break;
      if (pos >= n) {
        const double z0[3] = {0.0, 0.0, 0.0};
        warp_zdot(op.contact, pos & ~31, n, z0, wbuf, a.zdot);
        continue;
      }
    } else if (pos >= n) {
      break;
    }
    const int i = row_at(op, pos);
    const double r0 = a.rhs[3 * (size_t)i], r1 = a.rhs[3 * (size_t)i + 1], r2 = a.rhs[3 * (size_t)i + 2];
    double zv[3];
    apply_pinv6(op.pinv + PINV_STRIDE * (size_t)i, r0, r1, r2, zv);
    if (zmode) warp_zdot(op.contact, pos & ~31, n, zv, wbuf, a.zdot);
    double* zi = a.z + 3 * (size_t)i;
    double* xi = Xb(0) + 3 * (size_t)i;
    r_ref(k, i, 0) = r0;
    r_ref(k, i, 1) = r1;
    r_ref(k, i, 2) = r2;
    zi[0] = zv[0]; zi[1] = zv[1]; zi[2] = zv[2];
    xi[0] = 0.0; xi[1] = 0.0; xi[2] = 0.0;
    acc_b += r0 * r0 + r1 * r1 + r2 * r2;
    acc_rz += r0 * zv[0] + r1 * zv[1] + r2 * zv[2];
  }
  put_partials(a.part, 0, acc_b, red);
  put_partials(a.part, 1, acc_rz, red);
  if (a.n_chunks && blockIdx.x == 0 && threadIdx.x == 0) a.counter[0] = a.counter[1] = 0;
  grid.sync();
  const double bnorm = sqrt(grid_total(a.part, 0, bc));
  double rz = grid_total(a.part, 1, bc);
  int cur = 0, best = 0, result = 0;
  double best_res = bnorm;
  int64_t iters = 0;
  bool conv = false;
  double rel = 0.0;
  double beta = 0.0;
  bool first = true;   // p_k = z (first iteration and after a restart)
  unsigned bar_epoch = 0;  // split barriers passed
  int pb = 0;          // p[pb] receives p_k
  if (bnorm == 0.0) {
    conv = true;
  } else {
    bool done = false;
    for (int64_t it = 1; it <= a.max_iters; ++it) {
      const DirGather gd{a.z, a.p[pb ^ 1], beta, first};
      double* pk = a.p[pb];
      PCG_PT(5)
      // materialised direction (IBF_PCG_PMAT): p_k = z + beta p_{k-1} for the
      // own rows, a grid barrier, then phase A gathers p_k alone
      const bool pmat = IBF_PCG_PMAT && a.pmat && a.lanes == 1 && !a.n_chunks && !a.wdyn && !zmode && !qp_smem;
      if (pmat) {
        for (int k = 0; k < R; ++k) {
          const int pos = row_of(k);
          if (pos >= n) break;
          const int i = row_at(op, pos);
          double pv[3];
          gd.get(i, pv[0], pv[1], pv[2]);
          double* pki = pk + 3 * (size_t)i;
          pki[0] = pv[0]; pki[1] = pv[1]; pki[2] = pv[2];
        }
        // the term dots in the same phase, on the direction formed on the fly
        // (they overlap the p_k stream); barrier P then makes them visible
        // too, so phase A reads them without the ready counter
        if (IBF_PCG_PMAT_DOTS && (op.contact.n || op.friction.n)) term_dots(op, gd, true, a.tprev);
        grid.sync();
      }
      const PlainGather gpk{pk};
      // ---- A: contact dots on p_k, then q = H p_k, pAp.  With the ready
      // counter, the CTAs holding term dots compute them first and count
      // themselves in; rows touching terms wait for the count just before
      // their term loop, instead of every CTA waiting at a grid barrier.
      const bool counted = a.ready != nullptr && !(pmat && IBF_PCG_PMAT_DOTS);
      const CountedTerms sterms{a.ready, (unsigned)it * a.n_home};
      auto product = [&](int pos, int i, double v[3]) {
        if (counted)
          row_product(op, gd, pos, i, v, sterms);
        else
          row_product(op, gd, pos, i, v);
      };
      if (((op.contact.n && !zmode) || op.friction.n) && !(pmat && IBF_PCG_PMAT_DOTS)) {
        if (counted) {
          if (blockIdx.x < a.n_home) {
            if (pmat)
              term_dots(op, gpk, true);
            else
              term_dots(op, gd, !zmode, a.tprev);
            __syncthreads();
            if (threadIdx.x == 0) {
              __threadfence();
              atomicAdd(a.ready, 1u);
            }
          }
        } else {
          if (pmat)
            term_dots(op, gpk, true);
          else
            term_dots(op, gd, !zmode, a.tprev);
          grid.sync();
        }
      }
      PCG_PT(0)
      double pap;
      if (a.n_chunks) {
        // Dynamic row chunks (blockDim rows each, handed out in ascending
        // order, so the sweep keeps its L2 locality): per-CTA speed differs
        // by up to 2x (die / L2-slice locality), and a static split makes
        // every CTA wait for the slowest at the barrier.  Each chunk's p.q
        // partial goes to its own slot, summed in chunk order, so the result
        // does not depend on which CTA took which chunk.
        if (blockIdx.x == 0 && threadIdx.x == 0) a.counter[(it + 1) & 1] = 0;
        __shared__ int chunk_sh;
        while (true) {
          if (threadIdx.x == 0) chunk_sh = atomicAdd(a.counter + (it & 1), 1);
          __syncthreads();
          const int ch = chunk_sh;
          __syncthreads();
          if (ch >= a.n_chunks) break;
          const int pos = ch * blockDim.x + threadIdx.x;
          double accc = 0.0;
          if (pos < n) {
            const int i = row_at(op, pos);
            double v[3], pv[3];
            product(pos, i, v);
            gd.get(i, pv[0], pv[1], pv[2]);
            double* pki = pk + 3 * (size_t)i;
            pki[0] = pv[0]; pki[1] = pv[1]; pki[2] = pv[2];
            double* qi = a.hp + 3 * (size_t)i;
            qi[0] = v[0]; qi[1] = v[1]; qi[2] = v[2];
            accc = pv[0] * v[0] + pv[1] * v[1] + pv[2] * v[2];
          }
          accc = block_sum(accc, red);
          if (threadIdx.x == 0) a.part_chunk[ch] = accc;
        }
        PCG_PT(1)
        grid.sync();
        {
          // whole-CTA fixed-order sum of the chunk partials (strided, then
          // the block tree): identical in every CTA, ~8 loads per thread
          double v = 0.0;
          for (int c = threadIdx.x; c < a.n_chunks; c += blockDim.x) v += a.part_chunk[c];
          pap = block_sum(v, red);
        }
        PCG_PT(2)
      } else if (a.wdyn) {
        // Warp-granular dynamic phase A (IBF_PCG_WARPDYN): each warp takes
        // the next 32-row slice with one atomic, in ascending order, so the
        // CTAs that run fast (locality, memory-latency luck: measured
        // per-CTA spread +-11 %, weakly tied to their nnz) absorb the slow
        // ones' share and the barrier waits shrink.  p.q stays deterministic:
        // a slice's partial is the warp's fixed tree sum, stored by slice;
        // the last warp to finish a group of 64 slices sums the group's 64
        // partials in slice order, and every CTA sums the group partials in
        // group order after the barrier.
        const int lane = threadIdx.x & 31;
        if (blockIdx.x == 0 && threadIdx.x == 0) a.wcounter[(it + 1) & 1] = 0;
        const bool wt = IBF_PCG_WARP_TERMS && op.contact.n && op.contact.rec && !op.perm;
        while (true) {
          int u = 0;
          if (lane == 0) u = atomicAdd(a.wcounter + (it & 1), 1);
          u = __shfl_sync(0xffffffffu, u, 0);
          if (u >= a.n_units) break;
          const int pos = 32 * u + lane;
          double pq = 0.0;
          if (pos < n) {
            const int i = row_at(op, pos);
            double v[3], pv[3];
            if (wt) {
              if (counted)
                row_product<DirGather, CountedTerms, false>(op, gd, pos, i, v, sterms);
              else
                row_product<DirGather, StoredTerms, false>(op, gd, pos, i, v);
              if (counted)
                warp_terms(op.contact, sterms, pos & ~31, n, wbuf, v[0], v[1], v[2]);
              else
                warp_terms(op.contact, StoredTerms(), pos & ~31, n, wbuf, v[0], v[1], v[2]);
            } else {
              product(pos, i, v);
            }
            gd.get(i, pv[0], pv[1], pv[2]);
            double* pki = pk + 3 * (size_t)i;
            pki[0] = pv[0]; pki[1] = pv[1]; pki[2] = pv[2];
            double* qi = a.hp + 3 * (size_t)i;
            qi[0] = v[0]; qi[1] = v[1]; qi[2] = v[2];
            pq = pv[0] * v[0] + pv[1] * v[1] + pv[2] * v[2];
          } else if (wt) {
            if (counted)
              warp_terms(op.contact, sterms, pos & ~31, n, wbuf, dummy[0], dummy[1], dummy[2]);
            else
              warp_terms(op.contact, StoredTerms(), pos & ~31, n, wbuf, dummy[0], dummy[1], dummy[2]);
          }
          pq = warp_sum(pq);
          int last = 0;
          const int g = u >> 6, gsize = min(64, a.n_units - (g << 6));
          if (lane == 0) {
            a.part_unit[u] = pq;
            __threadfence();
            last = (atomicAdd(a.gcount + g, 1) == gsize - 1);
          }
          last = __shfl_sync(0xffffffffu, last, 0);
          if (last) {
            __threadfence();
            const double* P = a.part_unit + (g << 6);
            double v = (lane < gsize ? __ldcg(P + lane) : 0.0) + (lane + 32 < gsize ? __ldcg(P + lane + 32) : 0.0);
            v = warp_sum(v);
            if (lane == 0) {
              a.part_group[g] = v;
              a.gcount[g] = 0;
            }
          }
        }
        PCG_PT(1)
        grid.sync();
        {
          double v = 0.0;
          if (threadIdx.x < 32) {
            v = warp_sum_array(a.part_group, a.n_groups);
            if (threadIdx.x == 0) bc[0] = v;
          }
          __syncthreads();
          pap = bc[0];
          __syncthreads();
        }
        PCG_PT(2)
      } else {
        double acc = 0.0;
        if (a.lanes > 1) {
          // small system: L lanes per row; warp-uniform loop for the shuffles
          const int L = a.lanes, sub = threadIdx.x & (L - 1);
          for (int base = (blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / L; base < n; base += S / L) {
            const int pos = base + (threadIdx.x & 31) / L;
            const int i = pos < n ? row_at(op, pos) : n;
            double v[3] = {0.0, 0.0, 0.0};
            if (pos < n) {
              if (counted)
                row_product_lanes(op, gd, pos, i, v, sub, L, sterms);
              else
                row_product_lanes(op, gd, pos, i, v, sub, L);
            }
            for (int o = 1; o < L; o <<= 1)
              for (int c = 0; c < 3; ++c) v[c] += __shfl_xor_sync(0xffffffffu, v[c], o);
            if (i < n && sub == 0) {
              double pv[3];
              gd.get(i, pv[0], pv[1], pv[2]);
              double* pki = pk + 3 * (size_t)i;
              pki[0] = pv[0]; pki[1] = pv[1]; pki[2] = pv[2];
              double* qi = a.hp + 3 * (size_t)i;
              qi[0] = v[0]; qi[1] = v[1]; qi[2] = v[2];
              acc += pv[0] * v[0] + pv[1] * v[1] + pv[2] * v[2];
            }
          }
        }
        // warp-cooperative contact terms: positions are rows (no SELL
        // window permutation) and the records exist for this operator
        const bool wterms = IBF_PCG_WARP_TERMS && op.contact.n && op.contact.rec && !op.perm;
        for (int k = 0; k < R && a.lanes == 1; ++k) {
          const int pos = row_of(k);
          if (wterms) {
            // the warp's 32 positions are one aligned slice: exit together
            if (__all_sync(0xffffffffu, pos >= n)) break;
          } else if (pos >= n) {
            break;
          }
          if (pos >= n) {
            if (zmode)
              warp_terms_z(op.contact, pos & ~31, n, wbuf, first, beta, a.zdot, a.pdot, dummy[0], dummy[1],
                           dummy[2]);
            else if (counted)
              warp_terms(op.contact, sterms, pos & ~31, n, wbuf, dummy[0], dummy[1], dummy[2]);
            else
              warp_terms(op.contact, StoredTerms(), pos & ~31, n, wbuf, dummy[0], dummy[1], dummy[2]);
            continue;
          }
          const int i = row_at(op, pos);
          double v[3], pv[3];
          if (zmode) {
            if (counted)
              row_product<DirGather, CountedTerms, false>(op, gd, pos, i, v, sterms);
            else
              row_product<DirGather, StoredTerms, false>(op, gd, pos, i, v);
            warp_terms_z(op.contact, pos & ~31, n, wbuf, first, beta, a.zdot, a.pdot, v[0], v[1], v[2]);
          } else if (wterms && pmat) {
            if (counted) {
              row_product<PlainGather, CountedTerms, false>(op, gpk, pos, i, v, sterms);
              warp_terms(op.contact, sterms, pos & ~31, n, wbuf, v[0], v[1], v[2]);
            } else {
              row_product<PlainGather, StoredTerms, false>(op, gpk, pos, i, v);
              warp_terms(op.contact, StoredTerms(), pos & ~31, n, wbuf, v[0], v[1], v[2]);
            }
          } else if (pmat) {
            if (counted)
              row_product(op, gpk, pos, i, v, sterms);
            else
              row_product(op, gpk, pos, i, v);
          } else if (wterms) {
            if (counted) {
              row_product<DirGather, CountedTerms, false>(op, gd, pos, i, v, sterms);
              warp_terms(op.contact, sterms, pos & ~31, n, wbuf, v[0], v[1], v[2]);
            } else {
              row_product<DirGather, StoredTerms, false>(op, gd, pos, i, v);
              warp_terms(op.contact, StoredTerms(), pos & ~31, n, wbuf, v[0], v[1], v[2]);
            }
          } else {
            product(pos, i, v);
          }
          double* pki = pk + 3 * (size_t)i;
          if (pmat) {
            pv[0] = pki[0]; pv[1] = pki[1]; pv[2] = pki[2];
          } else {
            const double* Z = a.z + 3 * (size_t)i;
            if (first) {
              pv[0] = Z[0]; pv[1] = Z[1]; pv[2] = Z[2];
            } else {
              const double* P = gd.pold + 3 * (size_t)i;
              pv[0] = cg_dir(beta, P[0], Z[0]);
              pv[1] = cg_dir(beta, P[1], Z[1]);
              pv[2] = cg_dir(beta, P[2], Z[2]);
            }
            pki[0] = pv[0]; pki[1] = pv[1]; pki[2] = pv[2];
          }
          if (qp_smem) {
            for (int c = 0; c < 3; ++c) {
              sq[slot(k, c)] = v[c];
              sp[slot(k, c)] = pv[c];
            }
          } else {
            double* qi = a.hp + 3 * (size_t)i;
            qi[0] = v[0]; qi[1] = v[1]; qi[2] = v[2];
          }
          acc += pv[0] * v[0] + pv[1] * v[1] + pv[2] * v[2];
        }
        PCG_PT(1)
        put_partials(a.part, 2, acc, red);
        grid.sync();
        pap = grid_total(a.part, 2, bc);
        PCG_PT(2)
      }
      if (pap <= 0.0) {
        // lost positive definiteness along p: keep the best iterate
        result = best;
        iters = it - 1;
        conv = false;
        rel = best_res / bnorm;
        done = true;
        break;
      }
      // ---- B: x, r, z updates
      const double alpha = rz / pap;
      const int nxt = (cur != 0 && best != 0) ? 0 : ((cur != 1 && best != 1) ? 1 : 2);
      const double* xc = Xb(cur);
      double* xn = Xb(nxt);
      double acc_rr = 0.0;
      acc_rz = 0.0;
      const bool split = a.bar != nullptr && !qp_smem;
      for (int k = 0; k < R; ++k) {
        const int pos = row_of(k);
        if (zmode) {
          if (__all_sync(0xffffffffu, pos >= n)) break;
          if (pos >= n) {
            const double z0[3] = {0.0, 0.0, 0.0};
            warp_zdot(op.contact, pos & ~31, n, z0, wbuf, a.zdot);
            continue;
          }
        } else if (pos >= n) {
          break;
        }
        const int i = row_at(op, pos);
        double qv[3], pv[3], rv[3], zv[3];
        if (qp_smem) {
          for (int c = 0; c < 3; ++c) {
            qv[c] = sq[slot(k, c)];
            pv[c] = sp[slot(k, c)];
          }
        } else {
          for (int c = 0; c < 3; ++c) qv[c] = a.hp[3 * (size_t)i + c];
          if (!split)
            for (int c = 0; c < 3; ++c) pv[c] = pk[3 * (size_t)i + c];
        }
        for (int c = 0; c < 3; ++c) {
          const size_t e = 3 * (size_t)i + c;
          if (!split) xn[e] = xc[e] + alpha * pv[c];
          double& rr = r_ref(k, i, c);
          rv[c] = rr - alpha * qv[c];
          rr = rv[c];
          acc_rr += rv[c] * rv[c];
        }
        apply_pinv6(op.pinv + PINV_STRIDE * (size_t)i, rv[0], rv[1], rv[2], zv);
        double* zi = a.z + 3 * (size_t)i;
        zi[0] = zv[0]; zi[1] = zv[1]; zi[2] = zv[2];
        if (zmode) warp_zdot(op.contact, pos & ~31, n, zv, wbuf, a.zdot);
        acc_rz += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
      }
      PCG_PT(3)
      put_partials(a.part, 0, acc_rr, red);
      put_partials(a.part, 1, acc_rz, red);
      if (split) {
        // split barrier: arrive, update x (which nothing reads before the
        // next own-row update, a restart or the end, each behind a full
        // barrier), then wait — the x stream hides the barrier latency
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          atomicAdd(a.bar, 1u);
        }
        for (int k = 0; k < R; ++k) {
          const int pos = row_of(k);
          if (pos >= n) break;
          const int i = row_at(op, pos);
          for (int c = 0; c < 3; ++c) {
            const size_t e = 3 * (size_t)i + c;
            xn[e] = xc[e] + alpha * pk[e];
          }
        }
        ++bar_epoch;
        if (threadIdx.x == 0) wait_count(a.bar, bar_epoch * gridDim.x);
        __syncthreads();
      } else {
        grid.sync();
      }
      const double res = sqrt(grid_total(a.part, 0, bc));
      PCG_PT(4)
      cur = nxt;
      if (res < best_res) {
        best_res = res;
        best = cur;
      }
      if (res <= a.tol * bnorm) {
        result = cur;
        iters = it;
        conv = true;
        rel = res / bnorm;
        done = true;
        break;
      }
      if (it % 250 == 0) {
        // restart from the true residual r = b - H x
        if (a.bar) grid.sync();   // x of other rows: updated after the split barrier's arrive
        const PlainGather gx{Xb(cur)};
        if (op.contact.n || op.friction.n) {
          term_dots(op, gx);
          grid.sync();
        }
        acc_rz = 0.0;
        for (int k = 0; k < R; ++k) {
          const int pos = row_of(k);
          if (zmode) {
            if (__all_sync(0xffffffffu, pos >= n)) break;
            if (pos >= n) {
              const double z0[3] = {0.0, 0.0, 0.0};
              warp_zdot(op.contact, pos & ~31, n, z0, wbuf, a.zdot);
              continue;
            }
          } else if (pos >= n) {
            break;
          }
          const int i = row_at(op, pos);
          double v[3], zv[3];
          row_product(op, gx, pos, i, v);
          const double r0 = a.rhs[3 * (size_t)i] - v[0];
          const double r1 = a.rhs[3 * (size_t)i + 1] - v[1];
          const double r2 = a.rhs[3 * (size_t)i + 2] - v[2];
          apply_pinv6(op.pinv + PINV_STRIDE * (size_t)i, r0, r1, r2, zv);
          double* zi = a.z + 3 * (size_t)i;
          r_ref(k, i, 0) = r0;
          r_ref(k, i, 1) = r1;
          r_ref(k, i, 2) = r2;
          zi[0] = zv[0]; zi[1] = zv[1]; zi[2] = zv[2];
          if (zmode) warp_zdot(op.contact, pos & ~31, n, zv, wbuf, a.zdot);
          acc_rz += r0 * zv[0] + r1 * zv[1] + r2 * zv[2];
        }
        put_partials(a.part, 1, acc_rz, red);
        grid.sync();
        rz = grid_total(a.part, 1, bc);
        first = true;
        pb ^= 1;
        continue;
      }
      const double rz_new = grid_total(a.part, 1, bc);
      beta = rz_new / rz;
      rz = rz_new;
      first = false;
      pb ^= 1;
    }
    if (!done) {
      result = best;
      iters = a.max_iters;
      conv = false;
      rel = best_res / bnorm;
    }
  }
  if (a.bar) grid.sync();   // the last x update ran after the split barrier's arrive
  const double* xr = Xb(result);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 3LL * n; k += S)
    a.x_out[k] = (bnorm == 0.0) ? 0.0 : xr[k];
  if (IBF_PCG_PROFILE && threadIdx.x == 0 && a.prof) {
    for (int k = 0; k < 6; ++k) a.prof[8 * blockIdx.x + k] = prof[k];
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    a.prof[8 * blockIdx.x + 6] = sm;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.info[0] = (double)iters;
    a.info[1] = conv ? 1.0 : 0.0;
    a.info[2] = rel;
  }
}

#ifndef IBF_PCG_CARRY_QP
#define IBF_PCG_CARRY_QP 0
#endif
static size_t pcg_smem(int rows_per_thread, int threads) {
  return (size_t)(IBF_PCG_CARRY_QP ? 9 : 3) * rows_per_thread * threads * sizeof(double);
}

// Launch shape: a full wave of co-resident CTAs, rows_per_thread sweeps, and
// a block size trimmed (in warps) so the last sweep is nearly full — every
// CTA then carries the same number of rows and no SM idles at a barrier
// while others finish a partial sweep.
struct PcgShape {
  int grid, threads, rows_per_thread, smem_rows;
};

// Runtime overrides of the launch shape (ibf_pcg_tuning): the row count up
// to which rows get several lanes, and a cap on the CTA count (0: a full
// wave).  Tests use them to drive the one-thread-per-row path with several
// sweeps per thread on systems the oracle solves in seconds.
static std::atomic<long long> g_lanes_max_n{IBF_PCG_LANES_MAX_N};
static std::atomic<int> g_max_ctas{0};
// warp-granular dynamic phase A: IBF_PCG_WARPDYN default, the environment
// variable of the same name overrides (0 / 1) for A/B runs
#ifndef IBF_PCG_WARPDYN
#define IBF_PCG_WARPDYN 0
#endif
static int warpdyn_enabled() {
  static const int on = [] {
    const char* e = getenv("IBF_PCG_WARPDYN");
    return e ? (e[0] == '1' ? 1 : 0) : IBF_PCG_WARPDYN;
  }();
  return on;
}
// zdot mode on (IBF_PCG_ZDOT builds) unless the environment sets IBF_PCG_ZDOT=0 (A/B runs)
static int zdot_enabled() {
  static const int on = [] {
    const char* e = getenv("IBF_PCG_ZDOT");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return on;
}
// shape of the last PCG launch in the process (ibf_pcg_last_shape)
static std::atomic<long long> g_last_shape[6];

static PcgShape pcg_shape(int n) {
  static std::atomic<int> max_b_cache{-1};
  int max_b = max_b_cache.load();
  if (max_b < 0) {
    if (PCG_SMEM_BYTES > 0)
      cudaFuncSetAttribute(k_pcg, cudaFuncAttributeMaxDynamicSharedMemorySize, PCG_SMEM_BYTES);
#ifdef IBF_PCG_CARVEOUT
    // unified L1/SMEM split: the gathers want L1, the kernel needs ~1 KB SMEM per CTA
    cudaFuncSetAttribute(k_pcg, cudaFuncAttributePreferredSharedMemoryCarveout, IBF_PCG_CARVEOUT);
#endif
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pcg, PCG_THREADS, 0);
    max_b = nb > 0 ? nb : 1;
    max_b_cache.store(max_b);
  }
  n = std::max(n, 1);
  const int cap = g_max_ctas.load();
  auto shape_for = [&](int b) {
    int64_t g = std::min<int64_t>((int64_t)b * sm_count(), div_up(n, PCG_THREADS));
    if (cap > 0) g = std::min<int64_t>(g, cap);
    const int grid = (int)g;
    const int rpt = (int)div_up(n, (int64_t)grid * PCG_THREADS);
    return PcgShape{grid, PCG_THREADS, rpt, 0};
  };
  // the on-chip carry when a full wave of CTAs with it stays co-resident
  for (int b = max_b; b >= 1 && PCG_SMEM_BYTES > 0; --b) {
    PcgShape sh = shape_for(b);
    const size_t smem = pcg_smem(sh.rows_per_thread, sh.threads);
    if (smem > (size_t)PCG_SMEM_BYTES) continue;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pcg, sh.threads, smem);
    if ((int64_t)occ * sm_count() >= sh.grid) {
      sh.smem_rows = sh.rows_per_thread;
      return sh;
    }
  }
  return shape_for(max_b);
}

// L2 residency of the matrix across CG iterations: every iteration streams
// the whole matrix (221 MB at C4) through a 126 MB L2.  An access-policy
// window marks a fraction of its lines persisting, so that share stays in L2
// from one iteration to the next instead of being re-read from HBM.
// IBF_L2_PERSIST_MB sets the persisting budget (0 disables).
static size_t l2_persist_budget() {
  static long long mb = -2;
  if (mb == -2) {
    const char* e = getenv("IBF_L2_PERSIST_MB");
    mb = e ? atoll(e) : 0;
  }
  return mb > 0 ? (size_t)mb << 20 : 0;
}

// IBF_L2_VEC=1: the persisting window covers the gathered vectors (z, p)
// instead, with IBF_L2_PERSIST_MB (default 64) as the budget (experiment)
static bool l2_vec_enabled() {
  static const bool on = [] {
    const char* e = getenv("IBF_L2_VEC");
    return e && e[0] == '1';
  }();
  return on;
}

static void l2_window(cudaStream_t s, const void* base, size_t bytes, bool on) {
  static int max_persist = -1, max_window = -1;
  if (max_persist < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  }
  cudaStreamAttrValue attr = {};
  if (on) {
    const size_t want = l2_persist_budget() ? l2_persist_budget() : ((size_t)64 << 20);
    const size_t budget = std::min<size_t>(want, (size_t)max_persist);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, budget);
    const size_t win = std::min<size_t>(bytes, (size_t)max_window);
    attr.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr.accessPolicyWindow.num_bytes = win;
    attr.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)budget / (double)std::max<size_t>(win, 1));
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &attr);
  cudaGetLastError();  // the window is a hint: never fail the solve on it
}

int pcg_solve(const Operator& op, const double* rhs, double* x_out, double rel_tol, int64_t max_iters,
              PcgWork& w, cudaStream_t s) {
  const int n = op.n;
  if (max_iters <= 0) max_iters = 10LL * n;
  const size_t n3 = 3 * (size_t)std::max(n, 1);
  IBF_TRY(w.r.reserve(n3));
  // z and both directions in one allocation (the gathered vectors; an L2
  // persisting window can cover them, IBF_L2_VEC)
  IBF_TRY(w.p.reserve(3 * n3));
  IBF_TRY(w.hp.reserve(n3));
  IBF_TRY(w.X.reserve(3 * n3));
  IBF_TRY(w.info.reserve(4));
  const int lanes = (IBF_PCG_LANES > 1 && !IBF_PCG_CARRY_QP && n <= g_lanes_max_n.load()) ? IBF_PCG_LANES : 1;
  PcgShape sh = pcg_shape(n * lanes);   // grid sized for lanes x rows threads
  if (lanes > 1) {
    sh.rows_per_thread = (int)div_up(std::max(n, 1), (int64_t)sh.grid * sh.threads);
    if (sh.smem_rows) sh.smem_rows = sh.rows_per_thread;
  }
  IBF_TRY(w.part.reserve(4 * (size_t)sh.grid));
  w.grid = sh.grid;
  PcgArgs a;
  a.op = op;
  a.rhs = rhs;
  a.x_out = x_out;
  a.r = w.r.p;
  a.z = w.p.p + 2 * n3;
  a.p[0] = w.p.p;
  a.p[1] = w.p.p + n3;
  a.hp = w.hp.p;
  a.X = w.X.p;
  a.part = w.part.p;
  a.info = w.info.p;
  a.tol = rel_tol;
  a.max_iters = max_iters;
  a.rows_per_thread = sh.rows_per_thread;
  a.smem_rows = sh.smem_rows;
  a.carry_qp = IBF_PCG_CARRY_QP;
  a.n_chunks = 0;
  a.counter = nullptr;
  a.part_chunk = nullptr;
  if (IBF_PCG_DYNAMIC && !sh.smem_rows) {
    a.n_chunks = (int)div_up(std::max(n, 1), sh.threads);
    IBF_TRY(w.counter.reserve(2));
    IBF_TRY(w.part_chunk.reserve(a.n_chunks));
    a.counter = w.counter.p;
    a.part_chunk = w.part_chunk.p;
  }
  a.ready = nullptr;
  a.n_home = 0;
  IBF_TRY(w.ready.reserve(2));
  IBF_CUDA(cudaMemsetAsync(w.ready.p, 0, 2 * sizeof(unsigned), s));
  a.bar = IBF_PCG_SPLIT_BAR ? w.ready.p + 1 : nullptr;
  a.lanes = lanes;
  // contacts without a dot phase: one thread per row, rows = positions, term records built
  a.zmode = (IBF_PCG_ZDOT && IBF_PCG_WARP_TERMS && lanes == 1 && !a.n_chunks && op.contact.n && op.contact.rec &&
             !op.perm && zdot_enabled())
                ? 1
                : 0;
  a.zdot = a.pdot = nullptr;
  // The materialised direction pays a third grid barrier and saves the
  // dot phase's second gather and the direction's on-the-fly registers.
  // Before rows stopped at their padding it paid off only under heavy
  // contact (192.5 vs 184.8 us per CG iteration without contacts); with the
  // row stop it wins at every contact load measured (167 vs 187 us at 0.05
  // terms per row, 177 vs 196 at 0.15, 204 vs 227 at 0.37), so it is taken
  // whenever there is one thread per row.  IBF_PCG_PMAT_RATIO (terms per
  // row, default 0) keeps the on-the-fly direction below a given load.
  {
    const char* e = getenv("IBF_PCG_PMAT_RATIO");
    const double ratio = e ? atof(e) : 0.0;
    a.pmat = (IBF_PCG_PMAT && lanes == 1 && (double)op.contact.n >= ratio * (double)n) ? 1 : 0;
  }
  if (a.zmode) {
    const size_t nc4 = 4 * (size_t)op.contact.n;
    IBF_TRY(w.zdot.reserve(nc4));
    IBF_TRY(w.pdot.reserve(nc4));
    IBF_CUDA(cudaMemsetAsync(w.zdot.p, 0, nc4 * sizeof(double), s));
    a.zdot = w.zdot.p;
    a.pdot = w.pdot.p;
  }
  a.wdyn = 0;
  a.n_units = a.n_groups = 0;
  a.wcounter = a.gcount = nullptr;
  a.part_unit = a.part_group = nullptr;
  if (warpdyn_enabled() && lanes == 1 && !a.n_chunks && !IBF_PCG_CARRY_QP && !a.zmode) {
    a.wdyn = 1;
    a.n_units = (int)div_up(std::max(n, 1), 32);
    a.n_groups = (int)div_up(a.n_units, 64);
    IBF_TRY(w.wcounter.reserve(2 + (size_t)a.n_groups));
    IBF_TRY(w.part_unit.reserve((size_t)a.n_units + a.n_groups));
    IBF_CUDA(cudaMemsetAsync(w.wcounter.p, 0, (2 + (size_t)a.n_groups) * sizeof(int), s));
    a.wcounter = w.wcounter.p;
    a.gcount = w.wcounter.p + 2;
    a.part_unit = w.part_unit.p;
    a.part_group = w.part_unit.p + a.n_units;
  }
  a.tprev = nullptr;
  if (IBF_PCG_DOT_REC && op.contact.n && !a.zmode) {
    IBF_TRY(w.tprev.reserve(op.contact.n));
    a.tprev = w.tprev.p;
  }
  const int64_t n_dot_terms = std::max<int64_t>(a.zmode ? 0 : op.contact.n, op.friction.n);
  if (IBF_PCG_READY && n_dot_terms) {
    a.ready = w.ready.p;
    a.n_home = (unsigned)std::min<int64_t>(sh.grid, div_up(n_dot_terms, sh.threads));
  }
  a.prof = nullptr;
  if (IBF_PCG_PROFILE) {
    IBF_TRY(w.prof.reserve(8 * (size_t)sh.grid));
    a.prof = w.prof.p;
  }
  const size_t smem = sh.smem_rows ? pcg_smem(sh.smem_rows, sh.threads) : 0;
  void* args[] = {&a};
  const bool persist = l2_persist_budget() > 0 && op.val_bytes > 0;
  if (persist) l2_window(s, op.val, op.val_bytes, true);
  const bool vec_persist = !persist && l2_vec_enabled();
  if (vec_persist) l2_window(s, w.p.p, 3 * n3 * sizeof(double), true);
  IBF_CUDA(cudaLaunchCooperativeKernel((void*)k_pcg, sh.grid, sh.threads, args, smem, s));
  g_last_shape[0].store(sh.grid);
  g_last_shape[1].store(sh.threads);
  g_last_shape[2].store(sh.rows_per_thread);
  g_last_shape[3].store(lanes);
  g_last_shape[4].store(a.ready ? 1 : 0);
  g_last_shape[5].store((long long)op.contact.n + op.friction.n);
  if (persist) l2_window(s, op.val, op.val_bytes, false);
  if (vec_persist) l2_window(s, w.p.p, 3 * n3 * sizeof(double), false);
  ++g_launches;
  if (IBF_PCG_PROFILE) {
    std::vector<unsigned long long> h(8 * (size_t)sh.grid);
    IBF_CUDA(cudaMemcpyAsync(h.data(), w.prof.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaStreamSynchronize(s));
    double mean[6] = {0}, mx[6] = {0}, mn[6] = {1e30, 1e30, 1e30, 1e30, 1e30, 1e30};
    for (int b = 0; b < sh.grid; ++b)
      for (int k = 0; k < 6; ++k) {
        const double v = 1e-3 * (double)h[8 * b + k];
        mean[k] += v / sh.grid;
        mx[k] = std::max(mx[k], v);
        mn[k] = std::min(mn[k], v);
      }
    fprintf(stderr, "[ibf] pcg phases us (mean/min/max over CTAs): dots %.1f/%.1f/%.1f  A %.1f/%.1f/%.1f  "
                    "Abar %.1f/%.1f/%.1f  B %.1f/%.1f/%.1f  Bbar %.1f/%.1f/%.1f  loop %.1f/%.1f/%.1f\n",
            mean[0], mn[0], mx[0], mean[1], mn[1], mx[1], mean[2], mn[2], mx[2], mean[3], mn[3], mx[3], mean[4],
            mn[4], mx[4], mean[5], mn[5], mx[5]);
    // per-CTA rows (cta, sm, 6 phase totals in ns) for offline analysis
    if (const char* path = getenv("IBF_PCG_PROFILE_OUT")) {
      if (FILE* f = fopen(path, "a")) {
        for (int b = 0; b < sh.grid; ++b) {
          fprintf(f, "%d %llu", b, h[8 * b + 6]);
          for (int k = 0; k < 6; ++k) fprintf(f, " %llu", h[8 * b + k]);
          fprintf(f, "\n");
        }
        fprintf(f, "#\n");
        fclose(f);
      }
    }
  }
  return IBF_OK;
}

int pcg_info(PcgWork& w, double info[3], cudaStream_t s) {
  IBF_TRY(w.host.reserve(4 * sizeof(double)));
  IBF_CUDA(cudaMemcpyAsync(w.host.p, w.info.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  const double* h = (const double*)w.host.p;
  info[0] = h[0];
  info[1] = h[1];
  info[2] = h[2];
  return IBF_OK;
}

}  // namespace ibf

namespace ibf {

// Sliced-ELL pattern from real blocks sorted by (row, col) (internal.cuh).
int SellPattern::build(int64_t n_, const std::vector<int64_t>& rows_, const std::vector<int64_t>& cols_) {
  n = n_;
  rows = rows_;
  cols = cols_;
  nb = (int64_t)rows.size();
  n_slices = (int)div_up(n, SELL_C);
  const int S = n_slices;
  // per-row upper counts and the transpose lists (source rows ascending)
  std::vector<int> up(n + 1, 0), lo(n + 1, 0);
  nl = 0;
  for (int64_t b = 0; b < nb; ++b) {
    up[rows[b] + 1]++;
    if (rows[b] != cols[b]) {
      lo[cols[b] + 1]++;
      ++nl;
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    up[i + 1] += up[i];
    lo[i + 1] += lo[i];
  }
  auto ucount = [&](int64_t i) { return up[i + 1] - up[i]; };
  auto lcount = [&](int64_t i) { return lo[i + 1] - lo[i]; };
  // storage positions: windows of SELL_WINDOW rows sorted by (upper, lower)
  // slot counts, descending; ties keep row order
  perm_h.resize(n);
  std::vector<int> pos_of(n);
  for (int64_t w0 = 0; w0 < n; w0 += SELL_WINDOW) {
    const int64_t w1 = std::min<int64_t>(n, w0 + SELL_WINDOW);
    for (int64_t i = w0; i < w1; ++i) perm_h[i] = (int)i;
    std::stable_sort(perm_h.begin() + w0, perm_h.begin() + w1, [&](int a, int b) {
      return ucount(a) != ucount(b) ? ucount(a) > ucount(b) : lcount(a) > lcount(b);
    });
  }
  for (int64_t p = 0; p < n; ++p) pos_of[perm_h[p]] = (int)p;
  std::vector<int> sp(S + 1, 0), lp(S + 1, 0);
  for (int s = 0; s < S; ++s) {
    int w = 0, lw = 0;
    for (int64_t p = (int64_t)SELL_C * s; p < std::min<int64_t>(n, (int64_t)SELL_C * s + SELL_C); ++p) {
      w = std::max(w, ucount(perm_h[p]));
      lw = std::max(lw, lcount(perm_h[p]));
    }
    sp[s + 1] = sp[s] + SELL_C * w;
    lp[s + 1] = lp[s] + SELL_C * lw;
  }
  nq = sp[S];
  nlq = lp[S];
  zero_q = (int)nq;  // first block of the zero slice appended after the last
  if (nq + 32 >= (1LL << 31) || nlq >= (1LL << 31)) {
    set_error("sliced BSR: more than 2^31 storage blocks");
    return IBF_ERR_BAD_ARG;
  }
  std::vector<int> qc(nq + 32), qr(nq + 32), dq(n, -1);
  std::vector<uint8_t> qre(nq + 32, 0);
  for (int64_t q = 0; q < nq + 32; ++q) qc[q] = qr[q] = 0;
  // padding: the position's own row (positions past n in the last slice keep
  // row/col 0, zero values)
  for (int s = 0; s < S; ++s) {
    const int w = (sp[s + 1] - sp[s]) / SELL_C;
    for (int k = 0; k < w; ++k)
      for (int l = 0; l < SELL_C; ++l) {
        const int64_t p = (int64_t)SELL_C * s + l;
        const int64_t q = sp[s] + (int64_t)SELL_C * k + l;
        qc[q] = qr[q] = (p < n) ? perm_h[p] : 0;
      }
  }
  q_of_b.assign(nb, 0);
  for (int64_t i = 0; i < n; ++i) {
    const int p = pos_of[i];
    const int s = p >> SELL_SHIFT, l = p & (SELL_C - 1);
    for (int k = 0; k < ucount(i); ++k) {
      const int64_t b = up[i] + k;
      const int q = sp[s] + SELL_C * k + l;
      q_of_b[b] = q;
      qc[q] = (int)cols[b];
      qr[q] = (int)rows[b];
      qre[q] = 1;
      if (rows[b] == cols[b]) dq[i] = q;
    }
  }
  // lower entries: real off-diagonal blocks grouped by column, b ascending
  // (=> source rows ascending); padding (zero block, own row)
  std::vector<int2> le(std::max<int64_t>(nlq, 1));
  for (int s = 0; s < S; ++s) {
    const int w = (lp[s + 1] - lp[s]) / SELL_C;
    for (int t = 0; t < w; ++t)
      for (int l = 0; l < SELL_C; ++l) {
        const int64_t p = (int64_t)SELL_C * s + l;
        le[lp[s] + (int64_t)SELL_C * t + l] = make_int2(zero_q, (p < n) ? perm_h[p] : 0);
      }
  }
  std::vector<int> fill(n, 0);
  for (int64_t b = 0; b < nb; ++b) {
    if (rows[b] == cols[b]) continue;
    const int64_t j = cols[b];
    const int p = pos_of[j];
    const int s = p >> SELL_SHIFT, l = p & (SELL_C - 1);
    const int t = fill[j]++;
    le[lp[s] + (int64_t)SELL_C * t + l] = make_int2(q_of_b[b], (int)rows[b]);
  }
  if (n > 0) IBF_TRY(perm.upload(perm_h.data(), perm_h.size()));
  IBF_TRY(slice_ptr.upload(sp.data(), sp.size()));
  IBF_TRY(low_ptr.upload(lp.data(), lp.size()));
  IBF_TRY(col.upload(qc.data(), qc.size()));
  IBF_TRY(qrow.upload(qr.data(), qr.size()));
  IBF_TRY(qreal.upload(qre.data(), qre.size()));
  IBF_TRY(diag_q.upload(dq.data(), dq.size()));
  IBF_TRY(low.upload(le.data(), le.size()));
  IBF_TRY(val.reserve(9 * (size_t)(nq + 32)));
  IBF_CUDA(cudaMemset(val.p, 0, val.cap * sizeof(double)));
  return IBF_OK;
}

Operator SellPattern::op() const {
  Operator o;
  o.n = (int)n;
  o.perm = SELL_WINDOW > 1 ? perm.p : nullptr;   // identity: no lookup
  o.zero_q = zero_q;
  o.slice_ptr = slice_ptr.p;
  o.col = col.p;
  o.val = val.p;
  o.val_bytes = 9 * sizeof(double) * (size_t)(nq + 32);
  o.low_ptr = low_ptr.p;
  o.low = low.p;
  return o;
}

// host (nb,9) blocks in sorted order -> qel layout (padding zero)
static void to_sell(const SellPattern& P, const double* blocks, std::vector<double>& out) {
  out.assign(9 * (size_t)(P.nq + 32), 0.0);
  for (int64_t b = 0; b < P.nb; ++b)
    for (int e = 0; e < 9; ++e) out[qel(P.q_of_b[b], e)] = blocks[9 * b + e];
}
static void from_sell(const SellPattern& P, const std::vector<double>& in, double* blocks) {
  for (int64_t b = 0; b < P.nb; ++b)
    for (int e = 0; e < 9; ++e) blocks[9 * b + e] = in[qel(P.q_of_b[b], e)];
}

__global__ void k_mask_dirichlet(int64_t nq, const int* __restrict__ qrow, const int* __restrict__ col,
                                 const uint8_t* __restrict__ qreal, const uint8_t* __restrict__ mask,
                                 const double* __restrict__ diag, double* __restrict__ val) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    if (!qreal[q]) continue;
    const int r = qrow[q], c = col[q];
    if (!(mask[r] || mask[c])) continue;
    for (int k = 0; k < 9; ++k) val[qel((int)q, k)] = (r == c) ? diag[9 * (int64_t)r + k] : 0.0;
  }
}

int sell_export(const SellPattern& P, int64_t* rows, int64_t* cols, double* blocks, cudaStream_t s) {
  std::copy(P.rows.begin(), P.rows.end(), rows);
  std::copy(P.cols.begin(), P.cols.end(), cols);
  std::vector<double> hv(9 * (size_t)(P.nq + 32));
  IBF_CUDA(cudaMemcpyAsync(hv.data(), P.val.p, hv.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  from_sell(P, hv, blocks);
  return IBF_OK;
}
}  // namespace ibf

// ===================================================== standalone BSR handle

struct ibf_bsr {
  ibf::SellPattern pat;
  ibf::DevBuf<double> pinv;
  ibf::PcgWork work;
  ibf::Operator op() const {
    ibf::Operator o = pat.op();
    o.pinv = pinv.p;
    return o;
  }
};

using namespace ibf;

extern "C" int ibf_bsr_create(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                              const double* blocks, ibf_bsr** out) {
  if (n < 0 || nnz < 0 || !out || n >= (1LL << 30)) {
    set_error("ibf_bsr_create: bad arguments");
    return IBF_ERR_BAD_ARG;
  }
  for (int64_t k = 0; k < nnz; ++k)
    if (rows[k] < 0 || rows[k] >= n || cols[k] < 0 || cols[k] >= n) {
      set_error("ibf_bsr_create: index out of range");
      return IBF_ERR_BAD_ARG;
    }
  // stable sort by row*n+col, sequential coalescing (np.add.reduceat semantics)
  std::vector<int64_t> order(nnz);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return rows[a] * n + cols[a] < rows[b] * n + cols[b];
  });
  std::vector<int64_t> R, Cc;
  std::vector<double> vals;
  for (int64_t k = 0; k < nnz; ++k) {
    const int64_t s = order[k];
    const int64_t key = rows[s] * n + cols[s];
    if (k == 0 || key != R.back() * n + Cc.back()) {
      R.push_back(rows[s]);
      Cc.push_back(cols[s]);
      vals.insert(vals.end(), blocks + 9 * s, blocks + 9 * s + 9);
    } else {
      double* dst = vals.data() + vals.size() - 9;
      for (int e = 0; e < 9; ++e) dst[e] += blocks[9 * s + e];
    }
  }
  ibf_bsr* m = new ibf_bsr();
  int st = m->pat.build(n, R, Cc);
  std::vector<double> sv;
  if (st == IBF_OK) {
    to_sell(m->pat, vals.data(), sv);
    st = m->pat.val.upload(sv.data(), sv.size());
  }
  if (st == IBF_OK) st = m->pinv.reserve(PINV_STRIDE * (size_t)std::max<int64_t>(n, 1));
  if (st == IBF_OK) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      set_error(cudaGetErrorString(e));
      st = IBF_ERR_CUDA;
    }
  }
  if (st != IBF_OK) {
    delete m;
    return st;
  }
  *out = m;
  return IBF_OK;
}

extern "C" void ibf_bsr_destroy(ibf_bsr* m) { delete m; }

extern "C" int ibf_bsr_matvec(ibf_bsr* m, const double* x, double* y, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  return spmv(m->op(), x, y, (cudaStream_t)st);
}

extern "C" int ibf_bsr_mask_dirichlet(ibf_bsr* m, const uint8_t* vertex_mask, const double* diag, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  DevBuf<uint8_t> dm;
  DevBuf<double> dd;
  IBF_TRY(dm.upload(vertex_mask, (size_t)m->pat.n, s));
  IBF_TRY(dd.upload(diag, 9 * (size_t)m->pat.n, s));
  const int64_t nq = m->pat.nq;
  if (nq) {
    k_mask_dirichlet<<<(int)div_up(nq, 256), 256, 0, s>>>(nq, m->pat.qrow.p, m->pat.col.p, m->pat.qreal.p, dm.p,
                                                           dd.p, m->pat.val.p);
    IBF_LAUNCH_CHECK();
  }
  IBF_CUDA(cudaStreamSynchronize(s));
  return IBF_OK;
}

extern "C" int ibf_bsr_pcg(ibf_bsr* m, const double* rhs, double* x_out, double rel_tol, int64_t max_iters,
                           double* info_host, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  IBF_TRY(invert_diag_blocks((int)m->pat.n, m->pat.val.p, m->pat.diag_q.p, m->pinv.p, s));
  IBF_TRY(pcg_solve(m->op(), rhs, x_out, rel_tol, max_iters, m->work, s));
  return pcg_info(m->work, info_host, s);
}

extern "C" int64_t ibf_bsr_size(const ibf_bsr* m) { return m ? m->pat.nb : 0; }

extern "C" int ibf_bsr_export(const ibf_bsr* m, int64_t* rows, int64_t* cols, double* blocks, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  return sell_export(m->pat, rows, cols, blocks, (cudaStream_t)st);
}

extern "C" int ibf_pcg_tuning(int64_t lanes_max_n, int max_ctas) {
  if (max_ctas < 0) {
    set_error("ibf_pcg_tuning: max_ctas must be >= 0");
    return IBF_ERR_BAD_ARG;
  }
  ibf::g_lanes_max_n.store(lanes_max_n < 0 ? IBF_PCG_LANES_MAX_N : lanes_max_n);
  ibf::g_max_ctas.store(max_ctas);
  return IBF_OK;
}

extern "C" int ibf_pcg_last_shape(int64_t* out) {
  for (int k = 0; k < 6; ++k) out[k] = ibf::g_last_shape[k].load();
  return IBF_OK;
}

// ================================================ row-partitioned PCG
// (internal.cuh: DistWork).  Same arithmetic as k_pcg, split at the points
// where the partitions exchange data: per CG iteration
//   A  term dots (all terms: each partition's rows may touch any), q = H p_k
//      on own rows, p_k on own + halo rows, pAp partial      -> allreduce
//   B  x, r, z on own rows, |r|^2 and r.z partials           -> allreduce
//      own z rows                                            -> allgather
// Host-driven (the exchanges sit between phases); scalars on the host.
namespace ibf {

struct PartBuf {
  int64_t r0 = 0, r1 = 0;              // own rows
  DevBuf<double> z, p[2], q, r, X, t, tf, part, scal;
  DevBuf<int> halo;                    // rows outside [r0, r1) where p must stay valid
  DevBuf<uint8_t> hflag;
  std::vector<int> halo_static;        // structural halo (pattern), built once
  int n_halo = 0;
};

DistWork::~DistWork() {
  for (PartBuf* p : parts) delete p;
}

constexpr int PD_THREADS = 256;

static int pd_grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(div_up(n, PD_THREADS), 4LL * sm_count())); }

__global__ void k_pd_init(Operator op, int64_t r0, int64_t r1, const double* __restrict__ rhs, double* __restrict__ r,
                          double* __restrict__ z, double* __restrict__ x, double* __restrict__ part) {
  __shared__ double red[32];
  double bb = 0.0, rz = 0.0;
  for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x) {
    const double b0 = rhs[3 * i], b1 = rhs[3 * i + 1], b2 = rhs[3 * i + 2];
    double zv[3];
    apply_pinv6(op.pinv + PINV_STRIDE * i, b0, b1, b2, zv);
    r[3 * i] = b0; r[3 * i + 1] = b1; r[3 * i + 2] = b2;
    z[3 * i] = zv[0]; z[3 * i + 1] = zv[1]; z[3 * i + 2] = zv[2];
    x[3 * i] = 0.0; x[3 * i + 1] = 0.0; x[3 * i + 2] = 0.0;
    bb += b0 * b0 + b1 * b1 + b2 * b2;
    rz += b0 * zv[0] + b1 * zv[1] + b2 * zv[2];
  }
  bb = block_sum(bb, red);
  rz = block_sum(rz, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = bb;
    part[gridDim.x + blockIdx.x] = rz;
  }
}

// fixed-order sums of `slots` rows of G block partials -> out[slot]
__global__ void k_pd_sum(const double* __restrict__ part, int G, int slots, double* __restrict__ out) {
  const int slot = threadIdx.x >> 5;
  if (slot < slots) {
    const double v = warp_sum_array(part + (size_t)slot * G, G);
    if ((threadIdx.x & 31) == 0) out[slot] = v;
  }
}

// out[k] = sum over partitions (in partition order) of parts[j][k]
__global__ void k_pd_sum_parts(const double* const* __restrict__ parts, int np, int count, double* __restrict__ out) {
  const int k = threadIdx.x;
  if (k < count) {
    double v = 0.0;
    for (int j = 0; j < np; ++j) v += parts[j][k];
    out[k] = v;
  }
}

__global__ void k_pd_dots(Operator op, DirGather gd) { term_dots(op, gd); }
__global__ void k_pd_dots_plain(Operator op, PlainGather gx) { term_dots(op, gx); }

__global__ void __launch_bounds__(PD_THREADS) k_pd_a(Operator op, DirGather gd, int64_t r0, int64_t r1,
                                                     double* __restrict__ pk, double* __restrict__ q,
                                                     const int* __restrict__ halo, int nh, double* __restrict__ part) {
  __shared__ double red[32];
  double acc = 0.0;
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1; i += S) {
    double v[3], pv[3];
    row_product(op, gd, (int)i, (int)i, v);
    gd.get((int)i, pv[0], pv[1], pv[2]);
    pk[3 * i] = pv[0]; pk[3 * i + 1] = pv[1]; pk[3 * i + 2] = pv[2];
    q[3 * i] = v[0]; q[3 * i + 1] = v[1]; q[3 * i + 2] = v[2];
    acc += pv[0] * v[0] + pv[1] * v[1] + pv[2] * v[2];
  }
  // p_k on the halo: the same fused z + beta p as every reader forms
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nh; k += S) {
    const int j = halo[k];
    double pv[3];
    gd.get(j, pv[0], pv[1], pv[2]);
    pk[3 * (size_t)j] = pv[0]; pk[3 * (size_t)j + 1] = pv[1]; pk[3 * (size_t)j + 2] = pv[2];
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(PD_THREADS) k_pd_b(Operator op, int64_t r0, int64_t r1, double alpha,
                                                     const double* __restrict__ pk, const double* __restrict__ q,
                                                     double* __restrict__ r, double* __restrict__ z,
                                                     const double* __restrict__ xc, double* __restrict__ xn,
                                                     double* __restrict__ part) {
  __shared__ double red[32];
  double rr = 0.0, rz = 0.0;
  for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x) {
    double rv[3], zv[3];
    for (int c = 0; c < 3; ++c) {
      const size_t e = 3 * (size_t)i + c;
      xn[e] = xc[e] + alpha * pk[e];
      rv[c] = r[e] - alpha * q[e];
      r[e] = rv[c];
      rr += rv[c] * rv[c];
    }
    apply_pinv6(op.pinv + PINV_STRIDE * i, rv[0], rv[1], rv[2], zv);
    z[3 * i] = zv[0]; z[3 * i + 1] = zv[1]; z[3 * i + 2] = zv[2];
    rz += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
  }
  rr = block_sum(rr, red);
  rz = block_sum(rz, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = rr;
    part[gridDim.x + blockIdx.x] = rz;
  }
}

// restart: r = b - H x (x full), z = P^-1 r, r.z partials
__global__ void __launch_bounds__(PD_THREADS) k_pd_restart(Operator op, PlainGather gx, int64_t r0, int64_t r1,
                                                           const double* __restrict__ rhs, double* __restrict__ r,
                                                           double* __restrict__ z, double* __restrict__ part) {
  __shared__ double red[32];
  double rz = 0.0;
  for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x) {
    double v[3], zv[3], rv[3];
    row_product(op, gx, (int)i, (int)i, v);
    for (int c = 0; c < 3; ++c) {
      rv[c] = rhs[3 * i + c] - v[c];
      r[3 * i + c] = rv[c];
    }
    apply_pinv6(op.pinv + PINV_STRIDE * i, rv[0], rv[1], rv[2], zv);
    z[3 * i] = zv[0]; z[3 * i + 1] = zv[1]; z[3 * i + 2] = zv[2];
    rz += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
  }
  rz = block_sum(rz, red);
  if (threadIdx.x == 0) part[blockIdx.x] = rz;
}

// halo of a partition: static (pattern) rows plus every term vertex outside [r0, r1)
__global__ void k_pd_mark_terms(const int* __restrict__ quad, int64_t nq4, int64_t r0, int64_t r1,
                                uint8_t* __restrict__ flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nq4; k += (int64_t)gridDim.x * blockDim.x) {
    const int v = quad[k];
    if (v < r0 || v >= r1) flag[v] = 1;
  }
}
__global__ void k_pd_collect(const uint8_t* __restrict__ flag, int64_t n, int* __restrict__ out, int* __restrict__ cnt) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    if (flag[v]) out[atomicAdd(cnt, 1)] = (int)v;
}

__global__ void k_pd_copy_rows(const double* __restrict__ src, double* __restrict__ dst, int64_t r0, int64_t r1) {
  for (int64_t e = 3 * r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 3 * r1; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

}  // namespace ibf

namespace ibf {

// sum the partitions' scalars: NCCL allreduce of this rank's, or the local
// partitions' in partition order -> dw.gsc[0..count) -> host
static int pd_reduce(ibf_dist* d, DistWork& dw, int count, double* host, cudaStream_t s) {
  if (d->local) {
    // the partitions' scalar buffers never move after setup: upload their
    // addresses once
    if (dw.ptrs_n != (int)dw.parts.size()) {
      std::vector<unsigned long long> ptrs;
      for (PartBuf* p : dw.parts) ptrs.push_back((unsigned long long)p->scal.p);
      IBF_TRY(dw.ptrs.reserve(ptrs.size()));
      IBF_CUDA(cudaMemcpyAsync(dw.ptrs.p, ptrs.data(), ptrs.size() * sizeof(unsigned long long),
                               cudaMemcpyHostToDevice, s));
      IBF_CUDA(cudaStreamSynchronize(s));
      dw.ptrs_n = (int)dw.parts.size();
    }
    k_pd_sum_parts<<<1, 32, 0, s>>>(reinterpret_cast<const double* const*>(dw.ptrs.p), dw.ptrs_n, count, dw.gsc.p);
    IBF_LAUNCH_CHECK();
  } else {
    IBF_CUDA(cudaMemcpyAsync(dw.gsc.p, dw.parts[0]->scal.p, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    IBF_TRY(dist_allreduce_sum(d, dw.gsc.p, count, s));
  }
  IBF_CUDA(cudaMemcpyAsync(host, dw.gsc.p, count * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  return IBF_OK;
}

// every partition's own rows of the full vectors v(part) -> all partitions
static int pd_allgather(ibf_dist* d, DistWork& dw, DevBuf<double> PartBuf::*vec, cudaStream_t s) {
  if (d->local) {
    for (PartBuf* a : dw.parts)
      for (PartBuf* b : dw.parts)
        if (a != b && a->r1 > a->r0)
          IBF_CUDA(cudaMemcpyAsync((b->*vec).p + 3 * a->r0, (a->*vec).p + 3 * a->r0,
                                   3 * (a->r1 - a->r0) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return IBF_OK;
  }
  PartBuf* p = dw.parts[0];
  // the own chunk (padded length) in place: send = recv + rank * chunk
  double* full = (p->*vec).p;
  return dist_allgather(d, full + 3 * p->r0, full, 3 * (size_t)dw.chunk, s);
}

int pcg_solve_dist(const Operator& op, const std::vector<int64_t>& brows, const std::vector<int64_t>& bcols,
                   const double* rhs, double* x_out, double rel_tol, int64_t max_iters, PcgWork& w, DistWork& dw,
                   ibf_dist* d, cudaStream_t s) {
  const int64_t n = op.n;
  const int W = d->world;
  if (max_iters <= 0) max_iters = 10LL * n;
  const int64_t chunk = div_up(div_up(std::max<int64_t>(n, 1), W), 32) * 32;
  const int64_t npad = chunk * W;
  // (re)build the partitions: own ranges, buffers, static halos
  if (dw.n != n || dw.world != W) {
    for (PartBuf* p : dw.parts) delete p;
    dw.parts.clear();
    const int first = d->local ? 0 : d->rank, last = d->local ? W : d->rank + 1;
    for (int r = first; r < last; ++r) {
      PartBuf* p = new PartBuf();
      p->r0 = std::min<int64_t>(n, r * chunk);
      p->r1 = std::min<int64_t>(n, (r + 1) * chunk);
      std::vector<uint8_t> f(n, 0);
      for (size_t b = 0; b < brows.size(); ++b) {
        const int64_t i = brows[b], j = bcols[b];
        const bool oi = i >= p->r0 && i < p->r1, oj = j >= p->r0 && j < p->r1;
        if (oi && !oj) f[j] = 1;
        if (oj && !oi) f[i] = 1;
      }
      for (int64_t v = 0; v < n; ++v)
        if (f[v]) p->halo_static.push_back((int)v);
      dw.parts.push_back(p);
    }
    dw.n = n;
    dw.world = W;
    dw.chunk = chunk;
    dw.ptrs_n = -1;
  }
  IBF_TRY(dw.gsc.reserve(8));
  IBF_TRY(dw.xfull.reserve(3 * npad));
  IBF_TRY(dw.host.reserve(16 * sizeof(double)));
  double* hs = (double*)dw.host.p;
  const size_t nv = 3 * (size_t)npad;
  const int G = pd_grid(chunk);
  for (PartBuf* p : dw.parts) {
    IBF_TRY(p->z.reserve(nv));
    IBF_TRY(p->p[0].reserve(nv));
    IBF_TRY(p->p[1].reserve(nv));
    IBF_TRY(p->q.reserve(nv));
    IBF_TRY(p->r.reserve(nv));
    IBF_TRY(p->X.reserve(3 * nv));
    IBF_TRY(p->part.reserve(4 * (size_t)G));
    IBF_TRY(p->scal.reserve(4));
    IBF_TRY(p->t.reserve(std::max(op.contact.n, 1)));
    IBF_TRY(p->tf.reserve(3 * (size_t)std::max(op.friction.n, 1)));
    IBF_TRY(p->hflag.reserve(n));
    IBF_TRY(p->halo.reserve(n + 1));
    // halo = static rows | term vertices outside the own range
    IBF_CUDA(cudaMemsetAsync(p->hflag.p, 0, n, s));
    if (!p->halo_static.empty()) {
      std::vector<uint8_t> f(n, 0);
      for (int v : p->halo_static) f[v] = 1;
      IBF_CUDA(cudaMemcpyAsync(p->hflag.p, f.data(), n, cudaMemcpyHostToDevice, s));
      IBF_CUDA(cudaStreamSynchronize(s));    // f is a host temporary
    }
    if (op.contact.n)
      k_pd_mark_terms<<<pd_grid(4LL * op.contact.n), PD_THREADS, 0, s>>>(op.contact.quad, 4LL * op.contact.n, p->r0,
                                                                         p->r1, p->hflag.p);
    if (op.friction.n)
      k_pd_mark_terms<<<pd_grid(4LL * op.friction.n), PD_THREADS, 0, s>>>(op.friction.quad, 4LL * op.friction.n,
                                                                          p->r0, p->r1, p->hflag.p);
    IBF_TRY(dw.counter.reserve(2 * dw.parts.size() + 2));
    IBF_CUDA(cudaMemsetAsync(dw.counter.p, 0, sizeof(int), s));
    k_pd_collect<<<pd_grid(n), PD_THREADS, 0, s>>>(p->hflag.p, n, p->halo.p, dw.counter.p);
    IBF_LAUNCH_CHECK();
    int nh = 0;
    IBF_CUDA(cudaMemcpyAsync(&nh, dw.counter.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaStreamSynchronize(s));
    p->n_halo = nh;
  }
  auto op_of = [&](PartBuf* p) {
    Operator o = op;
    o.contact.t = p->t.p;
    o.friction.t = p->tf.p;
    return o;
  };
  auto Xb = [&](PartBuf* p, int k) { return p->X.p + (size_t)k * nv; };
  // ---- r = b, z = P^-1 r, x = 0
  for (PartBuf* p : dw.parts) {
    k_pd_init<<<G, PD_THREADS, 0, s>>>(op, p->r0, p->r1, rhs, p->r.p, p->z.p, Xb(p, 0), p->part.p);
    k_pd_sum<<<1, 64, 0, s>>>(p->part.p, G, 2, p->scal.p);
    IBF_LAUNCH_CHECK();
  }
  IBF_TRY(pd_reduce(d, dw, 2, hs, s));
  const double bnorm = sqrt(hs[0]);
  double rz = hs[1];
  IBF_TRY(pd_allgather(d, dw, &PartBuf::z, s));
  int cur = 0, best = 0, result = 0;
  double best_res = bnorm, rel = 0.0, beta = 0.0;
  int64_t iters = 0;
  bool conv = false, first = true, done = false;
  int pb = 0;
  if (bnorm == 0.0) {
    conv = true;
    done = true;
  }
  // done: converged or pAp <= 0; otherwise the cap is reached (best iterate)
  for (int64_t it = 1; !done && it <= max_iters; ++it) {
    // ---- A
    for (PartBuf* p : dw.parts) {
      const Operator o = op_of(p);
      const DirGather gd{p->z.p, p->p[pb ^ 1].p, beta, first};
      if (op.contact.n || op.friction.n) k_pd_dots<<<pd_grid(std::max(op.contact.n, op.friction.n)), PD_THREADS, 0, s>>>(o, gd);
      k_pd_a<<<G, PD_THREADS, 0, s>>>(o, gd, p->r0, p->r1, p->p[pb].p, p->q.p, p->halo.p, p->n_halo, p->part.p);
      k_pd_sum<<<1, 32, 0, s>>>(p->part.p, G, 1, p->scal.p);
      IBF_LAUNCH_CHECK();
    }
    IBF_TRY(pd_reduce(d, dw, 1, hs, s));
    const double pap = hs[0];
    if (pap <= 0.0) {
      result = best;
      iters = it - 1;
      rel = best_res / bnorm;
      done = true;
      break;
    }
    // ---- B
    const double alpha = rz / pap;
    const int nxt = (cur != 0 && best != 0) ? 0 : ((cur != 1 && best != 1) ? 1 : 2);
    for (PartBuf* p : dw.parts) {
      k_pd_b<<<G, PD_THREADS, 0, s>>>(op, p->r0, p->r1, alpha, p->p[pb].p, p->q.p, p->r.p, p->z.p, Xb(p, cur),
                                      Xb(p, nxt), p->part.p);
      k_pd_sum<<<1, 64, 0, s>>>(p->part.p, G, 2, p->scal.p);
      IBF_LAUNCH_CHECK();
    }
    IBF_TRY(pd_reduce(d, dw, 2, hs, s));
    const double res = sqrt(hs[0]);
    double rz_new = hs[1];
    cur = nxt;
    if (res < best_res) {
      best_res = res;
      best = cur;
    }
    if (res <= rel_tol * bnorm) {
      result = cur;
      iters = it;
      conv = true;
      rel = res / bnorm;
      done = true;
      break;
    }
    IBF_TRY(pd_allgather(d, dw, &PartBuf::z, s));
    if (it % 250 == 0) {
      // restart from the true residual r = b - H x (x gathered in full)
      for (PartBuf* p : dw.parts) {
        k_pd_copy_rows<<<G, PD_THREADS, 0, s>>>(Xb(p, cur), p->q.p, p->r0, p->r1);
        IBF_LAUNCH_CHECK();
      }
      IBF_TRY(pd_allgather(d, dw, &PartBuf::q, s));
      for (PartBuf* p : dw.parts) {
        const Operator o = op_of(p);
        const PlainGather gx{p->q.p};
        if (op.contact.n || op.friction.n) k_pd_dots_plain<<<pd_grid(std::max(op.contact.n, op.friction.n)), PD_THREADS, 0, s>>>(o, gx);
        k_pd_restart<<<G, PD_THREADS, 0, s>>>(o, gx, p->r0, p->r1, rhs, p->r.p, p->z.p, p->part.p);
        k_pd_sum<<<1, 32, 0, s>>>(p->part.p, G, 1, p->scal.p);
        IBF_LAUNCH_CHECK();
      }
      IBF_TRY(pd_reduce(d, dw, 1, hs, s));
      rz = hs[0];
      IBF_TRY(pd_allgather(d, dw, &PartBuf::z, s));
      first = true;
      pb ^= 1;
      continue;
    }
    beta = rz_new / rz;
    rz = rz_new;
    first = false;
    pb ^= 1;
  }
  if (!done) {
    result = best;
    iters = max_iters;
    rel = best_res / bnorm;
  }
  // ---- x_out = X[result], gathered to every partition
  if (bnorm == 0.0) {
    IBF_CUDA(cudaMemsetAsync(x_out, 0, 3 * n * sizeof(double), s));
  } else if (d->local) {
    for (PartBuf* p : dw.parts) {
      k_pd_copy_rows<<<G, PD_THREADS, 0, s>>>(Xb(p, result), x_out, p->r0, p->r1);
      IBF_LAUNCH_CHECK();
    }
  } else {
    PartBuf* p = dw.parts[0];
    k_pd_copy_rows<<<G, PD_THREADS, 0, s>>>(Xb(p, result), dw.xfull.p, p->r0, p->r1);
    IBF_LAUNCH_CHECK();
    IBF_TRY(dist_allgather(d, dw.xfull.p + 3 * p->r0, dw.xfull.p, 3 * (size_t)chunk, s));
    IBF_CUDA(cudaMemcpyAsync(x_out, dw.xfull.p, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  IBF_TRY(w.info.reserve(4));
  hs[8] = (double)iters;
  hs[9] = conv ? 1.0 : 0.0;
  hs[10] = rel;
  IBF_CUDA(cudaMemcpyAsync(w.info.p, hs + 8, 3 * sizeof(double), cudaMemcpyHostToDevice, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  ++g_launches;
  return IBF_OK;
}

}  // namespace ibf
