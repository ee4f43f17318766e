// Elastic system: static BSR pattern, per-tet element kernel, deterministic
// gather assembly, incremental energy, NH inversion cap.
//
// Replaces (paths relative to /root/reference/pkg/src):
//   assemble                 intact/solver.py:109-156
//   incremental_energy       intact/solver.py:88-106
//   psd_block_hessians / assemble_vertex_blocks / element_gradients
//                            intact/elasticity.py:167-170, :274-299
//   clique_contributions + BlockSparseMatrix coalescing + mask_dirichlet
//                            intact/sparse.py:17-62, :81-87
//   inversion_safe_step      intact/elasticity.py:321-356
//   stiffness_diagonal_max   intact/stepper.py:191-200
//
// Layout.  The sparsity pattern of mass + elasticity never changes, so it is
// built once: diagonal + strict-upper 3x3 blocks sorted by (row, col), a
// transpose index for the symmetric SpMV, and gather maps (block <- tet
// contributions, vertex <- tet incidences) in tet order.  Assembly is two
// passes with no floating-point atomics:
//   1. k_elem: one thread per tet computes F, psi, PK1, the rotation-variant
//      SVD and the analytic eigensystem, and writes its 4 gradient rows and
//      10 upper 3x3 blocks into tile-32 staging buffers (each warp's 32 tets
//      form contiguous 2.3 KB tiles, written fully coalesced via shared
//      memory);
//   2. k_gather_blocks / k_vertex_rows: each BSR block / vertex sums its
//      contributions in tet order (the order the reference's coalescing and
//      bincount use), applies the DBC mask, adds the contact terms, and
//      inverts the 3x3 diagonal for the block-Jacobi preconditioner.
#include <algorithm>
#include <numeric>
#include <vector>

#include "elastic_math.cuh"
#include "system.cuh"

namespace ibf {

constexpr int ELEM_THREADS = 128;
constexpr int MAXT = 8;        // trial points per energy launch
constexpr int MAX_SMEM_REGIONS = 64;

// local upper pairs (li <= lj) in np.triu_indices(4) order
__constant__ int c_qi[10] = {0, 0, 0, 0, 1, 1, 1, 2, 2, 3};
__constant__ int c_qj[10] = {0, 1, 2, 3, 1, 2, 3, 2, 3, 3};

__device__ __forceinline__ int region_of(int t, const RegionDev* regs, int nreg) {
  int lo = 0, hi = nreg - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (t < regs[mid].end) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ size_t grad_tile_index(int64_t t, int l) {
  return (size_t)(t >> 5) * 384 + (size_t)(t & 31) * 12 + 3 * l;
}
// Staged element blocks: one 288-double tile per (32 tets, local pair q).
// IBF_STAGE_SPLIT=1: the tile holds each lane's entries 0..7 as a 64-byte
// run (lane*8), then entry 8 of all lanes (256 + lane), so a block is read
// with two 256-bit loads and one 64-bit load; =0: 9 consecutive doubles
// per lane (nine 64-bit loads).
#ifndef IBF_STAGE_SPLIT
#define IBF_STAGE_SPLIT 1
#endif
__device__ __forceinline__ size_t blk_tile_index(int64_t t, int q) {
  return ((size_t)(t >> 5) * 10 + q) * 288 + (size_t)(t & 31) * (IBF_STAGE_SPLIT ? 8 : 9);
}
__device__ __forceinline__ double4 ld_nc_256(const double* p) {
  double4 r;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
// the 9 entries of the staged block of tet t, pair q
__device__ __forceinline__ void load_staged_block(const double* __restrict__ elem_blk, int64_t t, int q,
                                                  double v[9]) {
  const double* K = elem_blk + blk_tile_index(t, q);
  if (IBF_STAGE_SPLIT) {
    const double4 a = ld_nc_256(K), b = ld_nc_256(K + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    v[8] = __ldg(elem_blk + ((size_t)(t >> 5) * 10 + q) * 288 + 256 + (t & 31));
  } else {
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = __ldg(K + k);
  }
}

// warp-cooperative coalesced store of `per` doubles per lane into a
// contiguous tile of 32*per doubles.
template <int PER>
__device__ __forceinline__ void warp_store_tile(double* sm, const double v[PER], double* gtile) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < PER; ++k) sm[lane * PER + k] = v[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < PER; ++k) gtile[lane + 32 * k] = sm[lane + 32 * k];
  __syncwarp();
}

#ifndef IBF_GATHER_ILP
#define IBF_GATHER_ILP 2
#endif
// timing-only diagnostics (wrong results): IBF_DIAG_ELEM_NOSTORE drops the
// staging stores, IBF_DIAG_GATHER_L2 folds the staging reads onto 8,192 tets
#ifndef IBF_DIAG_ELEM_NOSTORE
#define IBF_DIAG_ELEM_NOSTORE 0
#endif
#ifndef IBF_DIAG_GATHER_L2
#define IBF_DIAG_GATHER_L2 0
#endif

struct ElemArgs {
  int64_t m;
  int64_t n_tiles;
  const int* tets;
  const double* rows;
  const double* vols;
  const RegionDev* regions;
  int nreg;
  const double* x;
  double h2;
  double* elem_grad;
  double* elem_blk;
  int* flags;
};

#ifndef IBF_ELEM_MINB
#define IBF_ELEM_MINB 1
#endif
template <bool HESS>
__global__ void __launch_bounds__(ELEM_THREADS, IBF_ELEM_MINB) k_elem(ElemArgs a) {
  __shared__ double stage[ELEM_THREADS / 32][384];
  __shared__ RegionDev sreg[MAX_SMEM_REGIONS];
  const bool use_smem = a.nreg <= MAX_SMEM_REGIONS;
  if (use_smem)
    for (int k = threadIdx.x; k < a.nreg; k += blockDim.x) sreg[k] = a.regions[k];
  __syncthreads();
  const int64_t t = blockIdx.x * (int64_t)ELEM_THREADS + threadIdx.x;
  if ((t >> 5) >= a.n_tiles) return;  // whole warp beyond the last tile
  const bool active = t < a.m;
  double* sm = stage[threadIdx.x >> 5];
  const int64_t tile_t = t;  // tile coordinates use t even for padding lanes

  double X[4][3], A[4][3], vol = 0.0;
  int ids[4] = {0, 0, 0, 0};
  int model = el::LIN;
  double mu = 0.0, lam = 0.0;
  if (active) {
    const RegionDev* R = use_smem ? sreg : a.regions;
    const RegionDev rg = R[region_of((int)t, R, a.nreg)];
    model = rg.model;
    mu = rg.mu;
    lam = rg.lam;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ids[k] = a.tets[4 * t + k];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        X[k][c] = a.x[3 * (int64_t)ids[k] + c];
        A[k][c] = a.rows[12 * t + 3 * k + c];
      }
    }
    vol = a.vols[t];
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) X[k][c] = A[k][c] = 0.0;
  }
  const el::M3 F = el::def_grad(X, A);
  el::M3 U, V;
  double s[3] = {1.0, 1.0, 1.0};
  if (model != el::LIN) {
    el::svd_rv(F, U, s, V);
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) U.m[i][j] = V.m[i][j] = (i == j) ? 1.0 : 0.0;
  }
  // energy finiteness check (assemble raises NonFiniteEnergyError, intact/solver.py:130-131)
  if (active) {
    double e;
    if (model == el::COR) {
      double d2 = 0.0;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          const double r = U.m[i][0] * V.m[j][0] + U.m[i][1] * V.m[j][1] + U.m[i][2] * V.m[j][2];
          d2 += (F.m[i][j] - r) * (F.m[i][j] - r);
        }
      const double tr = (s[0] + s[1] + s[2]) - 3.0;
      e = mu * d2 + 0.5 * lam * tr * tr;
    } else {
      e = el::psi(model, mu, lam, F);
    }
    if (!isfinite(e * vol)) atomicOr(a.flags, 1);
  }
  // gradient rows: h^2 * V * P A_k^T (element_gradients, intact/elasticity.py:167-170)
  {
    double g[12];
    if (active) {
      const el::M3 P = el::pk1(model, mu, lam, F, U, s, V);
      const double sc = a.h2 * vol;
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int r = 0; r < 3; ++r)
          g[3 * k + r] = sc * (P.m[r][0] * A[k][0] + P.m[r][1] * A[k][1] + P.m[r][2] * A[k][2]);
    } else {
#pragma unroll
      for (int k = 0; k < 12; ++k) g[k] = 0.0;
    }
    warp_store_tile<12>(sm, g, a.elem_grad + (size_t)(tile_t >> 5) * 384);
  }
  if (!HESS) return;
  // PSD vertex blocks (psd_block_hessians + assemble_vertex_blocks, :274-299)
  double W[3][3], tw[3], fl[3];
  el::mode_weights(model, mu, lam, s, W, tw, fl);
  double y[4][3];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) y[k][c] = V.m[0][c] * A[k][0] + V.m[1][c] * A[k][1] + V.m[2][c] * A[k][2];
  const double sc = active ? a.h2 * vol : 0.0;
#pragma unroll 1
  for (int q = 0; q < 10; ++q) {
    const int i = c_qi[q], j = c_qj[q];
    double K[9];
    // store in global-upper orientation: transpose when ids[i] > ids[j]
    if (ids[i] > ids[j]) {
      el::vertex_block(y[j], y[i], W, tw, fl, U, sc, K);
    } else {
      el::vertex_block(y[i], y[j], W, tw, fl, U, sc, K);
    }
    if (IBF_DIAG_ELEM_NOSTORE) {
      // timing-only bound: blocks computed but not staged
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < 9; ++k) sum += K[k];
      if (sum == 1.2345e300) a.elem_blk[t] = sum;
    } else {
      double* gt = a.elem_blk + ((size_t)(tile_t >> 5) * 10 + q) * 288;
      if (IBF_STAGE_SPLIT) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int k = 0; k < 9; ++k) sm[lane * 9 + k] = K[k];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = lane + 32 * k;  // lane j>>3, entry j&7
          gt[j] = sm[(j >> 3) * 9 + (j & 7)];
        }
        gt[256 + lane] = sm[lane * 9 + 8];
        __syncwarp();
      } else {
        warp_store_tile<9>(sm, K, gt);
      }
    }
  }
}

// per storage block: mass (real diagonal) + contributions in tet order, DBC
// mask; consecutive threads write consecutive lanes of one slot (coalesced)
__global__ void k_gather_blocks(int64_t nq, const int* __restrict__ qrow, const int* __restrict__ col,
                                const uint8_t* __restrict__ qreal, const int* __restrict__ blk_ptr,
                                const int* __restrict__ blk_src, const double* __restrict__ elem_blk,
                                const double* __restrict__ masses, const uint8_t* __restrict__ mask,
                                double* __restrict__ val) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const int r = qrow[q], c = col[q];
    double acc[9];
    const double m0 = (r == c && qreal[q]) ? masses[r] : 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = (k == 0 || k == 4 || k == 8) ? m0 : 0.0;
    if (!(mask && (mask[r] || mask[c]))) {
      const int e0 = blk_ptr[q], e1 = blk_ptr[q + 1];
      int e = e0;
      // IBF_GATHER_ILP contributions' loads in flight before their adds,
      // which stay in tet order
      for (; e + IBF_GATHER_ILP <= e1; e += IBF_GATHER_ILP) {
        double v[IBF_GATHER_ILP][9];
#pragma unroll
        for (int u = 0; u < IBF_GATHER_ILP; ++u) {
          const int src = blk_src[e + u];
          int t = src / 10;
          const int qq = src - 10 * t;
          if (IBF_DIAG_GATHER_L2) t &= 8191;  // timing-only bound: staging L2-resident
          load_staged_block(elem_blk, t, qq, v[u]);
        }
#pragma unroll
        for (int u = 0; u < IBF_GATHER_ILP; ++u)
#pragma unroll
          for (int k = 0; k < 9; ++k) acc[k] += v[u][k];
      }
      for (; e < e1; ++e) {
        const int src = blk_src[e];
        int t = src / 10;
        const int qq = src - 10 * t;
        if (IBF_DIAG_GATHER_L2) t &= 8191;
        double v[9];
        load_staged_block(elem_blk, t, qq, v);
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] += v[k];
      }
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) val[qel((int)q, k)] = acc[k];
  }
}

struct RowArgs {
  int64_t n;
  const double* x_hat;
  const double* x_tilde;
  const double* masses;
  const uint8_t* mask;
  const int* vt_ptr;
  const int* vt_src;
  const double* elem_grad;
  const int* diag_q;
  const double* val;
  ContactView cv;
  const double* coef_g;  // contact gradient coefficients (C)
  FrictionView fv;
  const double* fr_gw;   // friction world forces (K,3)
  double* grad;
  double* pinv;
  int* flags;
};

// per vertex: gradient row and block-Jacobi inverse
__global__ void k_vertex_rows(RowArgs a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    const double m = a.masses[i];
    double g[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) g[c] = m * (a.x_hat[3 * i + c] - a.x_tilde[3 * i + c]);
    double s[3] = {0.0, 0.0, 0.0};
    for (int e = a.vt_ptr[i]; e < a.vt_ptr[i + 1]; ++e) {
      const int src = a.vt_src[e];
      const double* gt = a.elem_grad + grad_tile_index(src >> 2, src & 3);
      s[0] += gt[0];
      s[1] += gt[1];
      s[2] += gt[2];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) g[c] += s[c];
    const bool masked = a.mask && a.mask[i];
    double D[9];
    const int dq = a.diag_q[i];
#pragma unroll
    for (int k = 0; k < 9; ++k) D[k] = a.val[qel(dq, k)];
    // masked (Dirichlet) rows take no contact terms; a pinned plate's
    // vertices can sit in 10^4 constraints, so skip the incidence walk
    if (a.cv.n && !masked) {
      double sc[3] = {0.0, 0.0, 0.0};
      for (int e = a.cv.vc_ptr[i]; e < a.cv.vc_ptr[i + 1]; ++e) {
        const int src = a.cv.vc_src[e];
        const int c = src >> 2, slot = src & 3;
        const double* gg = a.cv.grad + 12 * (size_t)c + 3 * slot;
        const double cg = a.coef_g[c];
        sc[0] += cg * gg[0];
        sc[1] += cg * gg[1];
        sc[2] += cg * gg[2];
        if (!masked) {
          const double ch = a.cv.coef[c];
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int q = 0; q < 3; ++q) D[3 * r + q] += ch * gg[r] * gg[q];
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) g[c] += sc[c];
    }
    if (a.fv.n && !masked) {
      // friction: g += w_slot F_k; D += w_slot^2 Hw_k (intact/friction.py:79-100)
      double sf[3] = {0.0, 0.0, 0.0};
      for (int e = a.fv.vf_ptr[i]; e < a.fv.vf_ptr[i + 1]; ++e) {
        const int src = a.fv.vf_src[e];
        const int k = src >> 2;
        const double wv = a.fv.w[src];
        const double* F = a.fr_gw + 3 * (size_t)k;
        const double* Hk = a.fv.hw + 9 * (size_t)k;
        sf[0] += wv * F[0];
        sf[1] += wv * F[1];
        sf[2] += wv * F[2];
        const double w2 = wv * wv;
#pragma unroll
        for (int q = 0; q < 9; ++q) D[q] += w2 * Hk[q];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) g[c] += sf[c];
    }
    if (masked) g[0] = g[1] = g[2] = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) a.grad[3 * i + c] = g[c];
    if (g[0] != 0.0 || g[1] != 0.0 || g[2] != 0.0) atomicOr(a.flags + 1, 1);
    inv3_sym6(D, a.pinv + PINV_STRIDE * i);
  }
}

// ------------------------------------------------------------ energy

struct EnergyArgs {
  int64_t n, m, nc;
  int T;
  const double* xh;
  const double* p;
  const double* r0;       // optional device base step; trial j uses r0 * rs[j]
  double rs[MAXT];
  const double* xt;
  const double* masses;
  const int* tets;
  const double* rows;
  const double* vols;
  const RegionDev* regions;
  int nreg;
  const int* cquad;
  const double* cad;
  const double* cag;
  const double* cax;
  const double* clam;
  const double* cgam;
  double mu, offset;
  int bv, bt, bc, bf;
  // friction terms (K)
  int64_t nf;
  const int* fquad;
  const double* fw;
  const double* ffr;
  const double* fcoeff;
  const double* fref;
  double feps;
  double* part;           // (bv+bt+bc+bf) * MAXT
};

__device__ __forceinline__ double fr_f0e(double y, double eps) {
  return y >= eps ? y : -(y * y * y) / (3.0 * eps * eps) + y * y / eps + eps / 3.0;
}

__device__ __forceinline__ double trial_r(const EnergyArgs& a, int j) {
  return a.r0 ? __dmul_rn(*a.r0, a.rs[j]) : a.rs[j];
}
// x_hat + r * p exactly as numpy evaluates it (no FMA)
__device__ __forceinline__ double trial_coord(const EnergyArgs& a, double r, int64_t k) {
  return a.p ? __dadd_rn(a.xh[k], __dmul_rn(r, a.p[k])) : a.xh[k];
}

#ifndef IBF_ENERGY_MINB
#define IBF_ENERGY_MINB 3  // 0: the compiler's register choice for 256 threads (128)
#endif
#if IBF_ENERGY_MINB > 0
#define IBF_ENERGY_BOUNDS __launch_bounds__(256, IBF_ENERGY_MINB)
#else
#define IBF_ENERGY_BOUNDS __launch_bounds__(256)
#endif
__global__ void IBF_ENERGY_BOUNDS k_energy(EnergyArgs a) {
  __shared__ double red[8];
  double acc[MAXT];
#pragma unroll
  for (int j = 0; j < MAXT; ++j) acc[j] = 0.0;
  double rj[MAXT];
#pragma unroll
  for (int j = 0; j < MAXT; ++j) rj[j] = (j < a.T) ? trial_r(a, j) : 0.0;
  const int b = blockIdx.x;
  if (b < a.bv) {
    // inertia: 0.5 * sum m ||y - x_tilde||^2 (the 0.5 is applied at the end)
    for (int64_t i = b * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)a.bv * blockDim.x) {
      const double mi = a.masses[i];
#pragma unroll
      for (int j = 0; j < MAXT; ++j) {
        if (j >= a.T) break;
        double ss = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double d = trial_coord(a, rj[j], 3 * i + c) - a.xt[3 * i + c];
          ss += d * d;
        }
        acc[j] += mi * ss;
      }
    }
  } else if (b < a.bv + a.bt) {
    const int bb = b - a.bv;
    for (int64_t t = bb * (int64_t)blockDim.x + threadIdx.x; t < a.m; t += (int64_t)a.bt * blockDim.x) {
      const RegionDev rg = a.regions[region_of((int)t, a.regions, a.nreg)];
      int ids[4];
      double A[4][3];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ids[k] = a.tets[4 * t + k];
#pragma unroll
        for (int c = 0; c < 3; ++c) A[k][c] = a.rows[12 * t + 3 * k + c];
      }
      const double vol = a.vols[t];
#pragma unroll 1
      for (int j = 0; j < MAXT; ++j) {
        if (j >= a.T) break;
        double X[4][3];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int c = 0; c < 3; ++c) X[k][c] = trial_coord(a, rj[j], 3 * (int64_t)ids[k] + c);
        const el::M3 F = el::def_grad(X, A);
        acc[j] += el::psi(rg.model, rg.mu, rg.lam, F) * vol;
      }
    }
  } else if (b >= a.bv + a.bt + a.bc) {
    // friction: sum coeff f0(|T^T (sum w y - ref)|) (intact/friction.py:75-77)
    const int bb = b - a.bv - a.bt - a.bc;
    for (int64_t k = bb * (int64_t)blockDim.x + threadIdx.x; k < a.nf; k += (int64_t)a.bf * blockDim.x) {
      const double* F = a.ffr + 6 * k;
#pragma unroll 1
      for (int j = 0; j < MAXT; ++j) {
        if (j >= a.T) break;
        double rel[3] = {0.0, 0.0, 0.0};
        for (int e = 0; e < 4; ++e) {
          const int64_t v = a.fquad[4 * k + e];
          const double wv = a.fw[4 * k + e];
          for (int c = 0; c < 3; ++c) rel[c] += wv * trial_coord(a, rj[j], 3 * v + c);
        }
        for (int c = 0; c < 3; ++c) rel[c] -= a.fref[3 * k + c];
        const double u0 = F[0] * rel[0] + F[2] * rel[1] + F[4] * rel[2];
        const double u1 = F[1] * rel[0] + F[3] * rel[1] + F[5] * rel[2];
        acc[j] += a.fcoeff[k] * fr_f0e(sqrt(u0 * u0 + u1 * u1), a.feps);
      }
    }
  } else {
    const int bb = b - a.bv - a.bt;
    for (int64_t c = bb * (int64_t)blockDim.x + threadIdx.x; c < a.nc; c += (int64_t)a.bc * blockDim.x) {
      const int* q = a.cquad + 4 * c;
      const double lam = a.clam[c], gam = a.cgam[c];
#pragma unroll 1
      for (int j = 0; j < MAXT; ++j) {
        if (j >= a.T) break;
        double dot = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int e = 0; e < 3; ++e)
            dot += a.cag[12 * c + 3 * k + e] * (trial_coord(a, rj[j], 3 * (int64_t)q[k] + e) - a.cax[12 * c + 3 * k + e]);
        const double cv = a.cad[c] + dot - a.offset;
        const double sl = fmax(0.0, cv - lam / a.mu);
        const double r = cv - sl;
        acc[j] += gam * (0.5 * a.mu * r * r - lam * r);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < MAXT; ++j) {
    if (j >= a.T) break;
    const double v = block_sum(acc[j], red);
    if (threadIdx.x == 0) a.part[(size_t)b * MAXT + j] = v;
  }
}

__global__ void k_energy_final(const double* __restrict__ part, int T, int bv, int bt, int bc, int bf, double h2,
                               double* __restrict__ out) {
  // one warp per trial: ((inertia + h^2 elastic) + AL) + friction, the
  // reference's accumulation order (intact/solver.py:98-106)
  const int j = threadIdx.x >> 5;
  if (j >= T) return;
  const int lane = threadIdx.x & 31;
  double si = 0.0, se = 0.0, sa = 0.0, sf = 0.0;
  for (int k = lane; k < bv; k += 32) si += part[(size_t)k * MAXT + j];
  for (int k = lane; k < bt; k += 32) se += part[(size_t)(bv + k) * MAXT + j];
  for (int k = lane; k < bc; k += 32) sa += part[(size_t)(bv + bt + k) * MAXT + j];
  for (int k = lane; k < bf; k += 32) sf += part[(size_t)(bv + bt + bc + k) * MAXT + j];
  si = warp_sum(si);
  se = warp_sum(se);
  sa = warp_sum(sa);
  sf = warp_sum(sf);
  if (lane == 0) out[j] = ((0.5 * si + h2 * se) + sa) + sf;
}

// ------------------------------------------------------------ inversion cap

// smallest positive real root of c3 t^3 + c2 t^2 + c1 t + c0 with the
// reference's filters (_smallest_positive_root, intact/elasticity.py:321-334):
// coefficients scaled by max |c|, leading exact zeros trimmed, roots "real"
// when |Im| < 1e-10 (1 + |Re|), positive when > 1e-12.
__device__ double first_positive_root(double c3, double c2, double c1, double c0) {
  const double big = fmax(fmax(fabs(c3), fabs(c2)), fmax(fabs(c1), fabs(c0)));
  if (big == 0.0) return INFINITY;
  double c[4] = {c3 / big, c2 / big, c1 / big, c0 / big};
  int lead = 0;
  while (lead < 4 && c[lead] == 0.0) ++lead;
  const int deg = 3 - lead;
  if (deg <= 0) return INFINITY;
  double re[3], im[3];
  int nr = 0;
  auto quad_roots = [&](double qa, double qb, double qc) {
    const double disc = qb * qb - 4.0 * qa * qc;
    if (disc >= 0.0) {
      const double sq = sqrt(disc);
      const double qq = -0.5 * (qb + copysign(sq, qb));
      if (qq != 0.0) {
        re[nr] = qq / qa; im[nr++] = 0.0;
        re[nr] = qc / qq; im[nr++] = 0.0;
      } else {
        re[nr] = 0.0; im[nr++] = 0.0;
        re[nr] = 0.0; im[nr++] = 0.0;
      }
    } else {
      const double rr = -qb / (2.0 * qa), ii = sqrt(-disc) / (2.0 * fabs(qa));
      re[nr] = rr; im[nr++] = ii;
      re[nr] = rr; im[nr++] = -ii;
    }
  };
  if (deg == 1) {
    re[nr] = -c[3] / c[2];
    im[nr++] = 0.0;
  } else if (deg == 2) {
    quad_roots(c[1], c[2], c[3]);
  } else {
    const double B = c[1] / c[0], C = c[2] / c[0], D = c[3] / c[0];
    auto f = [&](double x) { return ((x + B) * x + C) * x + D; };
    auto fp = [&](double x) { return (3.0 * x + 2.0 * B) * x + C; };
    const double p = C - B * B / 3.0;
    const double q = 2.0 * B * B * B / 27.0 - B * C / 3.0 + D;
    const double disc = 0.25 * q * q + p * p * p / 27.0;
    double x1;
    if (disc > 0.0) {
      const double u = cbrt(-0.5 * q - copysign(sqrt(disc), q));
      const double y = (u != 0.0) ? u - p / (3.0 * u) : 0.0;
      x1 = y - B / 3.0;
    } else {
      const double rr = sqrt(fmax(-p / 3.0, 0.0));
      double arg = (rr > 0.0) ? (-0.5 * q) / (rr * rr * rr) : 0.0;
      arg = fmin(1.0, fmax(-1.0, arg));
      const double phi = acos(arg);
      x1 = 2.0 * rr * cos(phi / 3.0) - B / 3.0;
    }
    for (int it = 0; it < 3; ++it) {
      const double d = fp(x1);
      if (d == 0.0) break;
      const double nx = x1 - f(x1) / d;
      if (!isfinite(nx)) break;
      x1 = nx;
    }
    re[nr] = x1;
    im[nr++] = 0.0;
    // deflate: x^2 + (B + x1) x + (C + (B + x1) x1)
    const double e1 = B + x1;
    quad_roots(1.0, e1, C + e1 * x1);
    for (int k = 1; k < nr; ++k) {
      if (im[k] != 0.0) continue;
      for (int it = 0; it < 2; ++it) {
        const double d = fp(re[k]);
        if (d == 0.0) break;
        const double nx = re[k] - f(re[k]) / d;
        if (!isfinite(nx)) break;
        re[k] = nx;
      }
    }
  }
  double best = INFINITY;
  for (int k = 0; k < nr; ++k) {
    if (!(fabs(im[k]) < 1e-10 * (1.0 + fabs(re[k])))) continue;
    if (re[k] > 1e-12 && re[k] < best) best = re[k];
  }
  return best;
}

__global__ void k_inversion_cap(int64_t m, const int* __restrict__ tets, const double* __restrict__ rows,
                                const RegionDev* __restrict__ regions, int nreg, const double* __restrict__ x,
                                const double* __restrict__ p, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    const RegionDev rg = regions[region_of((int)t, regions, nreg)];
    if (rg.model != el::NH) continue;
    double X[4][3], P[4][3], A[4][3];
    for (int k = 0; k < 4; ++k) {
      const int v = tets[4 * t + k];
      for (int c = 0; c < 3; ++c) {
        X[k][c] = x[3 * (int64_t)v + c];
        P[k][c] = p[3 * (int64_t)v + c];
        A[k][c] = rows[12 * t + 3 * k + c];
      }
    }
    const el::M3 Fa = el::def_grad(X, A), Fb = el::def_grad(P, A);
    bool moving = false;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) moving |= fabs(Fb.m[i][j]) > 0.0;
    if (!moving) continue;
    const el::M3 ca = el::cofactor(Fa), cb = el::cofactor(Fb);
    double c1 = 0.0, c2 = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        c1 += ca.m[i][j] * Fb.m[i][j];
        c2 += cb.m[i][j] * Fa.m[i][j];
      }
    const double c0 = (1.0 - 0.2) * el::det3(Fa);
    const double r = first_positive_root(el::det3(Fb), c2, c1, c0);
    if (r < INFINITY) atomic_min_nonneg(out, 0.9 * r);
  }
}

__global__ void k_fill(double* p, double v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_diag_max(int64_t n, const int* __restrict__ diag_q, const double* __restrict__ val,
                           double* __restrict__ out) {
  __shared__ double red[8];
  double v = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int q = diag_q[i];
    v = fmax(v, fmax(val[qel(q, 0)], fmax(val[qel(q, 4)], val[qel(q, 8)])));
  }
  v = block_max(v, red);
  if (threadIdx.x == 0) {
    // diagonal entries of mass + PSD blocks are >= 0: ordered-bit max
    atomic_max_nonneg(out, fmax(v, 0.0));
  }
}

// ------------------------------------------------------------ host side

// FP64 flops per tet of k_elem, frozen from ncu: 2 x DFMA + DMUL + DADD
// thread instructions per tet = 2 x 1273.2 + 846.6 + 66.5 = 3459.5 on the
// COR squishy-ball C4 assembly (profiles/r2v_k_elem_flops.json).  The
// reference's own counter gives 927 multiplies per tet for the 10-block PSD
// part alone (tests/test_elasticity.py:381-420); F, PK1, the rotation-variant
// SVD and the eigensystem make up the rest.
constexpr double kFlopPerTet = 3459.5;
// FP64 flops per tet and trial point of k_energy's elastic part, frozen the
// same way: 2 x 3.470e9 + 1.673e9 + 0.284e9 = 8.90e9 per launch of 2 trial
// points over the 2.30M COR tets (profiles/r2ah_k_energy_flops.json)
constexpr double kEnergyFlopPerTetPoint = 1937.0;

int system_assemble(ibf_system* s, ibf_contacts* c, const double* x_hat, const double* x_tilde, double mu,
                    double offset, double h, bool apply_dbc, double* grad, bool contacts_ready,
                    cudaStream_t st) {
  const double h2 = h * h;
  IBF_CUDA(cudaMemsetAsync(s->flags.p, 0, 2 * sizeof(int), st));
  if (s->m) {
    ElemArgs a{s->m, s->n_tiles, s->tets.p, s->shape_rows.p, s->volumes.p, s->regions.p, s->n_regions, x_hat, h2,
               s->elem_grad.p, s->elem_blk.p, s->flags.p};
    // algorithmic: tet data 120 B + x once; FLOP_PER_TET
    KernelClock kc(KC_ELEM, st, 120.0 * s->m + 24.0 * s->n, kFlopPerTet * s->m, (double)s->m);
    k_elem<true><<<(int)div_up(s->n_tiles, ELEM_THREADS / 32), ELEM_THREADS, 0, st>>>(a);
    IBF_LAUNCH_CHECK();
  }
  const uint8_t* mask = (apply_dbc && s->any_dbc) ? s->dbc.p : nullptr;
  // algorithmic: one 72 B write per stored block (N + E_u) — the staging
  // round trip k_elem -> k_gather_blocks is not algorithmic traffic
  {
    KernelClock kcg(KC_GATHER, st, 72.0 * s->pat.nb, 0.0, (double)s->pat.nb);
    k_gather_blocks<<<(int)std::min<int64_t>(div_up(s->pat.nq, 256), 148LL * 32), 256, 0, st>>>(
        s->pat.nq, s->pat.qrow.p, s->pat.col.p, s->pat.qreal.p, s->blk_ptr.p, s->blk_src.p, s->elem_blk.p,
        s->masses.p, mask, s->pat.val.p);
    IBF_LAUNCH_CHECK();
  }
  ContactView cv;
  const double* coef_g = nullptr;
  if (c && c->n) {
    if (!contacts_ready) {
      IBF_TRY(contact_build_incidence(c, s->n, st));
    }
    IBF_TRY(contact_prepare(c, x_hat, mu, offset, st));
    if (IBF_PCG_WARP_TERMS) IBF_TRY(contact_pack_terms(c, s->n, mask, st));
    cv = contact_view(c);
    coef_g = c->coef_g.p;
  }
  FrictionView fv;
  const double* fr_gw = nullptr;
  ibf_friction* fr = (s->friction && s->friction->n) ? s->friction : nullptr;
  if (fr) {
    IBF_TRY(friction_build_incidence(fr, s->n, st));
    IBF_TRY(friction_prepare(fr, x_hat, st));
    fv = friction_view(fr);
    fr_gw = fr->gw.p;
  }
  RowArgs r{s->n, x_hat, x_tilde, s->masses.p, mask, s->vt_ptr.p, s->vt_src.p, s->elem_grad.p,
            s->pat.diag_q.p, s->pat.val.p, cv, coef_g, fv, fr_gw, grad, s->pinv.p, s->flags.p};
  if (s->n) {
    // algorithmic: x_tilde 24 + mass 8 + grad 24 per vertex, 232 B per constraint
    KernelClock kc(KC_ROWS, st, 56.0 * s->n + 232.0 * cv.n, 0.0, (double)s->n);
    k_vertex_rows<<<(int)std::min<int64_t>(div_up(s->n, 256), 148LL * 32), 256, 0, st>>>(r);
    IBF_LAUNCH_CHECK();
  }
  s->assembled_contacts = (c && c->n) ? c : nullptr;
  s->assembled_friction = fr != nullptr;
  s->assembled_dbc = mask != nullptr;
  return IBF_OK;
}

int system_pcg(ibf_system* s, const double* rhs, double* x, double rel_tol, int64_t max_iters, cudaStream_t st) {
  if (s->dist && s->dist->world > 1)
    return pcg_solve_dist(s->op(), s->pat.rows, s->pat.cols, rhs, x, rel_tol, max_iters, s->work, s->dwork,
                          s->dist, st);
  return pcg_solve(s->op(), rhs, x, rel_tol, max_iters, s->work, st);
}

int system_energy_launch(ibf_system* s, ibf_contacts* c, const double* x_hat, const double* p, int n_r,
                         const double* r_host, const double* r0_dev, const double* x_tilde, double mu,
                         double offset, double h, double* out_dev, cudaStream_t st) {
  if (n_r < 1 || n_r > MAXT) {
    set_error("energy: 1..8 trial points per launch");
    return IBF_ERR_BAD_ARG;
  }
  EnergyArgs a{};
  a.n = s->n;
  a.m = s->m;
  a.nc = (c ? c->n : 0);
  a.T = n_r;
  a.xh = x_hat;
  a.p = p;
  a.r0 = r0_dev;
  for (int j = 0; j < MAXT; ++j) a.rs[j] = (j < n_r && r_host) ? r_host[j] : 0.0;
  a.xt = x_tilde;
  a.masses = s->masses.p;
  a.tets = s->tets.p;
  a.rows = s->shape_rows.p;
  a.vols = s->volumes.p;
  a.regions = s->regions.p;
  a.nreg = s->n_regions;
  if (a.nc) {
    a.cquad = c->quad.p;
    a.cad = c->anchor_d.p;
    a.cag = c->anchor_grad.p;
    a.cax = c->anchor_x.p;
    a.clam = c->lam.p;
    a.cgam = c->gamma.p;
  }
  a.mu = mu;
  a.offset = offset;
  a.bv = (int)std::max<int64_t>(1, std::min<int64_t>(div_up(s->n, 256), 148 * 2));
  a.bt = (int)std::max<int64_t>(1, std::min<int64_t>(div_up(s->m, 256), 148 * 8));
  a.bc = (int)std::max<int64_t>(1, std::min<int64_t>(div_up(a.nc, 256), 148 * 2));
  ibf_friction* fr = (s->friction && s->friction->n) ? s->friction : nullptr;
  a.nf = fr ? fr->n : 0;
  a.bf = fr ? (int)std::max<int64_t>(1, std::min<int64_t>(div_up(a.nf, 256), 148)) : 0;
  if (fr) {
    a.fquad = fr->quad.p;
    a.fw = fr->w.p;
    a.ffr = fr->frames.p;
    a.fcoeff = fr->coeff.p;
    a.fref = fr->ref.p;
    a.feps = fr->eps;
  }
  IBF_TRY(s->epart.reserve((size_t)(a.bv + a.bt + a.bc + a.bf) * MAXT));
  a.part = s->epart.p;
  {
    // algorithmic: 120 B/tet + x_hat, p, x_tilde, mass (80 B/vertex) + 232 B per
    // constraint, read once for all n_r trial points
    KernelClock kc(KC_ENERGY, st, 120.0 * s->m + 80.0 * s->n + 232.0 * a.nc,
                   kEnergyFlopPerTetPoint * (double)s->m * n_r, (double)n_r);
    k_energy<<<a.bv + a.bt + a.bc + a.bf, 256, 0, st>>>(a);
    IBF_LAUNCH_CHECK();
  }
  k_energy_final<<<1, 32 * MAXT, 0, st>>>(s->epart.p, n_r, a.bv, a.bt, a.bc, a.bf, h * h, out_dev);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

int system_inversion_cap_launch(ibf_system* s, const double* x, const double* p, double* out_dev,
                                cudaStream_t st) {
  k_fill<<<1, 1, 0, st>>>(out_dev, 1.0, 1);
  IBF_LAUNCH_CHECK();
  if (s->has_nh && s->m) {
    k_inversion_cap<<<(int)std::min<int64_t>(div_up(s->m, 128), 148LL * 16), 128, 0, st>>>(
        s->m, s->tets.p, s->shape_rows.p, s->regions.p, s->n_regions, x, p, out_dev);
    IBF_LAUNCH_CHECK();
  }
  return IBF_OK;
}

}  // namespace ibf

ibf::Operator ibf_system::op() const {
  ibf::Operator o = pat.op();
  o.pinv = pinv.p;
  o.mask = assembled_dbc ? dbc.p : nullptr;
  if (assembled_contacts) o.contact = ibf::contact_view(assembled_contacts);
  if (assembled_friction && friction) o.friction = ibf::friction_view(friction);
  return o;
}

using namespace ibf;

extern "C" int ibf_system_create(int64_t n_verts, const double* masses, const uint8_t* dbc_mask, int n_regions,
                                 const int* models, const double* mus, const double* lams,
                                 const int64_t* region_tets, const int64_t* tets, const double* shape_rows,
                                 const double* volumes, ibf_system** out) {
  if (n_verts < 0 || n_regions < 0 || !out || n_verts >= (1LL << 30)) {
    set_error("ibf_system_create: bad arguments");
    return IBF_ERR_BAD_ARG;
  }
  int64_t m = 0;
  for (int r = 0; r < n_regions; ++r) {
    if (models[r] < 0 || models[r] > 3 || region_tets[r] < 0) {
      set_error("ibf_system_create: bad region");
      return IBF_ERR_BAD_ARG;
    }
    m += region_tets[r];
  }
  if (m >= (1LL << 28)) {
    set_error("ibf_system_create: too many tets for int32 gather maps");
    return IBF_ERR_BAD_ARG;
  }
  for (int64_t k = 0; k < 4 * m; ++k)
    if (tets[k] < 0 || tets[k] >= n_verts) {
      set_error("ibf_system_create: tet index out of range");
      return IBF_ERR_BAD_ARG;
    }
  ibf_system* s = new ibf_system();
  s->n = n_verts;
  s->m = m;
  s->n_tiles = div_up(m, 32);
  s->n_regions = n_regions;
  int64_t off = 0;
  for (int r = 0; r < n_regions; ++r) {
    RegionDev rg;
    rg.model = models[r];
    rg.begin = (int)off;
    off += region_tets[r];
    rg.end = (int)off;
    rg.pad = 0;
    rg.mu = mus[r];
    rg.lam = lams[r];
    s->regions_host.push_back(rg);
    if (rg.model == IBF_NH && rg.end > rg.begin) s->has_nh = true;
  }
  const int n = (int)n_verts;
  // --- tets int32
  std::vector<int> t32(4 * m);
  for (int64_t k = 0; k < 4 * m; ++k) t32[k] = (int)tets[k];
  // --- pattern: per-row buckets of (col, src) in tet order, then unique cols
  std::vector<int> rcount(n + 1, 0);
  static const int QI[10] = {0, 0, 0, 0, 1, 1, 1, 2, 2, 3};
  static const int QJ[10] = {0, 1, 2, 3, 1, 2, 3, 2, 3, 3};
  for (int64_t t = 0; t < m; ++t)
    for (int q = 0; q < 10; ++q) {
      const int a = t32[4 * t + QI[q]], b = t32[4 * t + QJ[q]];
      rcount[std::min(a, b) + 1]++;
    }
  for (int i = 0; i < n; ++i) rcount[i + 1] += rcount[i];
  std::vector<int> fill(rcount.begin(), rcount.end() - 1);
  std::vector<int> ecol(rcount[n]), esrc(rcount[n]);
  for (int64_t t = 0; t < m; ++t)
    for (int q = 0; q < 10; ++q) {
      const int a = t32[4 * t + QI[q]], b = t32[4 * t + QJ[q]];
      const int r = std::min(a, b), k = fill[r]++;
      ecol[k] = std::max(a, b);
      esrc[k] = (int)(t * 10 + q);
    }
  std::vector<int> blk_ptr, blk_src;
  std::vector<int64_t> rows_h, cols_h;
  blk_src.reserve(rcount[n]);
  rows_h.reserve(rcount[n] / 3 + n);
  cols_h.reserve(rcount[n] / 3 + n);
  std::vector<int> idx;
  auto open_block = [&](int r, int c) {
    rows_h.push_back(r);
    cols_h.push_back(c);
    blk_ptr.push_back((int)blk_src.size());
  };
  for (int i = 0; i < n; ++i) {
    const int e0 = rcount[i], e1 = rcount[i + 1];
    idx.resize(e1 - e0);
    std::iota(idx.begin(), idx.end(), e0);
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return ecol[x] < ecol[y]; });
    // the diagonal (mass) block always exists and comes first (cols >= i)
    if (idx.empty() || ecol[idx[0]] != i) open_block(i, i);
    for (size_t k = 0; k < idx.size(); ++k) {
      const int c = ecol[idx[k]];
      if (k == 0 || c != ecol[idx[k - 1]]) open_block(i, c);
      blk_src.push_back(esrc[idx[k]]);
    }
  }
  blk_ptr.push_back((int)blk_src.size());
  // --- vertex <- tet incidences in tet order
  std::vector<int> vt_ptr(n + 1, 0), vt_src(4 * m);
  for (int64_t k = 0; k < 4 * m; ++k) vt_ptr[t32[k] + 1]++;
  for (int i = 0; i < n; ++i) vt_ptr[i + 1] += vt_ptr[i];
  {
    std::vector<int> f(vt_ptr.begin(), vt_ptr.end() - 1);
    for (int64_t t = 0; t < m; ++t)
      for (int l = 0; l < 4; ++l) vt_src[f[t32[4 * t + l]]++] = (int)(4 * t + l);
  }
  int st = IBF_OK;
  std::vector<uint8_t> dbc(n, 0);
  if (dbc_mask)
    for (int i = 0; i < n; ++i) {
      dbc[i] = dbc_mask[i] ? 1 : 0;
      s->any_dbc |= dbc[i] != 0;
    }
  if (st == IBF_OK) st = s->pat.build(n, rows_h, cols_h);
  // contribution lists re-indexed by storage block (padding blocks: none)
  std::vector<int> qptr, qsrc;
  if (st == IBF_OK) {
    std::vector<int> cnt(s->pat.nq + 1, 0), first(s->pat.nq, -1);
    for (int64_t b = 0; b < s->pat.nb; ++b) {
      cnt[s->pat.q_of_b[b] + 1] = blk_ptr[b + 1] - blk_ptr[b];
      first[s->pat.q_of_b[b]] = (int)b;
    }
    for (int64_t q = 0; q < s->pat.nq; ++q) cnt[q + 1] += cnt[q];
    qptr = cnt;
    qsrc.resize(std::max<size_t>(blk_src.size(), 1));
    for (int64_t q = 0; q < s->pat.nq; ++q)
      if (first[q] >= 0)
        std::copy(blk_src.begin() + blk_ptr[first[q]], blk_src.begin() + blk_ptr[first[q] + 1],
                  qsrc.begin() + qptr[q]);
  }
  const size_t nt = (size_t)std::max<int64_t>(s->n_tiles, 1);
  if (st == IBF_OK) st = s->blk_ptr.upload(qptr.data(), qptr.size());
  if (st == IBF_OK) st = s->blk_src.upload(qsrc.data(), qsrc.size());
  if (st == IBF_OK) st = s->vt_ptr.upload(vt_ptr.data(), vt_ptr.size());
  if (st == IBF_OK) st = s->vt_src.upload(vt_src.data(), vt_src.size());
  if (st == IBF_OK) st = s->tets.upload(t32.data(), t32.size());
  if (st == IBF_OK) st = s->shape_rows.upload(shape_rows, 12 * (size_t)m);
  if (st == IBF_OK) st = s->volumes.upload(volumes, (size_t)m);
  if (st == IBF_OK) st = s->masses.upload(masses, (size_t)n);
  if (st == IBF_OK) st = s->dbc.upload(dbc.data(), dbc.size());
  if (st == IBF_OK) st = s->regions.upload(s->regions_host.data(), s->regions_host.size());
  if (st == IBF_OK) st = s->pinv.reserve(PINV_STRIDE * (size_t)std::max(n, 1));
  if (st == IBF_OK) st = s->elem_grad.reserve(nt * 384);
  if (st == IBF_OK) st = s->elem_blk.reserve(nt * 2880);
  if (st == IBF_OK) st = s->flags.reserve(4);
  if (st == IBF_OK) st = s->dscal.reserve(64);
  if (st == IBF_OK) st = s->vec_a.reserve(3 * (size_t)std::max(n, 1));
  if (st == IBF_OK) st = s->vec_b.reserve(3 * (size_t)std::max(n, 1));
  if (st == IBF_OK) st = s->vec_c.reserve(3 * (size_t)std::max(n, 1));
  if (st == IBF_OK) st = s->host.reserve(256);
  if (st == IBF_OK) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      set_error(std::string("ibf_system_create: ") + cudaGetErrorString(e));
      st = IBF_ERR_CUDA;
    }
  }
  if (st != IBF_OK) {
    delete s;
    return st;
  }
  *out = s;
  return IBF_OK;
}

extern "C" void ibf_system_destroy(ibf_system* s) { delete s; }

extern "C" int ibf_system_pattern(const ibf_system* s, int64_t* n_blocks, int64_t* n_lower) {
  *n_blocks = s->pat.nb;
  *n_lower = s->pat.nl;
  return IBF_OK;
}

extern "C" int ibf_assemble(ibf_system* s, ibf_contacts* c, const double* x_hat, const double* x_tilde, double mu,
                            double offset, double h, int apply_dbc, double* grad, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t stream = (cudaStream_t)st;
  IBF_TRY(system_assemble(s, c, x_hat, x_tilde, mu, offset, h, apply_dbc != 0, grad, false, stream));
  // NonFiniteEnergyError semantics: report synchronously
  IBF_CUDA(cudaMemcpyAsync(s->host.p, s->flags.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream));
  IBF_CUDA(cudaStreamSynchronize(stream));
  if (((int*)s->host.p)[0]) {
    set_error("elastic energy is not finite at the evaluation point");
    return IBF_ERR_NONFINITE;
  }
  return IBF_OK;
}

extern "C" int ibf_system_matvec(ibf_system* s, const double* x, double* y, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  return spmv(s->op(), x, y, (cudaStream_t)st);
}

extern "C" int ibf_system_export_bsr(ibf_system* s, int64_t* rows, int64_t* cols, double* blocks, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  return sell_export(s->pat, rows, cols, blocks, (cudaStream_t)st);
}

// Explicit upper cliques of the matrix-free terms of the last assembly, in
// the reference's COO form (clique_contributions, intact/sparse.py:17-36):
// per term the 10 (i <= j) local pairs of triu_indices(4), block
// coef * g_i g_j^T (contacts, ConstraintBatch.hessian_grids,
// intact/contact.py:139-141) or w_i w_j H (friction, intact/friction.py:88-100),
// transposed when the global row > col.  Contacts first, then friction.
__global__ void k_term_blocks(ContactView cv, FrictionView fv, int64_t* rows, int64_t* cols, double* blocks) {
  const int64_t n_terms = (int64_t)cv.n + fv.n;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < 10 * n_terms;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = id / 10;
    int q = (int)(id - 10 * t), i = 0;
    while (q >= 4 - i) {   // q -> (i, j) of triu_indices(4), row-major
      q -= 4 - i;
      ++i;
    }
    const int j = i + q;
    double B[9];
    int vi, vj;
    if (t < cv.n) {
      const int c = (int)t;
      vi = cv.quad[4 * c + i];
      vj = cv.quad[4 * c + j];
      const double* gi = cv.grad + 12 * c + 3 * i;
      const double* gj = cv.grad + 12 * c + 3 * j;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) B[3 * a + b] = cv.coef[c] * gi[a] * gj[b];
    } else {
      const int k = (int)(t - cv.n);
      vi = fv.quad[4 * k + i];
      vj = fv.quad[4 * k + j];
      const double w = fv.w[4 * k + i] * fv.w[4 * k + j];
      for (int e = 0; e < 9; ++e) B[e] = w * fv.hw[9 * k + e];
    }
    const bool sw = vi > vj;
    rows[id] = sw ? vj : vi;
    cols[id] = sw ? vi : vj;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) blocks[9 * id + 3 * a + b] = sw ? B[3 * b + a] : B[3 * a + b];
  }
}

extern "C" int ibf_system_export_terms(ibf_system* s, int64_t* n_blocks, int64_t* rows, int64_t* cols,
                                       double* blocks, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t stream = (cudaStream_t)st;
  const Operator o = s->op();
  const int64_t nb = 10 * ((int64_t)o.contact.n + o.friction.n);
  if (n_blocks) *n_blocks = nb;
  if (!rows || nb == 0) return IBF_OK;
  DevBuf<int64_t> dr, dc;
  DevBuf<double> db;
  IBF_TRY(dr.reserve(nb));
  IBF_TRY(dc.reserve(nb));
  IBF_TRY(db.reserve(9 * nb));
  k_term_blocks<<<(int)std::min<int64_t>(div_up(nb, 256), 4LL * 148), 256, 0, stream>>>(o.contact, o.friction, dr.p,
                                                                                       dc.p, db.p);
  IBF_LAUNCH_CHECK();
  IBF_CUDA(cudaMemcpyAsync(rows, dr.p, nb * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  IBF_CUDA(cudaMemcpyAsync(cols, dc.p, nb * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  IBF_CUDA(cudaMemcpyAsync(blocks, db.p, 9 * nb * sizeof(double), cudaMemcpyDeviceToHost, stream));
  IBF_CUDA(cudaStreamSynchronize(stream));
  return IBF_OK;
}

extern "C" int ibf_system_pcg(ibf_system* s, const double* rhs, double* x_out, double rel_tol, int64_t max_iters,
                              double* info_host, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t stream = (cudaStream_t)st;
  IBF_TRY(system_pcg(s, rhs, x_out, rel_tol, max_iters, stream));
  return pcg_info(s->work, info_host, stream);
}

extern "C" int ibf_incremental_energy(ibf_system* s, ibf_contacts* c, const double* x_hat, const double* p, int n_r,
                                      const double* r_host, const double* x_tilde, double mu, double offset,
                                      double h, double* energies_host, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t stream = (cudaStream_t)st;
  const int T = p ? n_r : 1;
  IBF_TRY(system_energy_launch(s, c, x_hat, p, T, r_host, nullptr, x_tilde, mu, offset, h, s->dscal.p, stream));
  IBF_CUDA(cudaMemcpyAsync(energies_host, s->dscal.p, T * sizeof(double), cudaMemcpyDeviceToHost, stream));
  IBF_CUDA(cudaStreamSynchronize(stream));
  return IBF_OK;
}

extern "C" int ibf_inversion_safe_step(ibf_system* s, const double* x, const double* p, double* out_host,
                                       ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t stream = (cudaStream_t)st;
  IBF_TRY(system_inversion_cap_launch(s, x, p, s->dscal.p, stream));
  IBF_CUDA(cudaMemcpyAsync(out_host, s->dscal.p, sizeof(double), cudaMemcpyDeviceToHost, stream));
  IBF_CUDA(cudaStreamSynchronize(stream));
  *out_host = std::max(*out_host, 0.0);
  return IBF_OK;
}

extern "C" int ibf_stiffness_diagonal_max(ibf_system* s, const double* x, double h, double* out_host,
                                          ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t stream = (cudaStream_t)st;
  if (s->n == 0) {
    *out_host = 1.0;
    return IBF_OK;
  }
  // contact- and friction-free system (intact/stepper.py:197)
  ibf_friction* keep_friction = s->friction;
  s->friction = nullptr;
  const int st_asm = system_assemble(s, nullptr, x, x, 1.0, 1.0, h, false, s->vec_a.p, false, stream);
  s->friction = keep_friction;
  IBF_TRY(st_asm);
  k_fill<<<1, 1, 0, stream>>>(s->dscal.p + 8, 0.0, 1);
  k_diag_max<<<(int)std::min<int64_t>(div_up(s->n, 256), 148 * 4), 256, 0, stream>>>(s->n, s->pat.diag_q.p,
                                                                                       s->pat.val.p, s->dscal.p + 8);
  IBF_LAUNCH_CHECK();
  IBF_CUDA(cudaMemcpyAsync(s->host.p, s->flags.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream));
  IBF_CUDA(cudaMemcpyAsync(out_host, s->dscal.p + 8, sizeof(double), cudaMemcpyDeviceToHost, stream));
  IBF_CUDA(cudaStreamSynchronize(stream));
  if (((int*)s->host.p)[0]) {
    set_error("elastic energy is not finite at the evaluation point");
    return IBF_ERR_NONFINITE;
  }
  return IBF_OK;
}
