// Internal structures shared by the libibf translation units.
#pragma once

#include "common.cuh"

namespace ibf {

// Material region (ElasticRegion, intact/solver.py:40-47) over a tet range.
struct RegionDev {
  int model;
  int begin;
  int end;
  int pad;
  double mu;
  double lam;
};

// Matrix-free contact operator: H_c = sum_c coef_c g_c g_c^T over the 12-dof
// clique of constraint c, with DBC masking applied on both sides.
struct ContactView {
  int n = 0;                          // C
  const int* quad = nullptr;          // (C,4)
  const double* grad = nullptr;       // (C,12) anchor gradients
  const double* coef = nullptr;       // (C) mu * gamma
  const int* vc_ptr = nullptr;        // (N+1) vertex -> incidences
  const int* vc_src = nullptr;        // c*4 + slot, ordered by c
  double* t = nullptr;                // (C) workspace coef_c * g_c . p
};

// Symmetric operator: upper BSR (diagonal first in each row) + transpose
// index + optional matrix-free contact term + block-Jacobi inverse.
struct Operator {
  int n = 0;
  const int* row_ptr = nullptr;       // (n+1)
  const int* col = nullptr;           // (nb)
  const double* val = nullptr;        // (nb,9)
  const int* low_ptr = nullptr;       // (n+1)
  const int2* low_pair = nullptr;     // (nl) (block b, row(b)) with col(b) = row, row(b) < col
  const uint8_t* mask = nullptr;      // (n) DBC mask (contact masking) or null
  const double* pinv = nullptr;       // (n,9) inverse diagonal blocks
  ContactView contact;
};

struct PcgWork {
  DevBuf<double> r, z, p, hp, X, part, info;
  HostScratch host;
  int grid = 0;
  int n_alloc = -1;
};

int pcg_solve(const Operator& op, const double* rhs, double* x_out, double rel_tol,
              int64_t max_iters, PcgWork& w, cudaStream_t s);
// after pcg_solve: (iterations, converged, rel_residual) on the host (syncs).
int pcg_info(PcgWork& w, double info[3], cudaStream_t s);
int spmv(const Operator& op, const double* x, double* y, cudaStream_t s);
// inverse of 3x3 diagonal blocks into pinv (n,9): diag given as block ids
int invert_diag_blocks(int n, const double* val, const int* diag_blk, double* pinv, cudaStream_t s);

}  // namespace ibf

// ----------------------------------------------------------- opaque handles

struct ibf_contacts {
  int admit_all = 0;
  int64_t n = 0;              // resident count
  int64_t n_verts = 0;
  // SoA, insertion order
  ibf::DevBuf<int> kind, quad;
  ibf::DevBuf<double> lam, gamma, s, anchor_d, anchor_grad, anchor_x;
  // per-subproblem derived data
  ibf::DevBuf<double> coef_h, coef_g, cval;   // mu*gamma, gradient coefficient, c
  ibf::DevBuf<double> tdot;                   // SpMV workspace (C)
  ibf::DevBuf<int> vc_ptr, vc_src;
  ibf::DevBuf<int> sort_keys, sort_vals, sort_keys2, sort_vals2;
  ibf::DevBuf<unsigned char> cub_tmp;
  int64_t vc_nverts = -1;
  // update scratch
  ibf::DevBuf<int> v_count, v_ptr, v_list, k_count, k_ptr, k_list, flags, pos;
  ibf::DevBuf<double> earliest;
  ibf::DevBuf<int> tmp_kind, tmp_quad;
  ibf::DevBuf<double> tmp_tois;
  ibf::DevBuf<double> dscratch;
  ibf::DevBuf<int> iscratch;
  ibf::HostScratch host;
};

struct ibf_ccd {
  int64_t nt = 0, ne = 0, nv = 0;
  ibf::DevBuf<int> tris, edges, verts;
  // LBVH scratch (per tree)
  ibf::DevBuf<double> box_lo, box_hi, qlo, qhi;        // primitive boxes / query boxes (n,3)
  ibf::DevBuf<unsigned long long> keys, keys_sorted;
  ibf::DevBuf<int> order;                               // sorted primitive order
  ibf::DevBuf<int> node_left, node_right, node_parent, node_flag;
  ibf::DevBuf<double> node_lo, node_hi;
  ibf::DevBuf<unsigned char> cub_tmp;
  // candidate / survivor pairs
  ibf::DevBuf<unsigned long long> pairs, pairs_sorted;
  ibf::DevBuf<unsigned long long> counters;             // [0] emitted, [1] all candidates
  ibf::DevBuf<double> pair_toi;
  int64_t n_vf = 0, n_ee = 0;                           // candidates of the last call
  // blocking set
  ibf::DevBuf<int> b_kind, b_quad;
  ibf::DevBuf<double> b_toi;
  ibf::DevBuf<int> b_flag, b_pos;
  ibf::DevBuf<int> s_quad[2], s_pos;                    // survivors (VF, EE)
  ibf::DevBuf<double> s_toi[2];
  ibf::DevBuf<double> dscratch;
  int64_t n_block = 0;
  ibf::HostScratch host;
  ibf::PhaseTimer t_ccd;
  long long n_candidates = 0;    // broad-phase candidates since the last stats reset
};
