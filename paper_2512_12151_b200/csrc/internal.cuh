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

// k_pcg applies the contact terms of a warp's 32 rows cooperatively (lanes
// over the rows' concatenated term records) instead of one row per lane
#ifndef IBF_PCG_WARP_TERMS
#define IBF_PCG_WARP_TERMS 1
#endif

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
  // per-row term records of the unmasked rows (contact_pack_terms), or null
  const int* ip_ptr = nullptr;        // (N+1)
  const double4* rec = nullptr;       // {g_c[slot], c}, in vc order
};

// Symmetric 3x3-block matrix (diagonal + strict upper, the reference's
// information content, intact/sparse.py:1-5) in sliced-ELL storage:
//
//   rows are grouped in slices of C = SELL_C (16); slice s holds w_s = max
//   upper count of its rows "slots"; block (row i, slot k) has storage index
//   q = slice_ptr[s] + C k + (i mod C), and entry e (row-major 3x3) of block
//   q lives at val[qel(q, e)] = val[9 (q & ~(C-1)) + (q & (C-1)) + C e].
//
// So when the 32 lanes of a warp take the 32 rows of two slices, every load
// of one block entry is two contiguous 128-byte segments, and the transposed
// read of the lower blocks of consecutive rows touches a few contiguous
// segments (their source blocks sit in consecutive rows of the same slot on
// structured meshes).  C = 16 rather than 32 halves the rows a slice's width
// is the maximum over: on the squishy balls the upper padding falls from 26 %
// to 21 % and the lower from 29 % to 23 %, and k_pcg from 187 to 179 us per
// CG iteration without contacts (C = 8: 184 us, the 64-byte segments cost L1
// wavefronts).  Once rows stop at their first padded slot (pcg.cu,
// IBF_SELL_STOP) 16 and 32 measure the same; 16 builds without spills.  The lower triangle is applied via a
// per-row list of (storage block, source row) entries stored the same way.
// Padding blocks are zero with col = own row; padding lower entries point at
// a zero block past the last slice.
//
// IBF_BLOCK_AOS builds (experiment) keep each block's 9 entries contiguous
// instead: val[9 q + e].
#ifndef IBF_BLOCK_AOS
#define IBF_BLOCK_AOS 0
#endif
// slice height of the sliced-ELL storage (IBF_SELL_C: 32, 16 or 8 rows)
#ifndef IBF_SELL_C
#define IBF_SELL_C 16
#endif
constexpr int SELL_C = IBF_SELL_C;
constexpr int SELL_SHIFT = SELL_C == 32 ? 5 : (SELL_C == 16 ? 4 : (SELL_C == 8 ? 3 : -1));
static_assert(SELL_SHIFT > 0, "IBF_SELL_C must be 8, 16 or 32");
constexpr int QEL_ES = IBF_BLOCK_AOS ? 1 : SELL_C;   // stride between entries of a block
constexpr int QEL_LS = IBF_BLOCK_AOS ? 9 : 1;        // stride between lanes of a slice
__host__ __device__ __forceinline__ size_t qel(int q, int e) {
  if (IBF_BLOCK_AOS) return 9 * (size_t)q + e;
  return 9 * (size_t)(q & ~(SELL_C - 1)) + (size_t)(q & (SELL_C - 1)) + SELL_C * (size_t)e;
}

// Matrix-free friction term (intact/friction.py:85-100): per term k the
// 12x12 clique w w^T (x) Hw_k, Hw_k = coeff T [g2 uu^T + g1 (I - uu^T)] T^T
// (3x3, symmetric PSD), applied as t_k = Hw_k sum_j w_j p_j, y_i += w t_k.
struct FrictionView {
  int n = 0;                          // K terms
  const int* quad = nullptr;          // (K,4)
  const double* w = nullptr;          // (K,4) witness weights
  const double* hw = nullptr;         // (K,9) world-space Hessian
  const int* vf_ptr = nullptr;        // (N+1) vertex -> term incidences
  const int* vf_src = nullptr;        // k*4 + slot, ordered by k
  double* t = nullptr;                // (K,3) workspace
};

// Block-Jacobi inverse: the diagonal blocks are symmetric, so their inverse
// is stored as its upper triangle (00, 01, 02, 11, 12, 22) — 48 instead of
// 72 bytes per vertex streamed by every CG iteration.
constexpr int PINV_STRIDE = 6;

__device__ __forceinline__ void inv3_sym6(const double* A, double* P) {
  const double c00 = A[4] * A[8] - A[5] * A[7];
  const double c01 = A[5] * A[6] - A[3] * A[8];
  const double c02 = A[3] * A[7] - A[4] * A[6];
  const double id = 1.0 / (A[0] * c00 + A[1] * c01 + A[2] * c02);
  P[0] = c00 * id;
  P[1] = (A[2] * A[7] - A[1] * A[8]) * id;
  P[2] = (A[1] * A[5] - A[2] * A[4]) * id;
  P[3] = (A[0] * A[8] - A[2] * A[6]) * id;
  P[4] = (A[2] * A[3] - A[0] * A[5]) * id;
  P[5] = (A[0] * A[4] - A[1] * A[3]) * id;
}

__device__ __forceinline__ void apply_pinv6(const double* __restrict__ P, double r0, double r1, double r2,
                                            double z[3]) {
  const double p0 = P[0], p1 = P[1], p2 = P[2], p3 = P[3], p4 = P[4], p5 = P[5];
  z[0] = p0 * r0 + p1 * r1 + p2 * r2;
  z[1] = p1 * r0 + p3 * r1 + p4 * r2;
  z[2] = p2 * r0 + p4 * r1 + p5 * r2;
}

struct Operator {
  int n = 0;
  const int* perm = nullptr;          // (n) storage position -> row (null: identity)
  const int* slice_ptr = nullptr;     // (S+1) storage block offset per slice
  const int* col = nullptr;           // (nq) column of each storage block
  const double* val = nullptr;        // 9 (nq + 32) entries, qel layout
  size_t val_bytes = 0;
  const int* low_ptr = nullptr;       // (S+1) lower-entry offset per slice
  const int2* low = nullptr;          // (nlq) (storage block, source row)
  int zero_q = 0;                     // storage index of the zero block padded lower entries point at
  const uint8_t* mask = nullptr;      // (n) DBC mask (contact masking) or null
  const double* pinv = nullptr;       // (n,6) inverse diagonal blocks (upper triangle)
  ContactView contact;
  FrictionView friction;
};

// row held at storage position pos (slices are over positions, vectors over rows)
__device__ __forceinline__ int row_at(const Operator& op, int pos) { return op.perm ? __ldg(op.perm + pos) : pos; }

// Host + device halves of the sliced symmetric pattern (built once).
//
// Rows can be placed at storage positions in windows of SELL_WINDOW rows,
// each window sorted by (upper count, lower count) descending, so the 32 rows
// of a slice have near-equal slot counts (vectors stay in row order; the
// permutation only changes which thread takes which row).  On the squishy
// balls lattice order leaves 36 % of the upper slots and 41 % of the lower
// entries as padding, 256-row windows 6 % and 16 % — and k_pcg measured
// 201 / 219 / 255 us per CG iteration with windows of 1 / 64 / 256 rows
// (DESIGN.md): the scattered per-row vector accesses cost more than the
// padding.  Default 1 (positions = rows).
#ifndef IBF_SELL_WINDOW
#define IBF_SELL_WINDOW 1
#endif
constexpr int SELL_WINDOW = IBF_SELL_WINDOW;   // 1: no sorting (positions = rows)
struct SellPattern {
  int64_t n = 0, nb = 0, nl = 0;      // rows, real blocks, real strict-upper blocks
  int n_slices = 0;
  int64_t nq = 0, nlq = 0;            // storage blocks / lower entries incl. padding
  int zero_q = 0;                     // an all-zero storage block
  std::vector<int64_t> rows, cols;    // real blocks sorted by (row, col)
  std::vector<int> q_of_b;            // real block -> storage index
  std::vector<int> perm_h;            // storage position -> row
  DevBuf<int> perm, slice_ptr, col, qrow, low_ptr, diag_q;
  DevBuf<uint8_t> qreal;
  DevBuf<int2> low;
  DevBuf<double> val;
  // rows/cols: real blocks sorted by (row, col); uploads the device arrays
  // and allocates val (zeroed).
  int build(int64_t n, const std::vector<int64_t>& rows, const std::vector<int64_t>& cols);
  Operator op() const;
};

struct PcgWork {
  DevBuf<double> r, z, p, hp, X, part, info;
  HostScratch host;
  DevBuf<unsigned long long> prof;   // IBF_PCG_PROFILE builds only
  DevBuf<int> counter;               // dynamic phase-A chunk counters
  DevBuf<double> part_chunk;         // dynamic phase-A per-chunk partials
  DevBuf<unsigned> ready;            // term-dot ready counter
  DevBuf<double> zdot, pdot;         // zdot mode: per-record z and previous-direction products
  DevBuf<double> tprev;              // linear-recursion contact dots: g_c . p_{k-1}
  DevBuf<int> wcounter;              // warp-dynamic phase A: slice counters + group counts
  DevBuf<double> part_unit;          // warp-dynamic phase A: slice and group partials
  int grid = 0;
  int n_alloc = -1;
};

int pcg_solve(const Operator& op, const double* rhs, double* x_out, double rel_tol,
              int64_t max_iters, PcgWork& w, cudaStream_t s);

// ---- row-partitioned PCG (SURVEY.md §8(e), C4 over several GPUs) ----
// Rows are split into `world` contiguous chunks of `chunk` rows (a multiple
// of 32); partition r owns rows [r*chunk, min(n, (r+1)*chunk)).  Every
// partition holds the whole (replicated) operator and full-length z / p
// vectors, computes q = H p only for its own rows, keeps p valid on its halo
// (the rows its own rows' blocks and every contact / friction term touch),
// and exchanges per CG iteration: one allreduce of pAp, one of (|r|^2, r.z),
// and one allgather of its z rows.  The exchanges go through a DistComm:
// NCCL across processes (one GPU each), or "local" — all partitions in this
// process, allgather as device copies — which is how one GPU tests the
// partition arithmetic against the unpartitioned solve.
struct PartBuf;
struct DistWork {
  std::vector<PartBuf*> parts;         // the partitions this process runs
  DevBuf<double> gsc;                  // reduced scalars (allreduce result)
  DevBuf<double> xfull;                // padded full x (restart, result gather)
  DevBuf<int> counter;
  DevBuf<unsigned long long> ptrs;     // device copy of the partitions' scalar buffers (local mode)
  int ptrs_n = -1;
  HostScratch host;
  int64_t n = -1, chunk = 0;
  int world = 0;
  ~DistWork();
};
int pcg_solve_dist(const Operator& op, const std::vector<int64_t>& brows, const std::vector<int64_t>& bcols,
                   const double* rhs, double* x_out, double rel_tol, int64_t max_iters, PcgWork& w, DistWork& dw,
                   ibf_dist* d, cudaStream_t s);
// communicator primitives (dist.cu); in place, on stream s
int dist_allreduce_sum(ibf_dist* d, double* buf, int count, cudaStream_t s);
int dist_allgather(ibf_dist* d, const double* send, double* recv, size_t count_per_rank, cudaStream_t s);
// after pcg_solve: (iterations, converged, rel_residual) on the host (syncs).
int pcg_info(PcgWork& w, double info[3], cudaStream_t s);
// host copy of the real blocks (sorted (row, col) order, (nb,9)) of a pattern
int sell_export(const SellPattern& P, int64_t* rows, int64_t* cols, double* blocks, cudaStream_t s);
int spmv(const Operator& op, const double* x, double* y, cudaStream_t s);
// inverse of 3x3 diagonal blocks into pinv (n,9): diag given as block ids
int invert_diag_blocks(int n, const double* val, const int* diag_q, double* pinv, cudaStream_t s);

}  // namespace ibf

// ----------------------------------------------------------- opaque handles

// Row partition of the PCG over `world` partitions (ibf_dist_create*).
struct ibf_dist {
  int rank = 0, world = 1;
  bool local = true;        // all partitions in this process (no NCCL)
  void* comm = nullptr;     // ncclComm_t when !local
};

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
  ibf::DevBuf<int> ip_ptr;                    // PCG term records (contact_pack_terms)
  ibf::DevBuf<double4> trec;
  int64_t trec_nverts = -1;
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
  ibf::DevBuf<double> compact_tmp;            // pruning scratch (8-byte words)
  ibf::HostScratch host;
};

// Frozen friction terms (FrictionTerms, intact/friction.py:56-100).
struct ibf_friction {
  int64_t n = 0;
  double eps = 0.0;                 // h * eps_v
  ibf::DevBuf<int> quad;            // (K,4)
  ibf::DevBuf<double> w, frames, coeff, ref;   // (K,4), (K,3,2), (K), (K,3)
  ibf::DevBuf<double> gw, hw, tvec;            // per assembly: (K,3) force, (K,9) Hessian, SpMV workspace
  ibf::DevBuf<int> vf_ptr, vf_src, v_count, keys, keys2, vals;
  int64_t vf_nverts = -1;
  // precompute scratch (per constraint)
  ibf::DevBuf<int> flags, pos;
  ibf::DevBuf<double> t_w, t_frames, t_coeff, t_ref;
  ibf::DevBuf<int> t_quad;
  ibf::DevBuf<unsigned char> cub_tmp;
  ibf::HostScratch host;
};

struct ibf_ccd {
  int64_t nt = 0, ne = 0, nv = 0;
  ibf::DevBuf<int> tris, edges, verts;
  // LBVH scratch (per tree)
  ibf::DevBuf<double> box_lo, box_hi, qlo, qhi;        // primitive boxes / query boxes (n,3)
  ibf::DevBuf<unsigned long long> keys, keys_sorted;
  ibf::DevBuf<int> order;                               // sorted primitive order
  ibf::DevBuf<int> node_left, node_right, node_parent, node_flag, node_last;
  ibf::DevBuf<double> node_lo, node_hi;
  ibf::DevBuf<float4> node_packed;                      // 4 per internal node (ccd.cu PackedNode)
  ibf::DevBuf<float4> node_wide;                        // 8 per internal node (ccd.cu WideNode)
  ibf::DevBuf<uint8_t> node_odd;
  ibf::DevBuf<double4> node_lbox;
  // VF (triangle) and EE (edge) trees kept between calls: later calls refit
  // the cached topology to the new boxes; it is rebuilt every few calls
  struct TreeCache {
    ibf::DevBuf<unsigned long long> keys_sorted;
    ibf::DevBuf<int> left, right, parent, flag, last;
    ibf::DevBuf<double> lo, hi;
    ibf::DevBuf<float4> packed;
    ibf::DevBuf<float4> wide;                            // 4-wide records (8 float4 per internal node)
    ibf::DevBuf<uint8_t> odd;                            // internal-node depth parity
    ibf::DevBuf<double4> lbox;                           // exact leaf records by sorted slot
    ibf::DevBuf<int> first, titems, tcounts, tchunk;     // chunked treelet refit (per topology)
    ibf::DevBuf<uint8_t> tucode, troot;
    int64_t n = -1;
    int uses = 0;
  } tc[2];
  ibf::DevBuf<unsigned char> cub_tmp;
  // candidate / survivor pairs
  ibf::DevBuf<unsigned long long> pairs, pairs2, pairs_sorted;
  ibf::DevBuf<unsigned long long> vf_order;             // VF query order (Morton keys | query)
  int64_t vf_order_n = -1;
  ibf::DevBuf<unsigned long long> counters;             // [0] emitted, [1] all candidates, [2] min-distance
                                                        // pair, [3] traversal query fetch
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
