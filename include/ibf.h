/*
 * ibf.h — C ABI of libibf.so, the B200 (sm_100a) hot path of the barrier-free
 * augmented-Lagrangian elastodynamics solver (arXiv 2512.12151).
 *
 * The reference (`intact`, pure Python + numpy) has no FFI; its hot path sits
 * behind plain Python function seams.  Each entry point below replaces one of
 * those seams (paths relative to /root/reference/pkg/src) and keeps its
 * argument meaning and error behaviour; INTEGRATION.md shows the ctypes
 * binding a maintainer of `intact` would add.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "dev" pointers are CUDA device memory,
 *    "host" pointers are host memory.  Vectors of points are (n,3) float64
 *    row-major, exactly the reference's state layout (intact/mesh.py:52-60).
 *  - Every call is asynchronous on the given stream unless it returns a host
 *    scalar, in which case it synchronises that stream before returning.
 *  - Every call returns an ibf_status; on failure ibf_last_error() holds a
 *    message.  No exception crosses the ABI.  IBF_ERR_NONFINITE maps to the
 *    reference's NonFiniteEnergyError (intact/solver.py:35-37).
 *  - Handles are not re-entrant; one stream per handle.
 */
#ifndef IBF_H
#define IBF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ibf_stream;   /* == cudaStream_t */

typedef enum {
    IBF_OK = 0,
    IBF_ERR_BAD_ARG = 1,
    IBF_ERR_CUDA = 2,
    IBF_ERR_OOM = 3,
    IBF_ERR_NONFINITE = 4,   /* NonFiniteEnergyError, intact/solver.py:35 */
    IBF_ERR_NO_DEVICE = 5,
    IBF_ERR_IO = 6           /* file could not be written: OSError */
} ibf_status;

/* material models — MaterialModel, intact/elasticity.py:31-35 */
enum { IBF_SNH = 0, IBF_NH = 1, IBF_COR = 2, IBF_LIN = 3 };
/* pair kinds — PairKind, intact/distance.py:28-30 */
enum { IBF_VF = 0, IBF_EE = 1 };

const char* ibf_version(void);
const char* ibf_last_error(void);

/* ------------------------------------------------------------------ geometry */

/* Batched pair distance: d (n), grad (n,12), weights (n,4), degenerate (n).
 * Replaces vf_eval / ee_eval + _finish (intact/distance.py:153-189).
 * pts: (n,4,3) dev. Bit-identical to the reference on the build host. */
int ibf_pair_eval(int kind, int64_t n, const double* pts, double* d, double* grad,
                  double* weights, uint8_t* degenerate, ibf_stream s);

/* Additive-CCD TOI per pair in [0,1]. Replaces accd_batch (intact/ccd.py:37-91).
 * x0, x1: (n,4,3) dev; toi: (n) dev. Bit-identical to the reference. */
int ibf_accd(int kind, int64_t n, const double* x0, const double* x1, double min_gap,
             double* toi, ibf_stream s);

/* --------------------------------------------------------------- CCD handle */
typedef struct ibf_ccd ibf_ccd;

/* Surface primitives (host int64 arrays as System stores them,
 * intact/stepper.py:103-113): tris (nt,3), edges (ne,2), verts (nv). */
int ibf_ccd_create(int64_t n_tris, const int64_t* tris, int64_t n_edges, const int64_t* edges,
                   int64_t n_verts, const int64_t* verts, ibf_ccd** out);
void ibf_ccd_destroy(ibf_ccd* c);

/* Broad phase only: replaces candidate_pairs (intact/ccd.py:113-145).
 * Returns counts; fetch the pairs with ibf_ccd_get_candidates. Pairs are
 * ordered (vertex, triangle) / (edge a, edge b) ascending — the set equals the
 * reference's bit-exactly; the reference's order is its BVH frontier order. */
int ibf_ccd_candidates(ibf_ccd* c, const double* x0, const double* x1, double min_gap,
                       int64_t* n_vf, int64_t* n_ee, ibf_stream s);
int ibf_ccd_get_candidates(ibf_ccd* c, int64_t* vf_host, int64_t* ee_host, ibf_stream s);

/* Global step limit: replaces max_step_size (intact/ccd.py:168-193).
 * alpha = min(cap, min TOI); the blocking pairs (TOI < 1, VF first then EE)
 * stay on the device in the handle (ibf_ccd_blocking). */
int ibf_max_step_size(ibf_ccd* c, const double* x, const double* x_hat, double min_gap,
                      double cap, double* alpha_host, int64_t* n_blocking_host, ibf_stream s);
/* Device views of the last blocking set: kinds (n) int32, quads (n,4) int32, tois (n). */
int ibf_ccd_blocking(ibf_ccd* c, const int32_t** kinds, const int32_t** quads,
                     const double** tois, int64_t* n);
/* Host copy of the last blocking set (BlockingPairs, intact/ccd.py:148-165). */
int ibf_ccd_get_blocking(ibf_ccd* c, int64_t* kinds, int64_t* quads, double* tois, ibf_stream s);

/* ----------------------------------------------------- penetration monitor */
/* Static triangle-triangle intersection over the handle's surface triangles
 * at x: replaces static_intersection_test (intact/intersect.py:125-140).
 * n_hits = number of intersecting pairs (a < b, shared-vertex pairs
 * excluded); the first min(cap, n_hits) pairs (ascending) go to pairs_host
 * (cap,2) when it is not NULL. */
int ibf_static_intersection(ibf_ccd* c, const double* x, int64_t* n_hits, int64_t* pairs_host, int64_t cap,
                            ibf_stream s);
/* Nearest non-adjacent VF/EE pair among those whose boxes come within
 * `radius` at x: d_host = its distance (INFINITY without candidates),
 * pair_host (5) = (kind, 4 vertex ids) or -1.  Pairs not tested are farther
 * than radius apart, so d_host > 0 certifies that no surface primitives touch. */
int ibf_min_distance(ibf_ccd* c, const double* x, double radius, double* d_host, int64_t* pair_host,
                     ibf_stream s);

/* ------------------------------------------------------ scene build / export */
typedef struct ibf_surface ibf_surface;

/* Boundary surface of a tet mesh: replaces extract_surface_arrays
 * (intact/mesh.py:106-124).  tets: (m,4) int64 dev, ids in [0, 2^31).
 * Counts come back at once; ibf_surface_get copies tris (n_tris,3) in the
 * tets' face order and winding, edges (n_edges,2) unique sorted, verts
 * (n_verts) unique ascending (int64, host or dev pointers, NULL skips).
 * n_nonmanifold = edges shared by > 2 boundary faces (the reference's warning). */
int ibf_surface_extract(int64_t m, const int64_t* tets, ibf_surface** out, int64_t* n_tris,
                        int64_t* n_edges, int64_t* n_verts, int64_t* n_nonmanifold, ibf_stream s);
int ibf_surface_get(const ibf_surface* h, int64_t* tris, int64_t* edges, int64_t* verts, ibf_stream s);
void ibf_surface_destroy(ibf_surface* h);

/* OBJ frame: replaces export_frame (intact/io_utils.py:35-43).  Host
 * pointers; byte-identical file (repr coordinates, compacted 1-based faces).
 * n_threads <= 0 uses every hardware thread.  Needs no GPU. */
int ibf_export_obj(const char* path, const double* positions, int64_t n_positions, const int64_t* tris,
                   int64_t n_tris, int n_threads);

/* ------------------------------------------------------------ active set */
typedef struct ibf_contacts ibf_contacts;

/* ActiveSet (intact/contact.py:154-261) as device SoA with insertion order. */
int ibf_contacts_create(int64_t n_verts, int admit_all, ibf_contacts** out);
void ibf_contacts_destroy(ibf_contacts* c);
int64_t ibf_contacts_size(const ibf_contacts* c);
/* ActiveSet.update(blocking) with the blocking set of a ccd handle
 * (intact/contact.py:179-205). Returns (admitted, pruned) as the reference counts. */
int ibf_contacts_update(ibf_contacts* c, const ibf_ccd* blocking, int64_t* admitted,
                        int64_t* pruned, ibf_stream s);
/* Same from explicit host arrays: kinds (n), quads (n,4), tois (n). */
int ibf_contacts_update_host(ibf_contacts* c, int64_t n, const int64_t* kinds,
                             const int64_t* quads, const double* tois, int64_t* admitted,
                             int64_t* pruned, ibf_stream s);
/* refresh_anchors (intact/contact.py:207-235); returns the degenerate count. */
int ibf_contacts_refresh_anchors(ibf_contacts* c, const double* x, int64_t* n_degenerate,
                                 ibf_stream s);
/* dual_update_sweep (intact/contact.py:251-261); returns max |c| on the s == 0 branch. */
int ibf_contacts_dual_sweep(ibf_contacts* c, const double* x_hat, double offset, double mu,
                            double decay, double* worst_host, ibf_stream s);
/* Host export/import of the SoA state (kind, quad(4), lam, gamma, s, anchor_d,
 * anchor_grad(12), anchor_x(12)); import replaces the whole set (ActiveSet.add). */
int ibf_contacts_export(const ibf_contacts* c, int64_t* kind, int64_t* quad, double* lam,
                        double* gamma, double* s, double* anchor_d, double* anchor_grad,
                        double* anchor_x, ibf_stream st);
int ibf_contacts_import(ibf_contacts* c, int64_t n, const int64_t* kind, const int64_t* quad,
                        const double* lam, const double* gamma, const double* s,
                        const double* anchor_d, const double* anchor_grad,
                        const double* anchor_x, ibf_stream st);

/* -------------------------------------------------------------- friction */
typedef struct ibf_friction ibf_friction;

/* FrictionTerms (intact/friction.py:56-100) as a device handle. */
int ibf_friction_create(ibf_friction** out);
void ibf_friction_destroy(ibf_friction* f);
int64_t ibf_friction_size(const ibf_friction* f);
/* friction_precompute (intact/friction.py:103-151) from an accepted state x
 * (dev) and the active set's multipliers: one term per constraint with a
 * positive normal force, active-set order; eps = h * eps_v. */
int ibf_friction_precompute(ibf_friction* f, const ibf_contacts* c, const double* x, double mu, double offset,
                            double h, double mu_f, double eps_v, int64_t* n_terms, ibf_stream s);
/* Host import / export of the terms: quad (K,4), w (K,4), frames (K,3,2),
 * coeff (K), ref (K,3), eps. */
int ibf_friction_import(ibf_friction* f, int64_t n, const int64_t* quad, const double* w, const double* frames,
                        const double* coeff, const double* ref, double eps, ibf_stream s);
int ibf_friction_export(const ibf_friction* f, int64_t* quad, double* w, double* frames, double* coeff,
                        double* ref, double* eps, ibf_stream s);

/* --------------------------------------------------------- elastic system */
typedef struct ibf_system ibf_system;

/* System (intact/stepper.py:103-128) + ElasticRegion list (intact/solver.py:40-47):
 * masses (n) host, dbc_mask (n) host (uint8), regions given as per-region
 * (model, mu, lam, n_tets) with their tets (int64, global ids), shape_rows
 * (m,4,3) and volumes (m) concatenated in region order.  Builds the static
 * symmetric BSR pattern (diagonal + upper), the gather maps and workspaces. */
int ibf_system_create(int64_t n_verts, const double* masses, const uint8_t* dbc_mask,
                      int n_regions, const int* models, const double* mus,
                      const double* lams, const int64_t* region_tets,
                      const int64_t* tets, const double* shape_rows,
                      const double* volumes, ibf_system** out);
void ibf_system_destroy(ibf_system* s);
/* pattern sizes: n_blocks = diagonal + strict-upper blocks */
int ibf_system_pattern(const ibf_system* s, int64_t* n_blocks, int64_t* n_lower);

/* assemble (intact/solver.py:109-156): gradient into grad (n,3) dev and the
 * system matrix (mass + h^2 PSD elasticity + mu*gamma rank-one contact terms,
 * DBC-masked) kept in the handle; contacts may be NULL. */
int ibf_assemble(ibf_system* s, ibf_contacts* c, const double* x_hat, const double* x_tilde,
                 double mu, double offset, double h, int apply_dbc, double* grad,
                 ibf_stream st);
/* Friction terms entering subsequent assemble / energy / solve calls on s
 * (the `friction` argument of intact/solver.py:109-233); NULL removes them. */
int ibf_system_set_friction(ibf_system* s, ibf_friction* f);

/* y = H x with the last assembled matrix (BlockSparseMatrix.matvec,
 * intact/sparse.py:64-73, contact part applied matrix-free). */
int ibf_system_matvec(ibf_system* s, const double* x, double* y, ibf_stream st);
/* Host copy of the elastic BSR (rows, cols, blocks) of the last assembly. */
int ibf_system_export_bsr(ibf_system* s, int64_t* rows, int64_t* cols, double* blocks,
                          ibf_stream st);

/* Explicit upper cliques of the last assembly's matrix-free terms, as the
 * reference's COO (clique_contributions, intact/sparse.py:17-36, of
 * ConstraintBatch.hessian_grids, intact/contact.py:139-141, then
 * FrictionTerms.hessian_grids, intact/friction.py:88-100): 10 blocks per term,
 * unmasked, uncoalesced.  rows == NULL only returns the count in n_blocks;
 * otherwise rows, cols (n_blocks) and blocks (n_blocks,3,3) are host arrays. */
int ibf_system_export_terms(ibf_system* s, int64_t* n_blocks, int64_t* rows, int64_t* cols, double* blocks,
                            ibf_stream st);

/* pcg_solve on the last assembled matrix (intact/sparse.py:99-150).
 * info_host = (iterations, converged, rel_residual). max_iters <= 0 -> 10 n. */
int ibf_system_pcg(ibf_system* s, const double* rhs, double* x_out, double rel_tol,
                   int64_t max_iters, double* info_host, ibf_stream st);

/* incremental_energy (intact/solver.py:88-106) at x_hat + r_k p for k < n_r
 * (p may be NULL -> x_hat itself); contacts frozen at their anchors. */
int ibf_incremental_energy(ibf_system* s, ibf_contacts* c, const double* x_hat,
                           const double* p, int n_r, const double* r_host,
                           const double* x_tilde, double mu, double offset, double h,
                           double* energies_host, ibf_stream st);

/* min over regions of inversion_safe_step (intact/elasticity.py:337-356). */
int ibf_inversion_safe_step(ibf_system* s, const double* x, const double* p, double* out_host,
                            ibf_stream st);

/* stiffness_diagonal_max (intact/stepper.py:191-200). */
int ibf_stiffness_diagonal_max(ibf_system* s, const double* x, double h, double* out_host,
                               ibf_stream st);

/* solve_subproblem (intact/solver.py:178-233): Newton loop (cap 64, exit on a
 * full step or zero gradient), PCG, descent safeguard, NH cap, strict-decrease
 * backtracking, then one dual sweep.  x_hat: warm start in, result out.
 * result_host = (newton_iters, cg_iters, stalled, worst_violation). */
int ibf_solve_subproblem(ibf_system* s, ibf_contacts* c, const double* x_tilde,
                         const double* x, double* x_hat, double mu, double offset, double h,
                         double cg_tol, double decay, double* result_host, ibf_stream st);

/* The outer passes of Alg. 1 (intact/stepper.py:283-347) in native code:
 * per pass solve_subproblem, ActiveSet.update with the previous pass's
 * blocking pairs (none on the first pass), the NH inversion cap on x_hat - x
 * (p_scratch: 3n doubles, or null when no region is NH), max_step_size with
 * min_gap = 0.1 offset, clamp_state, the beta update from pass 1 on, and the
 * stagnation escape (mu x2, offset /2 after 50 passes with alpha < 1e-4);
 * stops when beta <= epsilon or after outer_cap passes.  x and x_hat are
 * updated in place.  records_host: outer_cap x 6 doubles per pass (alpha,
 * beta, constraints, newton iterations, CG iterations, wall ms).  out_host:
 * (passes, terminated, mu, offset, stagnation triggers, blocking pairs of the
 * last pass). */
int ibf_outer_loop(ibf_system* s, ibf_contacts* c, ibf_ccd* ccd, const double* x_tilde, double* x,
                   double* x_hat, double* p_scratch, double mu, double offset, double h, double cg_tol,
                   double decay, double epsilon, int min_iterations, int outer_cap, double* records_host,
                   double* out_host, ibf_stream st);

/* ------------------------------------------------------- step glue kernels */
/* x_tilde = x + h v + h^2 g (intact/stepper.py:263) */
int ibf_inertia_target(int64_t n, const double* x, const double* v, double h,
                       const double* gravity3_host, double* x_tilde, ibf_stream st);
/* clamp_state (intact/stepper.py:229-239), in place into x */
int ibf_clamp_state(int64_t n, double* x, const double* x_hat, double alpha, ibf_stream st);
/* out = a - b elementwise over n doubles (x_hat - x for the outer-pass cap,
 * intact/stepper.py:308) */
int ibf_vec_sub(int64_t n, const double* a, const double* b, double* out, ibf_stream st);
/* v = (x - x_t) / h (intact/stepper.py:225-226) */
int ibf_velocity_update(int64_t n, const double* x, const double* x_t, double h, double* v,
                        ibf_stream st);

/* ------------------------------------------- row-partitioned PCG (multi-GPU)
 * Replaces the single-process matvec / pcg_solve (intact/sparse.py:64-73,
 * :99-150) by a row partition over `world` partitions:
 * each holds the replicated operator, computes H p for its contiguous row
 * chunk, and per CG iteration allreduces pAp and (|r|^2, r.z) and allgathers
 * its z rows.  The reference has no counterpart (it is single-process). */
typedef struct ibf_dist ibf_dist;
/* NCCL unique id (128 bytes) for ibf_dist_create; rank 0 makes it and
 * broadcasts it (e.g. torch.distributed).  NCCL is loaded at run time
 * (libnccl.so.2, the one torch already loaded); IBF_ERR_CUDA without it. */
int ibf_dist_unique_id(void* out128);
/* One rank of a world-rank NCCL communicator on the current device. */
int ibf_dist_create(int rank, int world, const void* id128, ibf_dist** out);
/* All `parts` partitions in this process on the current device (exchanges
 * as device copies, reductions summed in partition order): the single-GPU
 * check of the partition arithmetic. */
int ibf_dist_create_local(int parts, ibf_dist** out);
void ibf_dist_destroy(ibf_dist* d);
/* Route the system's PCG solves (ibf_system_pcg, ibf_solve_subproblem) through
 * the partition (NULL: the single-GPU persistent kernel again). */
int ibf_system_set_dist(ibf_system* s, ibf_dist* d);

/* ---------------------------------------------- standalone sparse matrices */
typedef struct ibf_bsr ibf_bsr;
/* BlockSparseMatrix(n, rows, cols, blocks) (intact/sparse.py:49-62): coalesces
 * duplicate COO triplets; host inputs, blocks (nnz,3,3). */
int ibf_bsr_create(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                   const double* blocks, ibf_bsr** out);
void ibf_bsr_destroy(ibf_bsr* m);
int ibf_bsr_matvec(ibf_bsr* m, const double* x, double* y, ibf_stream st);
/* mask_dirichlet (intact/sparse.py:81-87): vertex_mask (n) host, diag (n,3,3) host */
int ibf_bsr_mask_dirichlet(ibf_bsr* m, const uint8_t* vertex_mask, const double* diag,
                           ibf_stream st);
/* coalesced block count and host copy (rows, cols, blocks (nb,3,3)) */
int64_t ibf_bsr_size(const ibf_bsr* m);
int ibf_bsr_export(const ibf_bsr* m, int64_t* rows, int64_t* cols, double* blocks, ibf_stream st);
int ibf_bsr_pcg(ibf_bsr* m, const double* rhs, double* x_out, double rel_tol,
                int64_t max_iters, double* info_host, ibf_stream st);

/* Launch-shape overrides for every subsequent PCG solve in the process
 * (tuning and tests; no reference counterpart — pcg_solve has no launch
 * shape, intact/sparse.py:99-150).  lanes_max_n: systems with at most this
 * many rows give each row 4 lanes of a warp (default 16384; < 0 restores the
 * default, 0 forces one thread per row).  max_ctas: cap on the cooperative
 * grid (0: a full co-resident wave), which raises the row sweeps per thread. */
int ibf_pcg_tuning(int64_t lanes_max_n, int max_ctas);
/* Shape of the last PCG launch in the process: out[0..5] = CTAs, threads per
 * CTA, row sweeps per thread, lanes per row, ready counter used (0/1),
 * matrix-free terms (contacts + friction). */
int ibf_pcg_last_shape(int64_t* out);

/* Algorithmic bytes of one symmetric SpMV over the elastic pattern
 * (BASELINE.md §4), for the bench's roofline line. */
int ibf_system_spmv_stats(const ibf_system* s, double* bytes_per_spmv);
/* Device-time phase counters since the last reset: out[0..8] = assembly ms,
 * assembly count, PCG ms, PCG launches, CG iterations, line-search energy ms,
 * energy launches, inversion-cap ms, sum over PCG launches of C x iterations. */
int ibf_system_stats(ibf_system* s, double* out, int reset);
/* Operation counts since the last reset: out[0] = Newton iterations of
 * ibf_solve_subproblem, out[1] = energy evaluations the reference's sequential
 * line search makes for the same iterations (base + trials up to the first
 * strict decrease, intact/solver.py:159-175) — the bench's CPU cost model. */
int ibf_system_counts(ibf_system* s, double* out, int reset);
/* CCD phase: out[0..2] = max_step_size device ms, calls, broad-phase candidates. */
int ibf_ccd_stats(ibf_ccd* c, double* out, int reset);
/* Per-kernel device clocks (roofline bookkeeping; no reference counterpart).
 * on: 1 starts bracketing the instrumented launches with events on their
 * stream, 0 stops, < 0 leaves the state.  out (may be NULL) receives 8 rows
 * of 5 doubles — ms, launches, algorithmic bytes, algorithmic flops, units —
 * for k_elem, k_gather_blocks, k_vertex_rows, k_energy, k_traverse,
 * k_pair_toi, k_pcg, k_prefilter (units: tets, blocks, vertices, trial
 * points, candidate pairs, narrow-phase pairs, -, candidate pairs); pending
 * events are harvested first (waits
 * for them).  reset != 0 zeroes the counters after reading. */
int ibf_kernel_clocks(int on, double* out, int reset);

/* Number of kernels libibf has launched in this process (CUB internals excluded). */
unsigned long long ibf_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* IBF_H */
