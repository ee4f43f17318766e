// The elastic system handle (System + ElasticRegion list) and the contact
// hooks the assembly needs.
#pragma once

#include "internal.cuh"

struct ibf_system {
  int64_t n = 0;        // vertices
  int64_t m = 0;        // tets
  int64_t n_tiles = 0;  // ceil(m / 32)
  int n_regions = 0;
  bool has_nh = false;
  std::vector<ibf::RegionDev> regions_host;
  ibf::DevBuf<ibf::RegionDev> regions;
  ibf::DevBuf<int> tets;                 // (m,4) int32
  ibf::DevBuf<double> shape_rows;        // (m,4,3)
  ibf::DevBuf<double> volumes;           // (m)
  ibf::DevBuf<double> masses;            // (n)
  ibf::DevBuf<uint8_t> dbc;              // (n)
  bool any_dbc = false;
  // static symmetric BSR pattern (diagonal + strict upper) in sliced-ELL
  // storage; pat.val holds the assembled matrix
  ibf::SellPattern pat;
  ibf::DevBuf<int> blk_ptr, blk_src;     // storage block <- (tet*10+q) contributions, tet order
  ibf::DevBuf<int> vt_ptr, vt_src;       // vertex <- (tet*4+l) incidences, tet order
  // assembled state
  ibf::DevBuf<double> pinv;              // (n,9)
  ibf::DevBuf<double> elem_grad, elem_blk;  // tile-32 layouts
  ibf::DevBuf<int> flags;                // [0] nonfinite energy, [1] gradient nonzero
  ibf::DevBuf<double> dscal;             // device scalars
  ibf::DevBuf<double> epart;             // energy partials
  ibf::DevBuf<double> vec_a, vec_b, vec_c;   // (n,3) scratch
  ibf::HostScratch host;
  ibf::PcgWork work;
  ibf_dist* dist = nullptr;      // row partition of the PCG (ibf_system_set_dist), or none
  ibf::DistWork dwork;
  // phase timers (device time): assembly, PCG, line-search energies, inversion cap
  ibf::PhaseTimer t_asm, t_pcg, t_ls, t_cap;
  long long pcg_iters = 0;       // CG iterations since the last stats reset
  long long contact_terms = 0;   // sum over PCG launches of C (matrix-free contact)
  long long ref_energy_evals = 0;  // energy evaluations the reference's sequential line search makes
  long long newton_iters = 0;      // Newton iterations since the last stats reset
  ibf_contacts* assembled_contacts = nullptr;  // contact term of the last assembly
  ibf_friction* friction = nullptr;            // frozen friction terms (ibf_system_set_friction)
  bool assembled_friction = false;
  bool assembled_dbc = false;
  ibf::Operator op() const;
};

namespace ibf {
// contact.cu
int contact_prepare(ibf_contacts* c, const double* x_hat, double mu, double offset, cudaStream_t s);
int contact_build_incidence(ibf_contacts* c, int64_t n_verts, cudaStream_t s);
ContactView contact_view(ibf_contacts* c);
// per-row PCG term records of the unmasked rows (mask: the assembled DBC mask or null)
int contact_pack_terms(ibf_contacts* c, int64_t n_verts, const uint8_t* mask, cudaStream_t s);

// friction.cu
int friction_build_incidence(ibf_friction* f, int64_t n_verts, cudaStream_t s);
int friction_prepare(ibf_friction* f, const double* x_hat, cudaStream_t s);
FrictionView friction_view(ibf_friction* f);

// system.cu
int system_assemble(ibf_system* s, ibf_contacts* c, const double* x_hat, const double* x_tilde, double mu,
                    double offset, double h, bool apply_dbc, double* grad, bool contacts_ready,
                    cudaStream_t st);
int system_energy_launch(ibf_system* s, ibf_contacts* c, const double* x_hat, const double* p, int n_r,
                         const double* r_host, const double* r0_dev, const double* x_tilde, double mu,
                         double offset, double h, double* out_dev, cudaStream_t st);
int system_inversion_cap_launch(ibf_system* s, const double* x, const double* p, double* out_dev,
                                cudaStream_t st);
// the system's PCG: the persistent single-GPU kernel, or the row partition
int system_pcg(ibf_system* s, const double* rhs, double* x, double rel_tol, int64_t max_iters, cudaStream_t st);
}  // namespace ibf
