// The AL subproblem's Newton loop and the time-step glue kernels, plus the
// library's infrastructure entry points.
//
// Replaces (paths relative to /root/reference/pkg/src):
//   solve_subproblem    intact/solver.py:178-233
//   line_search         intact/solver.py:159-175
//   x_tilde / clamp_state / velocity_update
//                       intact/stepper.py:263, :229-239, :225-226
//
// Host synchronisation: one device->host read per Newton iteration (PCG
// count, trial energy, step cap and flags arrive together).  The PCG runs as
// one persistent kernel; the inversion cap feeds the line search's first
// trial on the device; the base energy of iteration k+1 is the accepted trial
// energy of iteration k (bit-identical to re-evaluating it, since x_hat + r p
// is formed the same way in both places).
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <ctime>
#include <string>

#include "system.cuh"

namespace ibf {

std::atomic<unsigned long long> g_launches{0};

static int trace_level() {
  static int lvl = -1;
  if (lvl < 0) lvl = getenv("IBF_TRACE") ? atoi(getenv("IBF_TRACE")) : 0;
  return lvl;
}
bool trace_enabled() { return trace_level() > 0; }
bool alloc_log() {
  static int on = -1;
  if (on < 0) on = getenv("IBF_ALLOC_LOG") ? atoi(getenv("IBF_ALLOC_LOG")) : 0;
  return on > 0;
}
double wall_now() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}
int dev_alloc(void** p, size_t bytes) {
  static std::atomic<unsigned> pools_ready{0};   // bit per device
  int dev = 0;
  IBF_CUDA(cudaGetDevice(&dev));
  if (dev < 32 && !(pools_ready.load() & (1u << dev))) {
    cudaMemPool_t pool;
    IBF_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    IBF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    // Prime the pool: map one large block up front and return it, so buffer
    // growth mid-press is carved from memory the pool already holds.  Growth
    // that had to map new memory stalled single passes by 0.1-0.7 s on the
    // squishy press (bench "slowest_pass_wall_ms").  IBF_POOL_PRIME_GB
    // overrides the size (default: 20 % of free memory, at most 24 GB).
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      size_t prime = std::min<size_t>(free_b / 5, (size_t)24 << 30);
      if (const char* e = getenv("IBF_POOL_PRIME_GB")) prime = (size_t)(atof(e) * (double)(1ull << 30));
      void* q = nullptr;
      if (prime && cudaMallocAsync(&q, prime, 0) == cudaSuccess) {
        cudaFreeAsync(q, 0);
        cudaStreamSynchronize(0);
      }
      cudaGetLastError();
    }
    pools_ready.fetch_or(1u << dev);
  }
  const cudaStream_t s = tl_stream;
  IBF_CUDA(cudaMallocAsync(p, bytes, s));
  // legacy default stream: ordered after prior work on blocking streams; the
  // sync makes the block usable from any (non-blocking) stream at once
  if (!s) IBF_CUDA(cudaStreamSynchronize(0));
  return IBF_OK;
}

void dev_free(void* p) {
  const cudaStream_t s = tl_stream;
  // outside a stream-scoped call the old buffer may still be read by queued
  // kernels on any stream
  if (!s) cudaDeviceSynchronize();
  cudaFreeAsync(p, s);
}

thread_local cudaStream_t tl_stream = 0;

// ------------------------------------------------------- per-kernel clocks
std::atomic<bool> g_kclock_on{false};
namespace {
struct KcPending {
  cudaEvent_t b, e;
  double bytes, flops, units;
};
struct KcTable {
  std::mutex m;
  std::vector<cudaEvent_t> pool;
  std::vector<KcPending> pending[KC_COUNT];
  double ms[KC_COUNT] = {}, bytes[KC_COUNT] = {}, flops[KC_COUNT] = {}, units[KC_COUNT] = {};
  long long launches[KC_COUNT] = {};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void harvest(bool wait) {
    for (int k = 0; k < KC_COUNT; ++k) {
      auto& v = pending[k];
      size_t keep = 0;
      for (size_t j = 0; j < v.size(); ++j) {
        KcPending& q = v[j];
        if (!wait && cudaEventQuery(q.e) != cudaSuccess) {
          v[keep++] = q;
          continue;
        }
        cudaEventSynchronize(q.e);
        float t = 0.0f;
        if (cudaEventElapsedTime(&t, q.b, q.e) == cudaSuccess) {
          ms[k] += t;
          bytes[k] += q.bytes;
          flops[k] += q.flops;
          units[k] += q.units;
          ++launches[k];
        }
        pool.push_back(q.b);
        pool.push_back(q.e);
      }
      v.resize(keep);
    }
    cudaGetLastError();
  }
};
KcTable& kc_table() {
  static KcTable t;
  return t;
}
}  // namespace

KernelClock::KernelClock(int id_, cudaStream_t s_, double bytes_, double flops_, double units_)
    : id(id_), s(s_), bytes(bytes_), flops(flops_), units(units_) {
  if (!g_kclock_on.load(std::memory_order_relaxed)) return;
  KcTable& t = kc_table();
  std::lock_guard<std::mutex> lk(t.m);
  b = t.get();
  cudaEventRecord(b, s);
}

KernelClock::~KernelClock() {
  if (!b) return;
  KcTable& t = kc_table();
  std::lock_guard<std::mutex> lk(t.m);
  cudaEvent_t e = t.get();
  cudaEventRecord(e, s);
  t.pending[id].push_back({b, e, bytes, flops, units});
  if (t.pending[id].size() > 512) t.harvest(false);
}

void alloc_report(const char* what, size_t bytes, double t0) {
  const double ms = 1e3 * (wall_now() - t0);
  if (ms > 1.0) fprintf(stderr, "[ibf] slow %s: %.1f ms for %zu bytes\n", what, ms, bytes);
}
static double now_s() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}
Trace::Trace(const char* name) : on(trace_enabled()), last(0.0) {
  if (on) {
    last = now_s();
    out = name;
  }
}
void Trace::mark(const char* what, cudaStream_t s, long long v) {
  // level 1: only the first and last marks of a call (no extra syncs inside)
  if (!on || (trace_level() < 2 && strcmp(what, "enter") != 0 && strcmp(what, "exit") != 0)) return;
  cudaStreamSynchronize(s);
  const double t = now_s();
  char b[96];
  if (v >= 0) snprintf(b, sizeof b, " %s=%.3fms(%lld)", what, 1e3 * (t - last), v);
  else snprintf(b, sizeof b, " %s=%.3fms", what, 1e3 * (t - last));
  out += b;
  last = t;
}
Trace::~Trace() {
  if (on) fprintf(stderr, "[ibf] %s\n", out.c_str());
}
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

int sm_count() {
  static int n = -1;
  if (n < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

__global__ void k_neg(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = -a[i];
}

// out = sum a*b (fixed order: per-block partials, then one warp)
__global__ void k_dot_part(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ part) {
  __shared__ double red[8];
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v += a[i] * b[i];
  v = block_sum(v, red);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// descent safeguard (intact/solver.py:216-220): if g.p >= 0, p = -P^-1 g
__global__ void k_descent_fix(int64_t n, const double* __restrict__ part, int nparts, const double* __restrict__ g,
                              const double* __restrict__ pinv, double* __restrict__ p) {
  __shared__ double tot;
  if (threadIdx.x < 32) {
    const double v = warp_sum_array(part, nparts);
    if (threadIdx.x == 0) tot = v;
  }
  __syncthreads();
  if (!(tot >= 0.0)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double zv[3];
    apply_pinv6(pinv + PINV_STRIDE * i, g[3 * i], g[3 * i + 1], g[3 * i + 2], zv);
    p[3 * i] = -zv[0];
    p[3 * i + 1] = -zv[1];
    p[3 * i + 2] = -zv[2];
  }
}

__global__ void k_first_step(const double* __restrict__ cap, double* __restrict__ r0) { *r0 = fmin(1.0, *cap); }

// x <- x + r p exactly as numpy forms x_hat + r * p
__global__ void k_step(int64_t n, double r, const double* __restrict__ p, double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __dadd_rn(x[i], __dmul_rn(r, p[i]));
}

__global__ void k_inertia(int64_t n, const double* __restrict__ x, const double* __restrict__ v, double h, double gx,
                          double gy, double gz, double* __restrict__ xt) {
  const double h2 = __dmul_rn(h, h);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % 3);
    const double g = c == 0 ? gx : (c == 1 ? gy : gz);
    xt[i] = __dadd_rn(__dadd_rn(x[i], __dmul_rn(h, v[i])), __dmul_rn(h2, g));
  }
}

__global__ void k_clamp(int64_t n, double alpha, double* __restrict__ x, const double* __restrict__ xh) {
  const double om = __dsub_rn(1.0, alpha);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = x[i], b = xh[i];
    if (alpha >= 1.0) {
      x[i] = b;
    } else if (!(a == b)) {
      x[i] = __dadd_rn(__dmul_rn(om, a), __dmul_rn(alpha, b));
    }
  }
}

__global__ void k_velocity(int64_t n, const double* __restrict__ x, const double* __restrict__ xt, double h,
                           double* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = __dsub_rn(x[i], xt[i]) / h;
}

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(div_up(n, 256), 148LL * 8)); }

int contacts_refresh(ibf_contacts* c, const double* x, int* degen_dev, cudaStream_t s);
int contacts_dual(ibf_contacts* c, const double* x_hat, double offset, double mu, double decay, double* worst_dev,
                  cudaStream_t s);

}  // namespace ibf

using namespace ibf;

extern "C" int ibf_kernel_clocks(int on, double* out, int reset) {
  KcTable& t = kc_table();
  std::lock_guard<std::mutex> lk(t.m);
  t.harvest(true);
  if (out)
    for (int k = 0; k < KC_COUNT; ++k) {
      out[5 * k + 0] = t.ms[k];
      out[5 * k + 1] = (double)t.launches[k];
      out[5 * k + 2] = t.bytes[k];
      out[5 * k + 3] = t.flops[k];
      out[5 * k + 4] = t.units[k];
    }
  if (reset)
    for (int k = 0; k < KC_COUNT; ++k) {
      t.ms[k] = t.bytes[k] = t.flops[k] = t.units[k] = 0.0;
      t.launches[k] = 0;
    }
  if (on >= 0) g_kclock_on.store(on != 0);
  return IBF_OK;
}

extern "C" const char* ibf_version(void) { return "ibf-b200 0.1 (sm_100a)"; }
extern "C" const char* ibf_last_error(void) { return g_err.c_str(); }

extern "C" int ibf_inertia_target(int64_t n, const double* x, const double* v, double h, const double* g3,
                                  double* x_tilde, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  if (n <= 0) return IBF_OK;
  k_inertia<<<grid_for(3 * n), 256, 0, (cudaStream_t)st>>>(3 * n, x, v, h, g3[0], g3[1], g3[2], x_tilde);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

extern "C" int ibf_clamp_state(int64_t n, double* x, const double* x_hat, double alpha, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  if (n <= 0) return IBF_OK;
  k_clamp<<<grid_for(3 * n), 256, 0, (cudaStream_t)st>>>(3 * n, alpha, x, x_hat);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

extern "C" int ibf_velocity_update(int64_t n, const double* x, const double* x_t, double h, double* v, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  if (n <= 0) return IBF_OK;
  k_velocity<<<grid_for(3 * n), 256, 0, (cudaStream_t)st>>>(3 * n, x, x_t, h, v);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

extern "C" int ibf_system_spmv_stats(const ibf_system* s, double* bytes_per_spmv) {
  // algorithmic bytes of one symmetric SpMV:
  // 72 (N + E_u) + 4 E_u + 4 (N + 1) + 24 N + 24 N
  const double N = (double)s->n, Eu = (double)s->pat.nl;
  *bytes_per_spmv = 72.0 * (N + Eu) + 4.0 * Eu + 4.0 * (N + 1.0) + 48.0 * N;
  return IBF_OK;
}

extern "C" int ibf_solve_subproblem(ibf_system* s, ibf_contacts* c, const double* x_tilde, const double* x,
                                    double* x_hat, double mu, double offset, double h, double cg_tol, double decay,
                                    double* result_host, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t stream = (cudaStream_t)st;
  const int64_t n = s->n;
  const int64_t n3 = 3 * n;
  double* grad = s->vec_a.p;
  double* p = s->vec_b.p;
  double* rhs = s->vec_c.p;
  // device scalars: [0..7] energies, [8] cap, [9] r0, [10] worst, [16..] dot partials
  double* E = s->dscal.p;
  double* cap = s->dscal.p + 8;
  double* r0 = s->dscal.p + 9;
  double* worst = s->dscal.p + 10;
  const int dot_parts = 64;
  IBF_TRY(s->dscal.reserve(16 + dot_parts + 8));
  E = s->dscal.p;
  cap = E + 8;
  r0 = E + 9;
  worst = E + 10;
  double* dpart = E + 16;
  IBF_TRY(s->host.reserve(256));
  double* hd = (double*)s->host.p;      // hd[0..7] energies, hd[8] r0, hd[9..11] pcg info
  int* hi = (int*)(hd + 16);            // hi[0] nonfinite, hi[1] grad nonzero
  ibf_contacts* cc = (c && c->n) ? c : nullptr;
  Trace tr("solve_subproblem");
  tr.mark("enter", stream, cc ? cc->n : 0);
  if (cc) {
    IBF_TRY(c->iscratch.reserve(2));
    IBF_CUDA(cudaMemsetAsync(c->iscratch.p, 0, sizeof(int), stream));
    IBF_TRY(contacts_refresh(c, x, c->iscratch.p, stream));
    IBF_TRY(contact_build_incidence(c, n, stream));
  }
  tr.mark("refresh+incidence", stream);
  int newton = 0;
  int64_t cg_total = 0;
  bool stalled = false;
  bool have_base = false;
  double base = 0.0;
  bool capped = true;
  for (int it = 0; it < 64; ++it) {
    s->t_asm.begin(stream);
    IBF_TRY(system_assemble(s, cc, x_hat, x_tilde, mu, offset, h, true, grad, true, stream));
    s->t_asm.end(stream);
    tr.mark("assemble", stream);
    k_neg<<<grid_for(n3), 256, 0, stream>>>(n3, grad, rhs);
    IBF_LAUNCH_CHECK();
    s->t_pcg.begin(stream);
    IBF_TRY(system_pcg(s, rhs, p, cg_tol, 10 * n, stream));
    s->t_pcg.end(stream);
    tr.mark("pcg", stream);
    k_dot_part<<<dot_parts, 256, 0, stream>>>(n3, grad, p, dpart);
    IBF_LAUNCH_CHECK();
    k_descent_fix<<<grid_for(n), 256, 0, stream>>>(n, dpart, dot_parts, grad, s->pinv.p, p);
    IBF_LAUNCH_CHECK();
    s->t_cap.begin(stream);
    IBF_TRY(system_inversion_cap_launch(s, x_hat, p, cap, stream));
    s->t_cap.end(stream);
    k_first_step<<<1, 1, 0, stream>>>(cap, r0);
    IBF_LAUNCH_CHECK();
    const double rs_first[2] = {1.0, 0.0};
    const int T = have_base ? 1 : 2;  // second trial at r = 0 is the base energy
    s->t_ls.begin(stream);
    IBF_TRY(system_energy_launch(s, cc, x_hat, p, T, rs_first, r0, x_tilde, mu, offset, h, E, stream));
    s->t_ls.end(stream);
    IBF_CUDA(cudaMemcpyAsync(hd, E, 2 * sizeof(double), cudaMemcpyDeviceToHost, stream));
    IBF_CUDA(cudaMemcpyAsync(hd + 8, r0, sizeof(double), cudaMemcpyDeviceToHost, stream));
    IBF_CUDA(cudaMemcpyAsync(hd + 9, s->work.info.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, stream));
    IBF_CUDA(cudaMemcpyAsync(hi, s->flags.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream));
    IBF_CUDA(cudaStreamSynchronize(stream));
    tr.mark("safeguard+cap+energy+sync", stream);
    if (hi[0]) {
      set_error("elastic energy is not finite at the evaluation point");
      return IBF_ERR_NONFINITE;
    }
    if (!hi[1]) {  // not np.any(grad)
      capped = false;
      break;
    }
    cg_total += (int64_t)hd[9];
    s->t_asm.harvest();
    s->t_pcg.harvest();
    s->t_ls.harvest();
    s->t_cap.harvest();
    s->pcg_iters += (long long)hd[9];
    s->contact_terms += (cc ? cc->n : 0) * (long long)hd[9];  // C x CG iterations
    if (!have_base) base = hd[1];
    const double rfirst = hd[8];
    double r = rfirst, e_acc = hd[0];
    bool stall = false;
    // the reference evaluates the base energy and then trials r0, r0/2, ...
    // until the first strict decrease (intact/solver.py:159-175)
    long long ref_trials = 1;
    if (!(hd[0] < base)) {
      // backtracking: r0 / 2^k, k = 1..30, strict decrease (intact/solver.py:159-175)
      double best_r = rfirst, best_e = INFINITY;
      if (hd[0] < best_e) {
        best_r = rfirst;
        best_e = hd[0];
      }
      bool found = false;
      int k = 1;
      while (k <= 30 && !found) {
        const int T2 = std::min(8, 31 - k);
        double rs[8];
        double sc = 1.0;
        for (int j = 0; j < k; ++j) sc *= 0.5;
        for (int j = 0; j < T2; ++j) {
          rs[j] = sc;
          sc *= 0.5;
        }
        s->t_ls.begin(stream);
        IBF_TRY(system_energy_launch(s, cc, x_hat, p, T2, rs, r0, x_tilde, mu, offset, h, E, stream));
        s->t_ls.end(stream);
        IBF_CUDA(cudaMemcpyAsync(hd, E, T2 * sizeof(double), cudaMemcpyDeviceToHost, stream));
        IBF_CUDA(cudaStreamSynchronize(stream));
        s->t_ls.harvest();
        for (int j = 0; j < T2; ++j) {
          const double rj = rfirst * rs[j];
          ++ref_trials;
          if (hd[j] < base) {
            r = rj;
            e_acc = hd[j];
            found = true;
            break;
          }
          if (hd[j] < best_e) {
            best_r = rj;
            best_e = hd[j];
          }
        }
        k += T2;
      }
      if (!found) {
        r = best_r;
        e_acc = best_e;
        stall = true;
      }
    }
    k_step<<<grid_for(n3), 256, 0, stream>>>(n3, r, p, x_hat);
    IBF_LAUNCH_CHECK();
    s->ref_energy_evals += 1 + ref_trials;
    ++s->newton_iters;
    base = e_acc;
    have_base = e_acc < INFINITY;  // stalled on all-inf trials: recompute next time
    ++newton;
    stalled = stalled || stall;
    if (r == 1.0) {
      capped = false;
      break;
    }
  }
  if (capped) stalled = true;
  tr.mark("linesearch+step", stream);
  double w = 0.0;
  if (cc) {
    IBF_TRY(contacts_dual(c, x_hat, offset, mu, decay, worst, stream));
    IBF_CUDA(cudaMemcpyAsync(hd, worst, sizeof(double), cudaMemcpyDeviceToHost, stream));
    IBF_CUDA(cudaStreamSynchronize(stream));
    w = hd[0];
  }
  tr.mark("dual", stream);
  tr.mark("exit", stream);
  result_host[0] = newton;
  result_host[1] = (double)cg_total;
  result_host[2] = stalled ? 1.0 : 0.0;
  result_host[3] = w;
  return IBF_OK;
}

namespace ibf {
__global__ void k_sub(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ o) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = __dsub_rn(a[i], b[i]);
}
}  // namespace ibf

// Alg. 1's outer passes (stepper._outer_loop, intact/stepper.py:283-347):
// the same calls in the same order, the scalar logic in C++, so a pass costs
// no Python round trips.  The scalar helpers mirror beta_update,
// stagnation_advance and adaptive_mu (intact/stepper.py:178-213).
extern "C" int ibf_outer_loop(ibf_system* s, ibf_contacts* c, ibf_ccd* ccd, const double* x_tilde, double* x,
                              double* x_hat, double* p_scratch, double mu, double offset, double h, double cg_tol,
                              double decay, double epsilon, int min_iterations, int outer_cap, double* records_host,
                              double* out_host, ibf_stream st) {
  if (!s || !c || !ccd || !x_tilde || !x || !x_hat || !records_host || !out_host || outer_cap < 0) {
    set_error("ibf_outer_loop: bad arguments");
    return IBF_ERR_BAD_ARG;
  }
  const int64_t n = s->n;
  constexpr double kStagnationAlpha = 1e-4;   // stepper.STAGNATION_ALPHA
  constexpr int kStagnationLimit = 50;         // stepper.STAGNATION_LIMIT
  constexpr double kGapFraction = 0.1;         // stepper.CCD_GAP_FRACTION
  double beta = 1.0;
  int counter = 0, triggers = 0, passes = 0;
  int64_t last_block = 0;
  bool have_blocking = false, terminated = false;
  for (int k = 0; k < outer_cap; ++k) {
    const double t0 = wall_now();
    double res[4];
    IBF_TRY(ibf_solve_subproblem(s, c, x_tilde, x, x_hat, mu, offset, h, cg_tol, decay, res, st));
    int64_t adm = 0, pr = 0;
    if (have_blocking)
      IBF_TRY(ibf_contacts_update(c, ccd, &adm, &pr, st));
    else
      IBF_TRY(ibf_contacts_update_host(c, 0, nullptr, nullptr, nullptr, &adm, &pr, st));
    double cap = 1.0;
    if (p_scratch) {
      IBF_TRY(ibf_vec_sub(3 * n, x_hat, x, p_scratch, st));
      double a_nh = 1.0;
      IBF_TRY(ibf_inversion_safe_step(s, x, p_scratch, &a_nh, st));
      cap = std::min(cap, a_nh);
    }
    double alpha = 0.0;
    int64_t n_block = 0;
    IBF_TRY(ibf_max_step_size(ccd, x, x_hat, kGapFraction * offset, cap, &alpha, &n_block, st));
    last_block = n_block;
    have_blocking = true;
    IBF_TRY(ibf_clamp_state(n, x, x_hat, alpha, st));
    if ((k - 1) + 1 >= min_iterations) beta = (1.0 - alpha) * beta;
    double* r = records_host + 6 * (size_t)k;
    r[0] = alpha;
    r[1] = beta;
    r[2] = (double)ibf_contacts_size(c);
    r[3] = res[0];
    r[4] = res[1];
    r[5] = (wall_now() - t0) * 1e3;
    passes = k + 1;
    counter = alpha < kStagnationAlpha ? counter + 1 : 0;
    if (counter >= kStagnationLimit) {
      mu = 2.0 * mu;
      offset = 0.5 * offset;
      counter = 0;
      ++triggers;
    }
    if (beta <= epsilon) {
      terminated = true;
      break;
    }
  }
  out_host[0] = passes;
  out_host[1] = terminated ? 1.0 : 0.0;
  out_host[2] = mu;
  out_host[3] = offset;
  out_host[4] = triggers;
  out_host[5] = (double)last_block;
  return IBF_OK;
}

extern "C" int ibf_vec_sub(int64_t n, const double* a, const double* b, double* out, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  if (n <= 0) return IBF_OK;
  ibf::k_sub<<<ibf::grid_for(n), 256, 0, (cudaStream_t)st>>>(n, a, b, out);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

extern "C" unsigned long long ibf_launch_count(void) { return ibf::g_launches.load(); }

extern "C" int ibf_system_stats(ibf_system* s, double* out, int reset) {
  s->t_asm.harvest();
  s->t_pcg.harvest();
  s->t_ls.harvest();
  s->t_cap.harvest();
  out[0] = s->t_asm.ms;
  out[1] = (double)s->t_asm.count;
  out[2] = s->t_pcg.ms;
  out[3] = (double)s->t_pcg.count;
  out[4] = (double)s->pcg_iters;
  out[5] = s->t_ls.ms;
  out[6] = (double)s->t_ls.count;
  out[7] = s->t_cap.ms;
  out[8] = (double)s->contact_terms;
  if (reset) {
    s->t_asm.reset();
    s->t_pcg.reset();
    s->t_ls.reset();
    s->t_cap.reset();
    s->pcg_iters = 0;
    s->contact_terms = 0;
  }
  return IBF_OK;
}

extern "C" int ibf_system_counts(ibf_system* s, double* out, int reset) {
  out[0] = (double)s->newton_iters;
  out[1] = (double)s->ref_energy_evals;
  if (reset) s->newton_iters = s->ref_energy_evals = 0;
  return IBF_OK;
}

extern "C" int ibf_ccd_stats(ibf_ccd* c, double* out, int reset) {
  c->t_ccd.harvest();
  out[0] = c->t_ccd.ms;
  out[1] = (double)c->t_ccd.count;
  out[2] = (double)c->n_candidates;
  if (reset) {
    c->t_ccd.reset();
    c->n_candidates = 0;
  }
  return IBF_OK;
}
