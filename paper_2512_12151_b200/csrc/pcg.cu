// Symmetric 3x3-block SpMV and the device-resident block-Jacobi PCG.
//
// Replaces BlockSparseMatrix.matvec and pcg_solve (intact/sparse.py:64-73,
// :99-150; paths relative to /root/reference/pkg/src).
//
// Storage is the reference's: diagonal + strict-upper 3x3 blocks only.  The
// lower triangle is applied by a transpose index (row i lists the upper
// blocks b with col(b) = i), so every row's result is a fixed-order gather —
// no atomics, bit-reproducible run to run.  A block's second (transposed)
// read is an L2 hit because rows are processed roughly in order and the
// matrix bandwidth is small, so DRAM traffic stays ~1x the upper storage.
//
// The whole PCG (all iterations, the reference's stopping rule, best-iterate
// tracking, the 250-iteration restart, pAp <= 0 bail-out) runs in ONE
// persistent cooperative kernel: one CTA per SM slot, grid-wide barriers
// between phases, deterministic two-level reductions.  The host launches it
// once per linear solve and reads (iterations, converged, rel_res) back.
#include <cooperative_groups.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace ibf {

constexpr int PCG_THREADS = 256;

// ---------------------------------------------------------------- SpMV pieces

// t_c = coef_c * sum_slot g_c[slot] . p[v(slot)], masked columns excluded.
__device__ __forceinline__ void contact_dot(const Operator& op, const double* __restrict__ p, int c) {
  const ContactView& cv = op.contact;
  const int* q = cv.quad + 4 * c;
  const double* g = cv.grad + 12 * c;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int v = q[k];
    if (op.mask && op.mask[v]) continue;
    acc += g[3 * k] * p[3 * v] + g[3 * k + 1] * p[3 * v + 1] + g[3 * k + 2] * p[3 * v + 2];
  }
  cv.t[c] = cv.coef[c] * acc;
}

// 9 doubles of block b with 16-byte loads: val is a library allocation
// (256B-aligned), so 72b bytes is 16B-aligned exactly for even b.
template <bool NC>
__device__ __forceinline__ void load_block(const double* __restrict__ val, int b, double B[9]) {
  const double* src = val + 9 * (size_t)b;
  if ((b & 1) == 0) {
    const double2* v2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 t = NC ? __ldg(v2 + k) : v2[k];
      B[2 * k] = t.x;
      B[2 * k + 1] = t.y;
    }
    B[8] = NC ? __ldg(src + 8) : src[8];
  } else {
    B[0] = NC ? __ldg(src) : src[0];
    const double2* v2 = reinterpret_cast<const double2*>(src + 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 t = NC ? __ldg(v2 + k) : v2[k];
      B[1 + 2 * k] = t.x;
      B[2 + 2 * k] = t.y;
    }
  }
}

// p_j: caller-owned vectors carry no alignment promise beyond 8 bytes, so
// the gather stays scalar (these reads are L1/L2 hits).
__device__ __forceinline__ void load_vec3(const double* __restrict__ p, int j, double v[3]) {
  const double* src = p + 3 * (size_t)j;
  v[0] = src[0];
  v[1] = src[1];
  v[2] = src[2];
}

// (H p)_i[r] for one row and component (three threads per row): upper
// blocks, transposed lower blocks via the transpose index, then the
// matrix-free contact gather.  Block values are read-only for the whole
// solve (non-coherent loads are safe); p is rewritten between phases of the
// persistent kernel, so it is loaded coherently.
__device__ __forceinline__ double row_product(const Operator& op, const double* __restrict__ p, int i, int r) {
  double acc = 0.0;
  const int b0 = op.row_ptr[i], b1 = op.row_ptr[i + 1];
  for (int b = b0; b < b1; ++b) {
    const int j = __ldg(op.col + b);
    const double* B = op.val + 9 * (size_t)b + 3 * r;
    acc += __ldg(B) * p[3 * j] + __ldg(B + 1) * p[3 * j + 1] + __ldg(B + 2) * p[3 * j + 2];
  }
  const int l0 = op.low_ptr[i], l1 = op.low_ptr[i + 1];
  for (int e = l0; e < l1; ++e) {
    const int2 bk = __ldg(op.low_pair + e);
    const double* B = op.val + 9 * (size_t)bk.x + r;
    const int k = bk.y;
    acc += __ldg(B) * p[3 * k] + __ldg(B + 3) * p[3 * k + 1] + __ldg(B + 6) * p[3 * k + 2];
  }
  if (op.contact.n && !(op.mask && op.mask[i])) {
    const ContactView& cv = op.contact;
    const int e0 = cv.vc_ptr[i], e1 = cv.vc_ptr[i + 1];
    for (int e = e0; e < e1; ++e) {
      const int src = cv.vc_src[e];
      const int c = src >> 2, slot = src & 3;
      acc += cv.t[c] * cv.grad[12 * c + 3 * slot + r];
    }
  }
  return acc;
}

__global__ void k_contact_dot(Operator op, const double* __restrict__ p) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < op.contact.n; c += gridDim.x * blockDim.x)
    contact_dot(op, p, c);
}

__global__ void k_spmv(Operator op, const double* __restrict__ p, double* __restrict__ y) {
  const int64_t n3 = 3LL * op.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n3; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / 3), r = (int)(t - 3LL * i);
    y[t] = row_product(op, p, i, r);
  }
}

int spmv(const Operator& op, const double* x, double* y, cudaStream_t s) {
  if (op.n == 0) return IBF_OK;
  if (op.contact.n) {
    k_contact_dot<<<(int)div_up(op.contact.n, 256), 256, 0, s>>>(op, x);
    IBF_LAUNCH_CHECK();
  }
  const int grid = (int)std::min<int64_t>(div_up(3LL * op.n, 256), 148LL * 16);
  k_spmv<<<grid, 256, 0, s>>>(op, x, y);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

// ----------------------------------------------------------- 3x3 inverses

__device__ __forceinline__ void inv3(const double* A, double* O) {
  const double c00 = A[4] * A[8] - A[5] * A[7];
  const double c01 = A[5] * A[6] - A[3] * A[8];
  const double c02 = A[3] * A[7] - A[4] * A[6];
  const double det = A[0] * c00 + A[1] * c01 + A[2] * c02;
  const double id = 1.0 / det;
  O[0] = c00 * id;
  O[1] = (A[2] * A[7] - A[1] * A[8]) * id;
  O[2] = (A[1] * A[5] - A[2] * A[4]) * id;
  O[3] = c01 * id;
  O[4] = (A[0] * A[8] - A[2] * A[6]) * id;
  O[5] = (A[2] * A[3] - A[0] * A[5]) * id;
  O[6] = c02 * id;
  O[7] = (A[1] * A[6] - A[0] * A[7]) * id;
  O[8] = (A[0] * A[4] - A[1] * A[3]) * id;
}

__global__ void k_invert_diag(int n, const double* __restrict__ val, const int* __restrict__ diag_blk,
                              double* __restrict__ pinv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double A[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const int b = diag_blk[i];
    if (b >= 0)
      for (int k = 0; k < 9; ++k) A[k] = val[9 * (size_t)b + k];
    inv3(A, pinv + 9 * (size_t)i);
  }
}

int invert_diag_blocks(int n, const double* val, const int* diag_blk, double* pinv, cudaStream_t s) {
  if (n == 0) return IBF_OK;
  k_invert_diag<<<(int)div_up(n, 256), 256, 0, s>>>(n, val, diag_blk, pinv);
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
  double* p;
  double* hp;
  double* X;        // 3 iterate buffers of 3n
  double* part;     // 4 * gridDim partial sums
  double* info;     // (iterations, converged, rel_res)
  double tol;
  int64_t max_iters;
};

__device__ __forceinline__ void apply_pinv(const double* __restrict__ P, const double r[3], double z[3]) {
  z[0] = P[0] * r[0] + P[1] * r[1] + P[2] * r[2];
  z[1] = P[3] * r[0] + P[4] * r[1] + P[5] * r[2];
  z[2] = P[6] * r[0] + P[7] * r[1] + P[8] * r[2];
}

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

__global__ void __launch_bounds__(PCG_THREADS) k_pcg(PcgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[PCG_THREADS / 32];
  __shared__ double bc[1];
  const Operator& op = a.op;
  const int n = op.n;
  const int G = gridDim.x;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)G * blockDim.x;
  double* X0 = a.X;
  auto Xb = [&](int k) { return a.X + (size_t)k * 3 * n; };

  // phase 0: r = b, z = P^-1 r, p = z, x = 0
  double acc_b = 0.0, acc_rz = 0.0;
  for (int64_t i = tid; i < n; i += stride) {
    double rv[3] = {a.rhs[3 * i], a.rhs[3 * i + 1], a.rhs[3 * i + 2]};
    double zv[3];
    apply_pinv(op.pinv + 9 * i, rv, zv);
    for (int c = 0; c < 3; ++c) {
      a.r[3 * i + c] = rv[c];
      a.z[3 * i + c] = zv[c];
      a.p[3 * i + c] = zv[c];
      X0[3 * i + c] = 0.0;
      acc_b += rv[c] * rv[c];
      acc_rz += rv[c] * zv[c];
    }
  }
  acc_b = block_sum(acc_b, red);
  acc_rz = block_sum(acc_rz, red);
  if (threadIdx.x == 0) {
    a.part[0 * G + blockIdx.x] = acc_b;
    a.part[1 * G + blockIdx.x] = acc_rz;
  }
  grid.sync();
  const double bnorm = sqrt(grid_total(a.part, 0, bc));
  double rz = grid_total(a.part, 1, bc);
  int cur = 0, best = 0, result = 0;
  double best_res = bnorm;
  int64_t iters = 0;
  bool conv = false;
  double rel = 0.0;
  if (bnorm == 0.0) {
    conv = true;
  } else {
    bool done = false;
    for (int64_t it = 1; it <= a.max_iters; ++it) {
      // ---- hp = H p (+ contact), pAp partials
      if (op.contact.n) {
        for (int64_t c = tid; c < op.contact.n; c += stride) contact_dot(op, a.p, (int)c);
        grid.sync();
      }
      double acc = 0.0;
      for (int64_t t = tid; t < 3LL * n; t += stride) {
        const int i = (int)(t / 3), rr = (int)(t - 3LL * i);
        const double v = row_product(op, a.p, i, rr);
        a.hp[t] = v;
        acc += a.p[t] * v;
      }
      acc = block_sum(acc, red);
      if (threadIdx.x == 0) a.part[2 * G + blockIdx.x] = acc;
      grid.sync();
      const double pap = grid_total(a.part, 2, bc);
      if (pap <= 0.0) {
        // lost positive definiteness along p: keep the best iterate
        result = best;
        iters = it - 1;
        conv = false;
        rel = best_res / bnorm;
        done = true;
        break;
      }
      const double alpha = rz / pap;
      const int nxt = (cur != 0 && best != 0) ? 0 : ((cur != 1 && best != 1) ? 1 : 2);
      const double* xc = Xb(cur);
      double* xn = Xb(nxt);
      double acc_rr = 0.0;
      acc_rz = 0.0;
      for (int64_t i = tid; i < n; i += stride) {
        double rv[3], zv[3];
        for (int c = 0; c < 3; ++c) {
          const int64_t k = 3 * i + c;
          xn[k] = xc[k] + alpha * a.p[k];
          rv[c] = a.r[k] - alpha * a.hp[k];
          a.r[k] = rv[c];
          acc_rr += rv[c] * rv[c];
        }
        apply_pinv(op.pinv + 9 * i, rv, zv);
        for (int c = 0; c < 3; ++c) {
          a.z[3 * i + c] = zv[c];
          acc_rz += rv[c] * zv[c];
        }
      }
      acc_rr = block_sum(acc_rr, red);
      acc_rz = block_sum(acc_rz, red);
      if (threadIdx.x == 0) {
        a.part[0 * G + blockIdx.x] = acc_rr;
        a.part[1 * G + blockIdx.x] = acc_rz;
      }
      grid.sync();
      const double res = sqrt(grid_total(a.part, 0, bc));
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
        if (op.contact.n) {
          for (int64_t c = tid; c < op.contact.n; c += stride) contact_dot(op, Xb(cur), (int)c);
          grid.sync();
        }
        for (int64_t t = tid; t < 3LL * n; t += stride) {
          const int i = (int)(t / 3), rr = (int)(t - 3LL * i);
          a.hp[t] = row_product(op, Xb(cur), i, rr);
        }
        grid.sync();
        acc_rz = 0.0;
        for (int64_t i = tid; i < n; i += stride) {
          double rv[3], zv[3];
          for (int c = 0; c < 3; ++c) rv[c] = a.rhs[3 * i + c] - a.hp[3 * i + c];
          apply_pinv(op.pinv + 9 * i, rv, zv);
          for (int c = 0; c < 3; ++c) {
            a.r[3 * i + c] = rv[c];
            a.z[3 * i + c] = zv[c];
            a.p[3 * i + c] = zv[c];
            acc_rz += rv[c] * zv[c];
          }
        }
        acc_rz = block_sum(acc_rz, red);
        if (threadIdx.x == 0) a.part[1 * G + blockIdx.x] = acc_rz;
        grid.sync();
        rz = grid_total(a.part, 1, bc);
        continue;
      }
      const double rz_new = grid_total(a.part, 1, bc);
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int64_t k = tid; k < 3LL * n; k += stride) a.p[k] = a.z[k] + beta * a.p[k];
      grid.sync();
    }
    if (!done) {
      result = best;
      iters = a.max_iters;
      conv = false;
      rel = best_res / bnorm;
    }
  }
  const double* xr = Xb(result);
  for (int64_t k = tid; k < 3LL * n; k += stride) a.x_out[k] = (bnorm == 0.0) ? 0.0 : xr[k];
  if (tid == 0) {
    a.info[0] = (double)iters;
    a.info[1] = conv ? 1.0 : 0.0;
    a.info[2] = rel;
  }
}

static int pcg_grid(int n) {
  static int max_blocks_per_sm = -1;
  if (max_blocks_per_sm < 0) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pcg, PCG_THREADS, 0);
    max_blocks_per_sm = nb > 0 ? nb : 1;
  }
  const int64_t want = std::max<int64_t>(1, div_up(3LL * n, PCG_THREADS));
  return (int)std::min<int64_t>(want, (int64_t)max_blocks_per_sm * sm_count());
}

int pcg_solve(const Operator& op, const double* rhs, double* x_out, double rel_tol, int64_t max_iters,
              PcgWork& w, cudaStream_t s) {
  const int n = op.n;
  if (max_iters <= 0) max_iters = 10LL * n;
  const size_t n3 = 3 * (size_t)std::max(n, 1);
  IBF_TRY(w.r.reserve(n3));
  IBF_TRY(w.z.reserve(n3));
  IBF_TRY(w.p.reserve(n3));
  IBF_TRY(w.hp.reserve(n3));
  IBF_TRY(w.X.reserve(3 * n3));
  IBF_TRY(w.info.reserve(4));
  const int grid = pcg_grid(std::max(n, 1));
  IBF_TRY(w.part.reserve(4 * (size_t)grid));
  w.grid = grid;
  PcgArgs a;
  a.op = op;
  a.rhs = rhs;
  a.x_out = x_out;
  a.r = w.r.p;
  a.z = w.z.p;
  a.p = w.p.p;
  a.hp = w.hp.p;
  a.X = w.X.p;
  a.part = w.part.p;
  a.info = w.info.p;
  a.tol = rel_tol;
  a.max_iters = max_iters;
  void* args[] = {&a};
  IBF_CUDA(cudaLaunchCooperativeKernel((void*)k_pcg, grid, PCG_THREADS, args, 0, s));
  ++g_launches;
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

// ===================================================== standalone BSR handle

struct ibf_bsr {
  int64_t n = 0;
  std::vector<int64_t> rows, cols;           // coalesced, host copy
  ibf::DevBuf<int> row_ptr, col, low_ptr, low_blk, low_row, diag_blk, brow;
  ibf::DevBuf<double> val, pinv;
  ibf::PcgWork work;
  ibf::Operator op() const {
    ibf::Operator o;
    o.n = (int)n;
    o.row_ptr = row_ptr.p;
    o.col = col.p;
    o.val = val.p;
    o.low_ptr = low_ptr.p;
    o.low_pair = reinterpret_cast<const int2*>(low_blk.p);
    o.pinv = pinv.p;
    return o;
  }
};

namespace ibf {
// Build (row_ptr, lower index, diag ids) for coalesced upper blocks sorted by (row, col).
int build_upper_structure(int64_t n, const std::vector<int64_t>& rows, const std::vector<int64_t>& cols,
                          DevBuf<int>& row_ptr, DevBuf<int>& col, DevBuf<int>& low_ptr, DevBuf<int>& low_blk,
                          DevBuf<int>& low_row, DevBuf<int>& diag_blk, DevBuf<int>& brow) {
  // low_blk holds (block, row) pairs interleaved (int2), low_row is unused
  const int64_t nb = (int64_t)rows.size();
  std::vector<int> rp(n + 1, 0), cl(nb), db(n, -1), br(nb);
  for (int64_t b = 0; b < nb; ++b) {
    rp[rows[b] + 1]++;
    cl[b] = (int)cols[b];
    br[b] = (int)rows[b];
    if (rows[b] == cols[b]) db[rows[b]] = (int)b;
  }
  for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
  // transpose index: off-diagonal blocks grouped by column, rows ascending
  std::vector<int> lp(n + 1, 0);
  for (int64_t b = 0; b < nb; ++b)
    if (rows[b] != cols[b]) lp[cols[b] + 1]++;
  for (int64_t i = 0; i < n; ++i) lp[i + 1] += lp[i];
  std::vector<int> fill(lp.begin(), lp.end() - 1), lb(lp[n]), lr(lp[n]);
  for (int64_t b = 0; b < nb; ++b) {  // b ascending => rows ascending within a column
    if (rows[b] == cols[b]) continue;
    const int k = fill[cols[b]]++;
    lb[k] = (int)b;
    lr[k] = (int)rows[b];
  }
  IBF_TRY(row_ptr.upload(rp.data(), rp.size()));
  IBF_TRY(col.upload(cl.data(), cl.size()));
  IBF_TRY(low_ptr.upload(lp.data(), lp.size()));
  std::vector<int> pairs(2 * lb.size());
  for (size_t k = 0; k < lb.size(); ++k) {
    pairs[2 * k] = lb[k];
    pairs[2 * k + 1] = lr[k];
  }
  IBF_TRY(low_blk.upload(pairs.data(), pairs.size()));
  IBF_TRY(low_row.upload(lr.data(), lr.size()));
  IBF_TRY(diag_blk.upload(db.data(), db.size()));
  IBF_TRY(brow.upload(br.data(), br.size()));
  return IBF_OK;
}

__global__ void k_mask_dirichlet(int64_t nb, const int* __restrict__ brow, const int* __restrict__ col,
                                 const uint8_t* __restrict__ mask, const double* __restrict__ diag,
                                 double* __restrict__ val) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int r = brow[b], c = col[b];
    if (!(mask[r] || mask[c])) continue;
    for (int k = 0; k < 9; ++k) val[9 * b + k] = (r == c) ? diag[9 * (int64_t)r + k] : 0.0;
  }
}
}  // namespace ibf

using namespace ibf;

extern "C" int ibf_bsr_create(int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                              const double* blocks, ibf_bsr** out) {
  if (n < 0 || nnz < 0 || !out) {
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
  ibf_bsr* m = new ibf_bsr();
  m->n = n;
  std::vector<double> vals;
  for (int64_t k = 0; k < nnz; ++k) {
    const int64_t s = order[k];
    const int64_t key = rows[s] * n + cols[s];
    if (k == 0 || key != m->rows.back() * n + m->cols.back()) {
      m->rows.push_back(rows[s]);
      m->cols.push_back(cols[s]);
      vals.insert(vals.end(), blocks + 9 * s, blocks + 9 * s + 9);
    } else {
      double* dst = vals.data() + vals.size() - 9;
      for (int e = 0; e < 9; ++e) dst[e] += blocks[9 * s + e];
    }
  }
  int st = build_upper_structure(n, m->rows, m->cols, m->row_ptr, m->col, m->low_ptr, m->low_blk, m->low_row,
                                 m->diag_blk, m->brow);
  if (st == IBF_OK) st = m->val.upload(vals.data(), vals.size());
  if (st == IBF_OK) st = m->pinv.reserve(9 * (size_t)std::max<int64_t>(n, 1));
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
  return spmv(m->op(), x, y, (cudaStream_t)st);
}

extern "C" int ibf_bsr_mask_dirichlet(ibf_bsr* m, const uint8_t* vertex_mask, const double* diag, ibf_stream st) {
  cudaStream_t s = (cudaStream_t)st;
  DevBuf<uint8_t> dm;
  DevBuf<double> dd;
  IBF_TRY(dm.upload(vertex_mask, (size_t)m->n, s));
  IBF_TRY(dd.upload(diag, 9 * (size_t)m->n, s));
  const int64_t nb = (int64_t)m->rows.size();
  if (nb) {
    k_mask_dirichlet<<<(int)div_up(nb, 256), 256, 0, s>>>(nb, m->brow.p, m->col.p, dm.p, dd.p, m->val.p);
    IBF_LAUNCH_CHECK();
  }
  IBF_CUDA(cudaStreamSynchronize(s));
  return IBF_OK;
}

extern "C" int ibf_bsr_pcg(ibf_bsr* m, const double* rhs, double* x_out, double rel_tol, int64_t max_iters,
                           double* info_host, ibf_stream st) {
  cudaStream_t s = (cudaStream_t)st;
  IBF_TRY(invert_diag_blocks((int)m->n, m->val.p, m->diag_blk.p, m->pinv.p, s));
  IBF_TRY(pcg_solve(m->op(), rhs, x_out, rel_tol, max_iters, m->work, s));
  return pcg_info(m->work, info_host, s);
}

extern "C" int64_t ibf_bsr_size(const ibf_bsr* m) { return m ? (int64_t)m->rows.size() : 0; }

extern "C" int ibf_bsr_export(const ibf_bsr* m, int64_t* rows, int64_t* cols, double* blocks, ibf_stream st) {
  cudaStream_t s = (cudaStream_t)st;
  const int64_t nb = (int64_t)m->rows.size();
  std::copy(m->rows.begin(), m->rows.end(), rows);
  std::copy(m->cols.begin(), m->cols.end(), cols);
  if (nb) IBF_CUDA(cudaMemcpyAsync(blocks, m->val.p, 9 * nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  return IBF_OK;
}
