// Continuous collision detection on the device: swept-box LBVH broad phase,
// bit-exact additive-CCD narrow phase, global step limit, blocking pairs.
//
// Replaces (paths relative to /root/reference/pkg/src):
//   swept_boxes / AABBTree       intact/bvh.py:172-174, :54-154
//   candidate_pairs              intact/ccd.py:113-145
//   accd_batch                   intact/ccd.py:37-91
//   max_step_size, BlockingPairs intact/ccd.py:148-193
//   vf_eval / ee_eval            intact/distance.py:153-189
//
// Broad phase.  Boxes are the reference's swept (start U end) boxes with its
// asymmetric pads (triangles +min_gap, vertices 0, edges 0.5*min_gap), in
// FP64 — min/max/+-pad are exact, so the overlap set is bit-identical to the
// reference's whatever tree is used.  Tree: Karras LBVH over 30-bit Morton
// codes with the primitive index in the low 32 bits (unique keys), CUB radix
// sort, bottom-up refit with arrival flags.  One thread per query traverses
// with a private stack.
//
// Fused narrow-phase prefilter.  For max_step_size only pairs that can block
// matter: a candidate whose starting gap is <= 0 has TOI 0, and one whose
// motion bound l_p is below its gap keeps TOI 1 without advancement
// (intact/ccd.py:64-68).  The traversal evaluates that test in place and
// appends only the survivors (usually a tiny fraction), which are then sorted
// (deterministic order) and advanced by one thread each.
#include <mutex>
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "geometry.cuh"
#include "internal.cuh"

namespace ibf {

using geo::V3;

// ---------------------------------------------------------------- batched API kernels

__global__ void k_pair_eval(int kind, int64_t n, const double* __restrict__ pts, double* __restrict__ d,
                            double* __restrict__ grad, double* __restrict__ wts, uint8_t* __restrict__ degen) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    V3 P[4];
    for (int k = 0; k < 4; ++k) P[k] = geo::ld3(pts + 12 * i + 3 * k);
    double g[12], w[4];
    bool dg;
    const double dd = geo::pair_eval(kind, P, g, w, dg);
    if (d) d[i] = dd;
    if (grad)
      for (int k = 0; k < 12; ++k) grad[12 * i + k] = g[k];
    if (wts)
      for (int k = 0; k < 4; ++k) wts[4 * i + k] = w[k];
    if (degen) degen[i] = dg ? 1 : 0;
  }
}

__global__ void k_accd_batch(int kind, int64_t n, const double* __restrict__ x0, const double* __restrict__ x1,
                             double min_gap, double* __restrict__ toi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    V3 A[4], B[4];
    for (int k = 0; k < 4; ++k) {
      A[k] = geo::ld3(x0 + 12 * i + 3 * k);
      B[k] = geo::ld3(x1 + 12 * i + 3 * k);
    }
    toi[i] = geo::accd_toi(kind, A, B, min_gap);
  }
}

// ---------------------------------------------------------------- boxes

// swept boxes of primitives of arity K (1 point, 2 edge, 3 triangle)
template <int K>
__global__ void k_swept_boxes(int64_t n, const int* __restrict__ prims, const double* __restrict__ x0,
                              const double* __restrict__ x1, double pad, double* __restrict__ lo,
                              double* __restrict__ hi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      double l0 = INFINITY, h0 = -INFINITY, l1 = INFINITY, h1 = -INFINITY;
      for (int k = 0; k < K; ++k) {
        const int64_t v = prims[K * i + k];
        const double a = x0[3 * v + c], b = x1[3 * v + c];
        l0 = geo::np_min(l0, a);
        h0 = geo::np_max(h0, a);
        l1 = geo::np_min(l1, b);
        h1 = geo::np_max(h1, b);
      }
      lo[3 * i + c] = geo::sub(geo::np_min(l0, l1), pad);
      hi[3 * i + c] = geo::add(geo::np_max(h0, h1), pad);
    }
  }
}

// centre bounds for Morton normalisation: per-block partials
__global__ void k_bounds(int64_t n, const double* __restrict__ lo, const double* __restrict__ hi,
                         double* __restrict__ part) {
  __shared__ double red[8];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < 3; ++c) {
      const double ctr = 0.5 * (lo[3 * i + c] + hi[3 * i + c]);
      if (ctr == ctr) {
        mn[c] = fmin(mn[c], ctr);
        mx[c] = fmax(mx[c], ctr);
      }
    }
  for (int c = 0; c < 3; ++c) {
    const double a = -block_max(-mn[c], red);
    const double b = block_max(mx[c], red);
    if (threadIdx.x == 0) {
      part[6 * blockIdx.x + c] = a;
      part[6 * blockIdx.x + 3 + c] = b;
    }
  }
}

__device__ __forceinline__ unsigned int spread10(unsigned int v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void k_morton(int64_t n, const double* __restrict__ lo, const double* __restrict__ hi,
                         const double* __restrict__ part, int nparts, unsigned long long* __restrict__ keys) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int b = 0; b < nparts; ++b)
    for (int c = 0; c < 3; ++c) {
      mn[c] = fmin(mn[c], part[6 * b + c]);
      mx[c] = fmax(mx[c], part[6 * b + 3 + c]);
    }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned int q[3];
    for (int c = 0; c < 3; ++c) {
      const double span = mx[c] - mn[c];
      const double ctr = 0.5 * (lo[3 * i + c] + hi[3 * i + c]);
      double u = (span > 0.0 && ctr == ctr) ? (ctr - mn[c]) / span : 0.0;
      u = fmin(fmax(u, 0.0), 1.0);
      q[c] = (unsigned int)(u * 1023.0);
    }
    const unsigned long long code = (spread10(q[0]) << 2) | (spread10(q[1]) << 1) | spread10(q[2]);
    keys[i] = (code << 32) | (unsigned long long)i;
  }
}

// ---------------------------------------------------------------- LBVH (Karras 2012)

__device__ __forceinline__ int delta(const unsigned long long* k, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  return __clzll(k[i] ^ k[j]);
}

// internal nodes 0..n-2, leaves n-1..2n-2 (leaf n-1+i holds sorted slot i)
__global__ void k_build(int n, const unsigned long long* __restrict__ k, int* __restrict__ left,
                        int* __restrict__ right, int* __restrict__ parent, int* __restrict__ last,
                        int* __restrict__ first) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
    const int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) >= 0 ? 1 : -1;
    const int dmin = delta(k, n, i, i - d);
    int lmax = 2;
    while (delta(k, n, i, i + lmax * d) > dmin) lmax *= 2;
    int l = 0;
    for (int t = lmax / 2; t >= 1; t /= 2)
      if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
    const int j = i + l * d;
    const int dnode = delta(k, n, i, j);
    int s = 0;
    int div = 2;
    int t;
    do {
      t = (l + div - 1) / div;
      if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
      div *= 2;
    } while (t > 1);
    const int g = i + s * d + min(d, 0);
    const int lc = (min(i, j) == g) ? (n - 1 + g) : g;
    const int rc = (max(i, j) == g + 1) ? (n - 1 + g + 1) : g + 1;
    left[i] = lc;
    right[i] = rc;
    parent[lc] = i;
    parent[rc] = i;
    last[i] = max(i, j);   // the node covers sorted slots [min(i, j), max(i, j)]
    if (first) first[i] = min(i, j);
  }
}

// Traversal record of an internal node: both children's boxes in float,
// rounded outward (lo toward -inf, hi toward +inf), and the child indices —
// 64 bytes, one aligned half line per visited node, two children tested per
// fetch.  The float boxes contain the exact FP64 ones, so they never prune a
// real overlap; leaves are then tested exactly against the primitive's FP64
// box, so the candidate set is the one the FP64 tree gives (bit-identical to
// the reference's, intact/ccd.py:104-145).
struct __align__(16) PackedNode {
  float4 a;  // lo_L.xyz, hi_L.x
  float4 b;  // hi_L.yz, lo_R.xy
  float4 c;  // lo_R.z, hi_R.xyz
  int4 d;    // left, right, last sorted slot under left, last sorted slot under right
};

// write node `node`'s FP64 box (lo, hi) into its parent's packed record
__device__ __forceinline__ void pack_child(PackedNode* packed, int par, bool is_left, const double lo[3],
                                           const double hi[3]) {
  float* f = reinterpret_cast<float*>(packed + par);
  const int o = is_left ? 0 : 6;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    f[o + c] = __double2float_rd(lo[c]);
    f[o + 3 + c] = __double2float_ru(hi[c]);
  }
}

__global__ void k_refit(int n, const unsigned long long* __restrict__ k, const double* __restrict__ plo,
                        const double* __restrict__ phi, const int* __restrict__ left, const int* __restrict__ right,
                        const int* __restrict__ parent, int* __restrict__ flag, double* __restrict__ nlo,
                        double* __restrict__ nhi, PackedNode* __restrict__ packed) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int prim = (int)(k[i] & 0xffffffffull);
    int node = n - 1 + i;
    double lo[3], hi[3];
    for (int c = 0; c < 3; ++c) {
      lo[c] = plo[3 * prim + c];
      hi[c] = phi[3 * prim + c];
      nlo[3 * node + c] = lo[c];
      nhi[3 * node + c] = hi[c];
    }
    if (n == 1) continue;
    if (packed) {
      const int par = parent[node];
      pack_child(packed, par, left[par] == node, lo, hi);
    }
    __threadfence();
    node = parent[node];
    while (true) {
      const int old = atomicAdd(flag + node, 1);
      if (old == 0) break;  // first arrival: the sibling finishes this node
      const int a = left[node], b = right[node];
      for (int c = 0; c < 3; ++c) {
        lo[c] = fmin(__ldcg(nlo + 3 * a + c), __ldcg(nlo + 3 * b + c));
        hi[c] = fmax(__ldcg(nhi + 3 * a + c), __ldcg(nhi + 3 * b + c));
        nlo[3 * node + c] = lo[c];
        nhi[3 * node + c] = hi[c];
      }
      if (packed) {
        packed[node].d = make_int4(a, b, 0, 0);
        if (node != 0) {
          const int par = parent[node];
          pack_child(packed, par, left[par] == node, lo, hi);
        }
      }
      __threadfence();
      if (node == 0) break;
      node = parent[node];
    }
  }
}

// The ids half of the leaf records: {prim | v0 << 32, v1 | v2 << 32} with the
// primitive's vertex ids (-1 past its arity), so the walk's shared-vertex
// test loads nothing.  Once per topology (the sorted order changes only on
// a rebuild).
__global__ void k_leaf_ids(int n, const unsigned long long* __restrict__ k, const int* __restrict__ prims, int arity,
                           double4* __restrict__ lbox) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int prim = (int)(k[i] & 0xffffffffull);
    int v[3] = {-1, -1, -1};
    for (int j = 0; j < arity; ++j) v[j] = prims[arity * (size_t)prim + j];
    const long long w0 = (long long)(unsigned)prim | ((long long)(unsigned)v[0] << 32);
    const long long w1 = (long long)(unsigned)v[1] | ((long long)(unsigned)v[2] << 32);
    reinterpret_cast<double2*>(lbox)[4 * (size_t)i + 3] = make_double2(__longlong_as_double(w0), __longlong_as_double(w1));
  }
}

// Refit of the packed records alone (no FP64 node boxes): a leaf writes its
// primitive's FP64 box rounded outward into its parent's record; the second
// arrival at a node takes the union of the two float child boxes in its own
// record and writes it into its parent's.  A union of outward-rounded boxes
// contains the exact FP64 union, so the tree stays conservative; the leaves
// are still tested exactly (k_traverse), so the candidate set is unchanged.
__device__ __forceinline__ int slot_last(int c, int nl, const int* __restrict__ last) {
  return c >= nl ? c - nl : last[c];
}
__global__ void k_refit_packed(int n, const unsigned long long* __restrict__ k, const double* __restrict__ plo,
                               const double* __restrict__ phi, const int* __restrict__ left,
                               const int* __restrict__ right, const int* __restrict__ parent,
                               const int* __restrict__ last, int* __restrict__ flag, PackedNode* __restrict__ packed,
                               double4* __restrict__ lbox) {
  const int nl = n - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int prim = (int)(k[i] & 0xffffffffull);
    int node = nl + i;
    {
      const double lo[3] = {plo[3 * prim], plo[3 * prim + 1], plo[3 * prim + 2]};
      const double hi[3] = {phi[3 * prim], phi[3 * prim + 1], phi[3 * prim + 2]};
      if (lbox) {
        // the exact leaf record in sorted-slot order: {lo, hi.x}, {hi.yz,
        // ids}; the ids half is written once per topology (k_leaf_ids)
        lbox[2 * (size_t)i] = make_double4(lo[0], lo[1], lo[2], hi[0]);
        reinterpret_cast<double2*>(lbox)[4 * (size_t)i + 2] = make_double2(hi[1], hi[2]);
      }
      const int par = parent[node];
      pack_child(packed, par, left[par] == node, lo, hi);
    }
    __threadfence();
    node = parent[node];
    while (true) {
      const int old = atomicAdd(flag + node, 1);
      if (old == 0) break;  // first arrival: the sibling finishes this node
      const int a = left[node], b = right[node];
      const float* f = reinterpret_cast<const float*>(packed + node);
      float lo[3], hi[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        lo[c] = fminf(__ldcg(f + c), __ldcg(f + 6 + c));
        hi[c] = fmaxf(__ldcg(f + 3 + c), __ldcg(f + 9 + c));
      }
      packed[node].d = make_int4(a, b, slot_last(a, nl, last), slot_last(b, nl, last));
      if (node == 0) break;
      const int par = parent[node];
      float* g = reinterpret_cast<float*>(packed + par) + (left[par] == node ? 0 : 6);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        g[c] = lo[c];
        g[3 + c] = hi[c];
      }
      __threadfence();
      node = par;
    }
  }
}

// Chunked treelet refit (IBF_CCD_REFIT_CAP = CAP > 0 threads per CTA).  A
// Karras subtree covering the sorted slots [f, l] has its internal nodes
// among the indices [f, l].  Once per topology, k_treelet_lists marks the
// treelet roots (subtrees of <= S = CAP/4 leaves whose parent covers more)
// and the single leaves hanging directly off a larger node; treelets and
// such leaves tile [0, n) into contiguous units.  k_chunk_starts cuts the
// slots into chunks at unit starts, one chunk every T = CAP - S slots
// (snapped forward to the next unit start, so a chunk holds < CAP slots and
// only whole treelets).  Per refit, k_refit_chunks does one chunk per CTA:
// the topology of its slot range staged in shared memory, the same
// bottom-up climb as k_refit_packed with the arrival counters and the
// children's float boxes in shared memory (CTA-scope fences), every finished
// record written to global memory once, and a treelet root's box written
// into its parent's record.  k_refit_top then climbs the top part from the
// treelet roots and single leaves with the device-scope protocol.  Every
// record is a union of the same float boxes (fminf / fmaxf are exact), so
// the records are bit-identical to k_refit_packed's.
#ifndef IBF_TRAV_MINB
#define IBF_TRAV_MINB 0  // 0: the compiler's register choice for 128 threads
#endif
#if IBF_TRAV_MINB > 0
#define IBF_TRAV_BOUNDS __launch_bounds__(128, IBF_TRAV_MINB)
#else
#define IBF_TRAV_BOUNDS __launch_bounds__(128)
#endif
#ifndef IBF_PREFILTER_MINB
#define IBF_PREFILTER_MINB 3
#endif
#if IBF_PREFILTER_MINB > 0
#define IBF_PREFILTER_BOUNDS __launch_bounds__(256, IBF_PREFILTER_MINB)
#else
#define IBF_PREFILTER_BOUNDS __launch_bounds__(256)
#endif
#ifndef IBF_TOI_MINB
#define IBF_TOI_MINB 3
#endif
#if IBF_TOI_MINB > 0
#define IBF_TOI_BOUNDS __launch_bounds__(256, IBF_TOI_MINB)
#else
#define IBF_TOI_BOUNDS
#endif
#ifndef IBF_CCD_TREELET_DIV
#define IBF_CCD_TREELET_DIV 4  // treelets of at most CAP / DIV leaves
#endif
#ifndef IBF_CCD_REFIT_CAP
#define IBF_CCD_REFIT_CAP 256
#endif
__global__ void k_treelet_lists(int n, const int* __restrict__ first, const int* __restrict__ last,
                                const int* __restrict__ parent, int S, uint8_t* __restrict__ ucode,
                                uint8_t* __restrict__ is_root, int* __restrict__ items, int* __restrict__ counts) {
  const int nl = n - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nl + n; i += gridDim.x * blockDim.x) {
    const int sz = i < nl ? last[i] - first[i] + 1 : 1;
    if (sz > S) continue;
    if (i == 0) {  // the whole tree is one treelet
      is_root[0] = 1;
      ucode[0] = 1;
      continue;
    }
    const int p = parent[i];
    if (last[p] - first[p] + 1 <= S) continue;
    if (i < nl) {
      is_root[i] = 1;
      ucode[first[i]] = 1;
    } else {
      ucode[i - nl] = 2;
    }
    items[atomicAdd(counts, 1)] = i;
  }
}

__global__ void k_chunk_starts(int n, int T, int nchunks, const uint8_t* __restrict__ ucode,
                               int* __restrict__ chunk) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= nchunks; c += gridDim.x * blockDim.x) {
    int s = c == nchunks ? n : c * T;
    while (s < n && ucode[s] == 0) ++s;
    chunk[c] = s;
  }
}

__device__ __forceinline__ void leaf_box(int slot, const unsigned long long* __restrict__ k,
                                         const double* __restrict__ plo, const double* __restrict__ phi,
                                         double4* __restrict__ lbox, double lo[3], double hi[3]) {
  const int prim = (int)(k[slot] & 0xffffffffull);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[c] = plo[3 * prim + c];
    hi[c] = phi[3 * prim + c];
  }
  if (lbox) {
    lbox[2 * (size_t)slot] = make_double4(lo[0], lo[1], lo[2], hi[0]);
    reinterpret_cast<double2*>(lbox)[4 * (size_t)slot + 2] = make_double2(hi[1], hi[2]);
  }
}

constexpr size_t refit_chunk_smem(int cap) { return (size_t)cap * (12 * sizeof(float) + 6 * sizeof(int) + 1); }

template <int CAP>
__global__ void __launch_bounds__(CAP) k_refit_chunks(int n, const unsigned long long* __restrict__ k,
                                                      const double* __restrict__ plo, const double* __restrict__ phi,
                                                      const int* __restrict__ left, const int* __restrict__ right,
                                                      const int* __restrict__ parent, const int* __restrict__ last,
                                                      const int* __restrict__ chunk,
                                                      const uint8_t* __restrict__ ucode,
                                                      const uint8_t* __restrict__ is_root,
                                                      PackedNode* __restrict__ packed, double4* __restrict__ lbox) {
  extern __shared__ float smem[];
  float(*sb)[12] = reinterpret_cast<float(*)[12]>(smem);  // children's float boxes of internal node f + j
  int* sflag = reinterpret_cast<int*>(smem + 12 * CAP);
  int* sl = sflag + CAP;     // internal node f + j: children,
  int* sr = sl + CAP;
  int* sp = sr + CAP;        // parent,
  int* slast = sp + CAP;     // last slot
  int* slp = slast + CAP;    // parent of leaf slot f + j
  uint8_t* sroot = reinterpret_cast<uint8_t*>(slp + CAP);
  const int nl = n - 1;
  const int f = chunk[blockIdx.x], m = chunk[blockIdx.x + 1] - f;
  const int j = threadIdx.x;
  uint8_t code = 0;
  if (j < m) {
    sflag[j] = 0;
    if (f + j < nl) {
      sl[j] = left[f + j];
      sr[j] = right[f + j];
      sp[j] = parent[f + j];
      slast[j] = last[f + j];
      sroot[j] = is_root[f + j];
    }
    slp[j] = parent[nl + f + j];
    code = ucode[f + j];
  }
  __syncthreads();
  if (j >= m) return;
  const int slot = f + j;
  double dlo[3], dhi[3];
  leaf_box(slot, k, plo, phi, lbox, dlo, dhi);
  int node = nl + slot;
  int par = slp[j];
  if (code == 2) {  // a single leaf under a top node
    pack_child(packed, par, left[par] == node, dlo, dhi);
    return;
  }
  {
    volatile float* g = sb[par - f] + (sl[par - f] == node ? 0 : 6);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      g[c] = __double2float_rd(dlo[c]);
      g[3 + c] = __double2float_ru(dhi[c]);
    }
  }
  node = par;
  while (true) {
    const int q = node - f;
    __threadfence_block();
    if (atomicAdd(&sflag[q], 1) == 0) return;  // the sibling's thread finishes this node
    __threadfence_block();
    const volatile float* b = sb[q];
    float v[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) v[c] = b[c];
    const int a = sl[q], bb = sr[q];
    const int la = a >= nl ? a - nl : slast[a - f], lb = bb >= nl ? bb - nl : slast[bb - f];
    packed[node].a = make_float4(v[0], v[1], v[2], v[3]);
    packed[node].b = make_float4(v[4], v[5], v[6], v[7]);
    packed[node].c = make_float4(v[8], v[9], v[10], v[11]);
    packed[node].d = make_int4(a, bb, la, lb);
    float lo[3], hi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fminf(v[c], v[6 + c]);
      hi[c] = fmaxf(v[3 + c], v[9 + c]);
    }
    if (sroot[q]) {
      if (node != 0) {
        par = sp[q];
        float* g = reinterpret_cast<float*>(packed + par) + (left[par] == node ? 0 : 6);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          g[c] = lo[c];
          g[3 + c] = hi[c];
        }
      }
      return;
    }
    par = sp[q];
    volatile float* g = sb[par - f] + (sl[par - f] == node ? 0 : 6);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      g[c] = lo[c];
      g[3 + c] = hi[c];
    }
    node = par;
  }
}

// the top part: climbs from the treelet roots and single leaves, whose
// boxes k_refit_chunks wrote into their parents' records
__global__ void k_refit_top(int n, const int* __restrict__ left, const int* __restrict__ right,
                            const int* __restrict__ parent, const int* __restrict__ last,
                            const int* __restrict__ items, const int* __restrict__ counts, int* __restrict__ flag,
                            PackedNode* __restrict__ packed) {
  const int nl = n - 1;
  const int nitems = counts[0];
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < nitems; it += gridDim.x * blockDim.x) {
    int node = parent[items[it]];
    while (true) {
      const int old = atomicAdd(flag + node, 1);
      if (old == 0) break;
      const int a = left[node], b = right[node];
      const float* f = reinterpret_cast<const float*>(packed + node);
      float lo[3], hi[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        lo[c] = fminf(__ldcg(f + c), __ldcg(f + 6 + c));
        hi[c] = fmaxf(__ldcg(f + 3 + c), __ldcg(f + 9 + c));
      }
      packed[node].d = make_int4(a, b, slot_last(a, nl, last), slot_last(b, nl, last));
      if (node == 0) break;
      const int par = parent[node];
      float* g = reinterpret_cast<float*>(packed + par) + (left[par] == node ? 0 : 6);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        g[c] = lo[c];
        g[3 + c] = hi[c];
      }
      __threadfence();
      node = par;
    }
  }
}

// 4-wide traversal records (IBF_CCD_WIDE): the binary tree collapsed two
// levels at a time.  The record of an even-depth internal node holds its
// grandchildren (or a leaf child itself, with an empty slot beside it):
// four float boxes (SoA across the slots), the child ids (>= n-1: leaf,
// else an even-depth internal node with its own record, -1: empty) and each
// child's last sorted slot.  128 bytes, one L2 line, per visited node — a
// walk takes about half the dependent fetches of the binary records.
struct __align__(128) WideNode {
  float4 lx, ly, lz, hx, hy, hz;
  int4 child;
  int4 last;
};

// depth parity of every internal node (1: odd), once per topology
__global__ void k_depth_parity(int n, const int* __restrict__ parent, uint8_t* __restrict__ odd) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
    int x = i, d = 0;
    while (x != 0) {
      x = parent[x];
      d ^= 1;
    }
    odd[i] = (uint8_t)d;
  }
}

// wide records of the even-depth internal nodes from the refitted binary records
__global__ void k_widen(int n, const uint8_t* __restrict__ odd, const PackedNode* __restrict__ packed,
                        WideNode* __restrict__ wide) {
  const int nl = n - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) {
    if (odd[i]) continue;
    const float* P = reinterpret_cast<const float*>(packed + i);
    const int4 D = packed[i].d;
    float lo[4][3], hi[4][3];
    int ch[4], la[4];
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int cid = side ? D.y : D.x;
      const int clast = side ? D.w : D.z;
      const int s0 = 2 * side;
      if (cid >= nl) {
        ch[s0] = cid;
        la[s0] = clast;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          lo[s0][c] = P[6 * side + c];
          hi[s0][c] = P[6 * side + 3 + c];
        }
        ch[s0 + 1] = -1;
        la[s0 + 1] = -1;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          lo[s0 + 1][c] = INFINITY;
          hi[s0 + 1][c] = -INFINITY;
        }
      } else {
        const float* Q = reinterpret_cast<const float*>(packed + cid);
        const int4 E = packed[cid].d;
        ch[s0] = E.x;
        ch[s0 + 1] = E.y;
        la[s0] = E.z;
        la[s0 + 1] = E.w;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          lo[s0][c] = Q[c];
          hi[s0][c] = Q[3 + c];
          lo[s0 + 1][c] = Q[6 + c];
          hi[s0 + 1][c] = Q[9 + c];
        }
      }
    }
    WideNode w;
    w.lx = make_float4(lo[0][0], lo[1][0], lo[2][0], lo[3][0]);
    w.ly = make_float4(lo[0][1], lo[1][1], lo[2][1], lo[3][1]);
    w.lz = make_float4(lo[0][2], lo[1][2], lo[2][2], lo[3][2]);
    w.hx = make_float4(hi[0][0], hi[1][0], hi[2][0], hi[3][0]);
    w.hy = make_float4(hi[0][1], hi[1][1], hi[2][1], hi[3][1]);
    w.hz = make_float4(hi[0][2], hi[1][2], hi[2][2], hi[3][2]);
    w.child = make_int4(ch[0], ch[1], ch[2], ch[3]);
    w.last = make_int4(la[0], la[1], la[2], la[3]);
    wide[i] = w;
  }
}

struct Tree {
  int n;
  const unsigned long long* keys;  // sorted
  const int* left;
  const int* right;
  const double* lo;
  const double* hi;
  const PackedNode* packed;        // internal-node records (null: FP64 node arrays only)
  const WideNode* wide;            // 4-wide records of the even-depth internal nodes, or null
  const double4* lbox;             // exact leaf records by sorted slot (2 double4 each), or null
  const double* plo;               // primitive boxes (exact leaf test with `packed`)
  const double* phi;
};

__device__ __forceinline__ bool overlap(const double ql[3], const double qh[3], const double* lo, const double* hi) {
  return ql[0] <= hi[0] && ql[1] <= hi[1] && ql[2] <= hi[2] && qh[0] >= lo[0] && qh[1] >= lo[1] && qh[2] >= lo[2];
}

struct TraverseArgs {
  Tree tree;
  int64_t nq;
  const double* qlo;
  const double* qhi;
  int kind;            // 0: vertex-vs-triangle, 1: edge-vs-edge (a < b)
  const int* qprim;    // verts (VF) or edges (EE)
  const int* tprim;    // tris (VF) or edges (EE)
  const double* x0;
  const double* x1;
  double min_gap;
  int filter;          // 1: keep only pairs that can block (TOI 0 or needs advancement)
  unsigned long long* out;
  unsigned long long cap;
  // self-queries (EE, tri-tri): visit the queries in the tree's Morton order
  // (its sorted keys), so a warp's 32 traversals follow nearly the same path
  const unsigned long long* qorder;
  unsigned long long* counters;  // [0] emitted, [1] all candidates
  // 1: leaves are tested exactly (FP64 primitive boxes) inside the walk;
  // 0: the walk emits every leaf whose float box overlaps and k_prefilter
  // runs the exact test (it recomputes both swept boxes from the vertex
  // positions it loads anyway, bit-identically to k_swept_boxes)
  int exact_leaf;
};

__device__ __forceinline__ bool make_quad(const TraverseArgs& a, int qi, int pi, int q[4]) {
  if (a.kind == 2) {  // triangle-triangle (static intersection test): a < b, no shared vertex
    if (!(qi < pi)) return false;
    const int* A = a.qprim + 3 * qi;
    const int* B = a.tprim + 3 * pi;
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (A[i] == B[0] || A[i] == B[1] || A[i] == B[2]) return false;
    q[0] = qi; q[1] = pi; q[2] = q[3] = 0;
    return true;
  }
  if (a.kind == 0) {
    const int v = a.qprim[qi];
    const int t0 = a.tprim[3 * pi], t1 = a.tprim[3 * pi + 1], t2 = a.tprim[3 * pi + 2];
    if (v == t0 || v == t1 || v == t2) return false;
    q[0] = v; q[1] = t0; q[2] = t1; q[3] = t2;
    return true;
  }
  if (!(qi < pi)) return false;
  const int a0 = a.qprim[2 * qi], a1 = a.qprim[2 * qi + 1];
  const int b0 = a.tprim[2 * pi], b1 = a.tprim[2 * pi + 1];
  if (a0 == b0 || a0 == b1 || a1 == b0 || a1 == b1) return false;
  q[0] = a0; q[1] = a1; q[2] = b0; q[3] = b1;
  return true;
}

// one leaf of the query's traversal: shared-vertex / ordering filter, the
// ACCD prefilter, warp-aggregated append
template <bool FILTER>
__device__ __forceinline__ void traverse_leaf(const TraverseArgs& a, int64_t qi, int pi,
                                              unsigned long long& n_cand) {
  int q[4];
  if (!make_quad(a, (int)qi, pi, q)) return;
  ++n_cand;
  bool emit = true;
  if (FILTER) {
    V3 X0[4], X1[4];
    for (int k = 0; k < 4; ++k) {
      X0[k] = geo::ld3(a.x0 + 3 * (int64_t)q[k]);
      X1[k] = geo::ld3(a.x1 + 3 * (int64_t)q[k]);
    }
    emit = geo::accd_class(a.kind, X0, X1, a.min_gap) != 1;
  }
  if (emit) {
    // warp-aggregated append: the lanes emitting at this point take
    // consecutive slots with one atomic for the group
    const unsigned grp = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(grp) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(a.counters, (unsigned long long)__popc(grp));
    base = __shfl_sync(grp, base, leader);
    const unsigned long long slot = base + __popc(grp & ((1u << lane) - 1u));
    if (slot < a.cap) a.out[slot] = ((unsigned long long)qi << 32) | (unsigned long long)pi;
  }
}

__device__ __forceinline__ bool overlap_f(const float ql[3], const float qh[3], float lx, float ly, float lz,
                                          float hx, float hy, float hz) {
  return ql[0] <= hx && ql[1] <= hy && ql[2] <= hz && qh[0] >= lx && qh[1] >= ly && qh[2] >= lz;
}

template <bool FILTER, bool PACKED>
__global__ void __launch_bounds__(128) k_traverse(TraverseArgs a) {
  unsigned long long n_cand = 0;
  const int nl = a.tree.n - 1;   // first leaf node
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < a.nq; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qi = a.qorder ? (int64_t)(a.qorder[t] & 0xffffffffull) : t;
    const double ql[3] = {a.qlo[3 * qi], a.qlo[3 * qi + 1], a.qlo[3 * qi + 2]};
    const double qh[3] = {a.qhi[3 * qi], a.qhi[3 * qi + 1], a.qhi[3 * qi + 2]};
    if (PACKED) {
      // packed records: both children per fetch, float tests, exact FP64
      // test at the leaves; near child first, the other on the stack
      const float qlf[3] = {__double2float_rd(ql[0]), __double2float_rd(ql[1]), __double2float_rd(ql[2])};
      const float qhf[3] = {__double2float_ru(qh[0]), __double2float_ru(qh[1]), __double2float_ru(qh[2])};
      int stack[64];
      int sp = 0;
      int node = 0;
      while (true) {
        const PackedNode* P = a.tree.packed + node;
        const float4 A = __ldg(&P->a), B = __ldg(&P->b), Cq = __ldg(&P->c);
        const int4 D = __ldg(&P->d);
        bool hl = overlap_f(qlf, qhf, A.x, A.y, A.z, A.w, B.x, B.y);
        bool hr = overlap_f(qlf, qhf, B.z, B.w, Cq.x, Cq.y, Cq.z, Cq.w);
        if (hl && D.x >= nl) {
          const int pi = (int)(a.tree.keys[D.x - nl] & 0xffffffffull);
          if (overlap(ql, qh, a.tree.plo + 3 * pi, a.tree.phi + 3 * pi)) traverse_leaf<FILTER>(a, qi, pi, n_cand);
          hl = false;
        }
        if (hr && D.y >= nl) {
          const int pi = (int)(a.tree.keys[D.y - nl] & 0xffffffffull);
          if (overlap(ql, qh, a.tree.plo + 3 * pi, a.tree.phi + 3 * pi)) traverse_leaf<FILTER>(a, qi, pi, n_cand);
          hr = false;
        }
        if (hl && hr) {
          stack[sp++] = D.y;
          node = D.x;
        } else if (hl) {
          node = D.x;
        } else if (hr) {
          node = D.y;
        } else {
          if (sp == 0) break;
          node = stack[--sp];
        }
      }
      continue;
    }
    // LBVH depth is bounded by the 64 key bits, so depth+1 entries suffice
    int stack[80];
    int sp = 0;
    stack[sp++] = 0;  // root: internal node 0, or the single leaf when n == 1
    while (sp) {
      const int node = stack[--sp];
      if (!overlap(ql, qh, a.tree.lo + 3 * node, a.tree.hi + 3 * node)) continue;
      if (node >= nl) {
        traverse_leaf<FILTER>(a, qi, (int)(a.tree.keys[node - nl] & 0xffffffffull), n_cand);
      } else {
        stack[sp++] = a.tree.right[node];
        stack[sp++] = a.tree.left[node];
      }
    }
  }
  if (n_cand) atomicAdd(a.counters + 1, n_cand);
}

// Packed-tree traversal with dynamic query fetching.  Query walks differ in
// length by an order of magnitude, so a warp that takes 32 queries and runs
// until the longest ends keeps ~8 of its lanes busy (ncu: 8.2-9.0 threads
// per executed instruction).  Here a lane whose walk ends takes the next
// query at once: each warp claims chunks of TRAV_CHUNK queries with one
// global atomic and deals them to its idle lanes by ballot rank, so the
// lanes stay busy until the queries run out.
//
// SELF (EE, triangle-triangle): the queries are the tree's own leaves in
// sorted order, query t sitting at sorted slot t.  Each unordered pair is
// found once, from the leaf with the smaller slot: a child whose last slot is
// <= t is skipped (PackedNode.d.zw), which halves the walks, and the pair is
// emitted in the canonical (smaller id, larger id) orientation the per-query
// `qi < pi` test gave — the same set (intact/ccd.py:131-138).
#ifndef IBF_TRAV_CHUNK
#define IBF_TRAV_CHUNK 32
#endif
constexpr int TRAV_CHUNK = IBF_TRAV_CHUNK;
#ifndef IBF_CCD_PREFETCH
#define IBF_CCD_PREFETCH 0
#endif
template <bool FILTER, bool SELF>
__global__ void __launch_bounds__(128) k_traverse_dyn(TraverseArgs a) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int nl = a.tree.n - 1;
  const long long nq = a.nq;
  unsigned long long n_cand = 0;
  long long pool = 0, pool_end = 0;   // warp-uniform: this warp's unclaimed queries
  bool exhausted = false;             // warp-uniform
  long long t = -1;                   // this lane's query (slot), -1: idle
  int qi = 0;
  double ql[3], qh[3];
  float qlf[3], qhf[3];
  int stack[64];
  int sp = 0, node = 0;
  while (true) {
    unsigned need = __ballot_sync(0xffffffffu, t < 0);
    while (need && !exhausted) {
      if (pool == pool_end) {
        long long b = 0;
        if (lane == 0) b = (long long)atomicAdd(a.counters + 3, (unsigned long long)TRAV_CHUNK);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b >= nq) {
          exhausted = true;
          break;
        }
        pool = b;
        pool_end = b + TRAV_CHUNK < nq ? b + TRAV_CHUNK : nq;
      }
      const long long take = min((long long)__popc(need), pool_end - pool);
      const int rank = __popc(need & lt);
      if (t < 0 && rank < take) {
        t = pool + rank;
        qi = a.qorder ? (int)(a.qorder[t] & 0xffffffffull) : (int)t;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ql[c] = a.qlo[3 * (int64_t)qi + c];
          qh[c] = a.qhi[3 * (int64_t)qi + c];
          qlf[c] = __double2float_rd(ql[c]);
          qhf[c] = __double2float_ru(qh[c]);
        }
        sp = 0;
        node = 0;
      }
      pool += take;
      need = __ballot_sync(0xffffffffu, t < 0);
    }
    if (__ballot_sync(0xffffffffu, t >= 0) == 0) break;
    if (t < 0) continue;
    // one node of this lane's walk
    const PackedNode* P = a.tree.packed + node;
    const float4 A = __ldg(&P->a), B = __ldg(&P->b), Cq = __ldg(&P->c);
    const int4 D = __ldg(&P->d);
    bool hl = overlap_f(qlf, qhf, A.x, A.y, A.z, A.w, B.x, B.y);
    bool hr = overlap_f(qlf, qhf, B.z, B.w, Cq.x, Cq.y, Cq.z, Cq.w);
    if (SELF) {
      hl = hl && D.z > t;
      hr = hr && D.w > t;
    }
    if (hl && D.x >= nl) {
      const int pi = (int)(a.tree.keys[D.x - nl] & 0xffffffffull);
      if (overlap(ql, qh, a.tree.plo + 3 * pi, a.tree.phi + 3 * pi))
        traverse_leaf<FILTER>(a, SELF ? min(qi, pi) : qi, SELF ? max(qi, pi) : pi, n_cand);
      hl = false;
    }
    if (hr && D.y >= nl) {
      const int pi = (int)(a.tree.keys[D.y - nl] & 0xffffffffull);
      if (overlap(ql, qh, a.tree.plo + 3 * pi, a.tree.phi + 3 * pi))
        traverse_leaf<FILTER>(a, SELF ? min(qi, pi) : qi, SELF ? max(qi, pi) : pi, n_cand);
      hr = false;
    }
    if (hl && hr) {
      stack[sp++] = D.y;
      node = D.x;
      // the deferred child's record: start its fetch now (IBF_CCD_PREFETCH)
      if (IBF_CCD_PREFETCH == 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.tree.packed + D.y));
      if (IBF_CCD_PREFETCH == 2) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.tree.packed + D.y));
    } else if (hl) {
      node = D.x;
    } else if (hr) {
      node = D.y;
    } else if (sp > 0) {
      node = stack[--sp];
    } else {
      t = -1;   // walk done
    }
  }
  if (n_cand) atomicAdd(a.counters + 1, n_cand);
}

// k_traverse_dyn over the 4-wide records: same query fetching, slot pruning
// and leaf handling; up to three internal children are pushed per step.
template <bool FILTER, bool SELF>
__global__ void IBF_TRAV_BOUNDS k_traverse_wide(TraverseArgs a) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int nl = a.tree.n - 1;
  const long long nq = a.nq;
  unsigned long long n_cand = 0;
  long long pool = 0, pool_end = 0;
  bool exhausted = false;
  long long t = -1;
  int qi = 0;
  double ql[3], qh[3];
  float qlf[3], qhf[3];
  int qv[3] = {-2, -2, -2};   // the query primitive's vertex ids (-2: none)
  int stack[100];
  int sp = 0, node = 0;
  while (true) {
    unsigned need = __ballot_sync(0xffffffffu, t < 0);
    while (need && !exhausted) {
      if (pool == pool_end) {
        long long b = 0;
        if (lane == 0) b = (long long)atomicAdd(a.counters + 3, (unsigned long long)TRAV_CHUNK);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b >= nq) {
          exhausted = true;
          break;
        }
        pool = b;
        pool_end = b + TRAV_CHUNK < nq ? b + TRAV_CHUNK : nq;
      }
      const long long take = min((long long)__popc(need), pool_end - pool);
      const int rank = __popc(need & lt);
      if (t < 0 && rank < take) {
        t = pool + rank;
        qi = a.qorder ? (int)(a.qorder[t] & 0xffffffffull) : (int)t;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ql[c] = a.qlo[3 * (int64_t)qi + c];
          qh[c] = a.qhi[3 * (int64_t)qi + c];
          qlf[c] = __double2float_rd(ql[c]);
          qhf[c] = __double2float_ru(qh[c]);
        }
        const int ar = a.kind == 0 ? 1 : (a.kind == 1 ? 2 : 3);
#pragma unroll
        for (int j = 0; j < 3; ++j) qv[j] = j < ar ? a.qprim[ar * (int64_t)qi + j] : -2;
        sp = 0;
        node = 0;
      }
      pool += take;
      need = __ballot_sync(0xffffffffu, t < 0);
    }
    if (__ballot_sync(0xffffffffu, t >= 0) == 0) break;
    if (t < 0) continue;
    const WideNode* W = a.tree.wide + node;
    const float4 lx = __ldg(&W->lx), ly = __ldg(&W->ly), lz = __ldg(&W->lz);
    const float4 hx = __ldg(&W->hx), hy = __ldg(&W->hy), hz = __ldg(&W->hz);
    const int4 ch = __ldg(&W->child), la = __ldg(&W->last);
    const int cid[4] = {ch.x, ch.y, ch.z, ch.w};
    const int cl[4] = {la.x, la.y, la.z, la.w};
    const float Lx[4] = {lx.x, lx.y, lx.z, lx.w}, Ly[4] = {ly.x, ly.y, ly.z, ly.w}, Lz[4] = {lz.x, lz.y, lz.z, lz.w};
    const float Hx[4] = {hx.x, hx.y, hx.z, hx.w}, Hy[4] = {hy.x, hy.y, hy.z, hy.w}, Hz[4] = {hz.x, hz.y, hz.z, hz.w};
    int next = -1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bool h = overlap_f(qlf, qhf, Lx[k], Ly[k], Lz[k], Hx[k], Hy[k], Hz[k]);
      if (SELF) h = h && cl[k] > t;
      if (!h) continue;
      const int c = cid[k];
      if (c >= nl) {
        int pi;
        bool hit;
        if (a.tree.lbox) {
          // one 64-byte record per leaf, sibling leaves in adjacent slots
          const double2* L = reinterpret_cast<const double2*>(a.tree.lbox + 2 * (size_t)(c - nl));
          const double2 l0 = __ldg(L), l1 = __ldg(L + 1), l2 = __ldg(L + 2), l3 = __ldg(L + 3);
          const double4 b0 = make_double4(l0.x, l0.y, l1.x, l1.y), b1 = make_double4(l2.x, l2.y, l3.x, l3.y);
          const long long w0 = __double_as_longlong(b1.z), w1 = __double_as_longlong(b1.w);
          pi = (int)(w0 & 0xffffffffll);
          hit = !a.exact_leaf || (ql[0] <= b0.w && ql[1] <= b1.x && ql[2] <= b1.y && qh[0] >= b0.x &&
                                  qh[1] >= b0.y && qh[2] >= b0.z);
          if (hit && !FILTER) {
            // the candidate filter of make_quad on the ids in hand: no shared
            // vertex (and, for self-queries, each pair once: done by the slot
            // pruning); then the warp-aggregated append
            const int tv0 = (int)(w0 >> 32), tv1 = (int)(w1 & 0xffffffffll), tv2 = (int)(w1 >> 32);
            bool shared = false;
#pragma unroll
            for (int j = 0; j < 3; ++j) shared |= qv[j] >= 0 && (qv[j] == tv0 || qv[j] == tv1 || qv[j] == tv2);
            if (!shared) {
              ++n_cand;
              const int lo_i = SELF ? min(qi, pi) : qi, hi_i = SELF ? max(qi, pi) : pi;
              const unsigned grp = __activemask();
              const int leader = __ffs(grp) - 1;
              unsigned long long base = 0;
              if (lane == leader) base = atomicAdd(a.counters, (unsigned long long)__popc(grp));
              base = __shfl_sync(grp, base, leader);
              const unsigned long long slot = base + __popc(grp & lt);
              if (slot < a.cap) a.out[slot] = ((unsigned long long)lo_i << 32) | (unsigned long long)hi_i;
            }
            continue;
          }
        } else {
          pi = (int)(a.tree.keys[c - nl] & 0xffffffffull);
          hit = !a.exact_leaf || overlap(ql, qh, a.tree.plo + 3 * pi, a.tree.phi + 3 * pi);
        }
        if (hit) traverse_leaf<FILTER>(a, SELF ? min(qi, pi) : qi, SELF ? max(qi, pi) : pi, n_cand);
      } else if (next < 0) {
        next = c;
      } else {
        stack[sp++] = c;
      }
    }
    if (next >= 0) {
      node = next;
    } else if (sp > 0) {
      node = stack[--sp];
    } else {
      t = -1;
    }
  }
  if (n_cand) atomicAdd(a.counters + 1, n_cand);
}

// Second stage of the filtered broad phase: the traversal emits every
// candidate (no FP64 work inside the tree walk, so it keeps ~40 % of the
// registers and its warps stay converged between leaves), then one thread
// per candidate runs the ACCD prefilter and appends the survivors.
// swept box of vertices X0/X1[k0 .. k0+K) exactly as k_swept_boxes forms it
__device__ __forceinline__ void quad_box(const V3* X0, const V3* X1, int k0, int K, double pad, double lo[3],
                                         double hi[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double l0 = INFINITY, h0 = -INFINITY, l1 = INFINITY, h1 = -INFINITY;
    for (int k = k0; k < k0 + K; ++k) {
      const double av = c == 0 ? X0[k].x : (c == 1 ? X0[k].y : X0[k].z);
      const double bv = c == 0 ? X1[k].x : (c == 1 ? X1[k].y : X1[k].z);
      l0 = geo::np_min(l0, av);
      h0 = geo::np_max(h0, av);
      l1 = geo::np_min(l1, bv);
      h1 = geo::np_max(h1, bv);
    }
    lo[c] = geo::sub(geo::np_min(l0, l1), pad);
    hi[c] = geo::add(geo::np_max(h0, h1), pad);
  }
}

__global__ void IBF_PREFILTER_BOUNDS k_prefilter(TraverseArgs a, int64_t n, const unsigned long long* __restrict__ cand) {
  unsigned long long n_exact = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long e = cand[i];
    const int qi = (int)(e >> 32), pi = (int)(e & 0xffffffffull);
    int q[4];
    make_quad(a, qi, pi, q);
    V3 X0[4], X1[4];
    for (int k = 0; k < 4; ++k) {
      X0[k] = geo::ld3(a.x0 + 3 * (int64_t)q[k]);
      X1[k] = geo::ld3(a.x1 + 3 * (int64_t)q[k]);
    }
    bool cand_ok = true;
    if (!a.exact_leaf) {
      // the exact FP64 swept-box overlap the walk skipped: VF = vertex (pad 0)
      // vs triangle (pad min_gap), EE = both edges (pad min_gap / 2)
      double la[3], ha[3], lb[3], hb[3];
      if (a.kind == 0) {
        quad_box(X0, X1, 0, 1, 0.0, la, ha);
        quad_box(X0, X1, 1, 3, a.min_gap, lb, hb);
      } else {
        quad_box(X0, X1, 0, 2, 0.5 * a.min_gap, la, ha);
        quad_box(X0, X1, 2, 2, 0.5 * a.min_gap, lb, hb);
      }
      cand_ok = overlap(la, ha, lb, hb);
      n_exact += cand_ok ? 1 : 0;
    }
    if (cand_ok && geo::accd_class(a.kind, X0, X1, a.min_gap) != 1) {
      const unsigned grp = __activemask();
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(grp) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(a.counters, (unsigned long long)__popc(grp));
      base = __shfl_sync(grp, base, leader);
      a.out[base + __popc(grp & ((1u << lane) - 1u))] = e;
    }
  }
  if (n_exact) atomicAdd(a.counters + 1, n_exact);
}

__global__ void IBF_TOI_BOUNDS k_pair_toi(int64_t n, int kind, const unsigned long long* __restrict__ pairs,
                           const int* __restrict__ qprim, const int* __restrict__ tprim,
                           const double* __restrict__ x0, const double* __restrict__ x1, double min_gap,
                           double* __restrict__ toi, int* __restrict__ quad_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int qi = (int)(pairs[i] >> 32), pi = (int)(pairs[i] & 0xffffffffull);
    int q[4];
    if (kind == 0) {
      q[0] = qprim[qi]; q[1] = tprim[3 * pi]; q[2] = tprim[3 * pi + 1]; q[3] = tprim[3 * pi + 2];
    } else {
      q[0] = qprim[2 * qi]; q[1] = qprim[2 * qi + 1]; q[2] = tprim[2 * pi]; q[3] = tprim[2 * pi + 1];
    }
    for (int k = 0; k < 4; ++k) quad_out[4 * i + k] = q[k];
    if (toi) {
      V3 A[4], B[4];
      for (int k = 0; k < 4; ++k) {
        A[k] = geo::ld3(x0 + 3 * (int64_t)q[k]);
        B[k] = geo::ld3(x1 + 3 * (int64_t)q[k]);
      }
      toi[i] = geo::accd_toi(kind, A, B, min_gap);
    }
  }
}

__global__ void k_min_toi(int64_t n, const double* __restrict__ toi, double* __restrict__ out) {
  __shared__ double red[8];
  double v = INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v = fmin(v, toi[i]);
  v = -block_max(-v, red);
  if (threadIdx.x == 0 && v < INFINITY) atomic_min_nonneg(out, v);
}

__global__ void k_block_flag(int64_t n, const double* __restrict__ toi, int* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = toi[i] < 1.0 ? 1 : 0;
}

__global__ void k_block_write(int64_t n, int64_t base, int kind, const int* __restrict__ flag,
                              const int* __restrict__ pos, const int* __restrict__ quad, const double* __restrict__ toi,
                              int* __restrict__ bkind, int* __restrict__ bquad, double* __restrict__ btoi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    const int64_t d = base + pos[i];
    bkind[d] = kind;
    for (int k = 0; k < 4; ++k) bquad[4 * d + k] = quad[4 * i + k];
    btoi[d] = toi[i];
  }
}

__global__ void k_set(double* p, double v) { *p = v; }

static int grid_for(int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(div_up(n, threads), 148LL * 16));
}

// Build the LBVH over n primitive boxes (c->box_lo/hi) into c's node arrays.
// LBVH over the n boxes in c->box_lo/hi (Karras split on sorted Morton keys,
// bottom-up refit).  cache != null: reuse its topology when it was built for
// the same n fewer than IBF_CCD_REBUILD calls ago, refitting only — the
// refit bounds are exact unions of the current leaf boxes, so traversal
// returns the same overlapping pairs; only the tree's tightness ages.
#ifndef IBF_CCD_REBUILD
#define IBF_CCD_REBUILD 16
#endif
// traversal over packed float child-box records (1) or the FP64 node arrays (0)
#ifndef IBF_CCD_PACKED
#define IBF_CCD_PACKED 1
#endif
// VF queries visited in Morton order of their boxes (1) or in vertex order (0):
// 15.7 vs 15.2 ms per CCD pass on the squishy press (the sort costs more)
#ifndef IBF_CCD_VF_ORDER
#define IBF_CCD_VF_ORDER 0
#endif
// exact leaf box test moved from the walk into k_prefilter (1) or kept in the walk (0)
#ifndef IBF_CCD_DEFER_EXACT
#define IBF_CCD_DEFER_EXACT 0
#endif
// exact leaf boxes in sorted-slot records for the wide walk's leaf test (1),
// or through the primitive index and the primitive box arrays (0)
#ifndef IBF_CCD_LEAF_RECORDS
#define IBF_CCD_LEAF_RECORDS 1
#endif
// 4-wide traversal records (1) or the binary packed records (0)
#ifndef IBF_CCD_WIDE
#define IBF_CCD_WIDE 1
#endif
// packed traversal with dynamic query fetching (1) or one query per thread (0)
#ifndef IBF_CCD_DYNAMIC
#define IBF_CCD_DYNAMIC 1
#endif
// filtered broad phase as traversal + a separate prefilter pass (1) or with
// the prefilter inside the traversal (0)
#ifndef IBF_CCD_SPLIT
#define IBF_CCD_SPLIT 1
#endif
static int build_tree(ibf_ccd* c, int64_t n, cudaStream_t s, Tree& t, ibf_ccd::TreeCache* cache = nullptr,
                      const int* prims = nullptr, int arity = 0) {
  const int64_t nn = std::max<int64_t>(2 * n - 1, 1);
  unsigned long long* keys_sorted = c->keys_sorted.p;
  int *left, *right, *parent, *flag, *last;
  double *lo, *hi;
  float4* packed4;
  WideNode* wide = nullptr;
  uint8_t* odd = nullptr;
  double4* lbox = nullptr;
  bool refit_only = false;
  // chunked treelet refit (per-topology lists)
  int *tfirst = nullptr, *titems = nullptr, *tcounts = nullptr, *tchunk = nullptr;
  uint8_t *tucode = nullptr, *troot = nullptr;
  constexpr int kCap = IBF_CCD_REFIT_CAP > 0 ? IBF_CCD_REFIT_CAP : 32, kS = kCap / IBF_CCD_TREELET_DIV, kT = kCap - kS;
  const int nchunks = (int)((n + kT - 1) / kT);
  if (cache) {
    if (IBF_CCD_REFIT_CAP > 0 && IBF_CCD_PACKED) {
      IBF_TRY(cache->first.reserve(nn));
      IBF_TRY(cache->titems.reserve(nn));
      IBF_TRY(cache->tcounts.reserve(2));
      IBF_TRY(cache->tchunk.reserve(nchunks + 1));
      IBF_TRY(cache->tucode.reserve(n));
      IBF_TRY(cache->troot.reserve(nn));
      tfirst = cache->first.p, titems = cache->titems.p, tcounts = cache->tcounts.p, tchunk = cache->tchunk.p;
      tucode = cache->tucode.p, troot = cache->troot.p;
    }
    IBF_TRY(cache->keys_sorted.reserve(n));
    IBF_TRY(cache->left.reserve(nn));
    IBF_TRY(cache->right.reserve(nn));
    IBF_TRY(cache->parent.reserve(nn));
    IBF_TRY(cache->flag.reserve(nn));
    IBF_TRY(cache->last.reserve(nn));
    if (!IBF_CCD_PACKED) {
      IBF_TRY(cache->lo.reserve(3 * nn));
      IBF_TRY(cache->hi.reserve(3 * nn));
    }
    IBF_TRY(cache->packed.reserve(4 * nn));
    if (IBF_CCD_WIDE && IBF_CCD_PACKED && n > 1) {
      IBF_TRY(cache->wide.reserve(8 * (size_t)(n - 1)));
      IBF_TRY(cache->odd.reserve(n - 1));
      wide = reinterpret_cast<WideNode*>(cache->wide.p);
      odd = cache->odd.p;
      if (IBF_CCD_LEAF_RECORDS) {
        IBF_TRY(cache->lbox.reserve(2 * (size_t)n));
        lbox = cache->lbox.p;
      }
    }
    refit_only = cache->n == n && cache->uses < IBF_CCD_REBUILD;
    keys_sorted = cache->keys_sorted.p;
    left = cache->left.p, right = cache->right.p, parent = cache->parent.p, flag = cache->flag.p;
    last = cache->last.p;
    lo = cache->lo.p, hi = cache->hi.p;
    packed4 = cache->packed.p;
  } else {
    IBF_TRY(c->keys_sorted.reserve(n));
    IBF_TRY(c->node_left.reserve(nn));
    IBF_TRY(c->node_right.reserve(nn));
    IBF_TRY(c->node_parent.reserve(nn));
    IBF_TRY(c->node_flag.reserve(nn));
    IBF_TRY(c->node_last.reserve(nn));
    IBF_TRY(c->node_lo.reserve(3 * nn));
    IBF_TRY(c->node_hi.reserve(3 * nn));
    IBF_TRY(c->node_packed.reserve(4 * nn));
    if (IBF_CCD_WIDE && IBF_CCD_PACKED && n > 1) {
      IBF_TRY(c->node_wide.reserve(8 * (size_t)(n - 1)));
      IBF_TRY(c->node_odd.reserve(n - 1));
      wide = reinterpret_cast<WideNode*>(c->node_wide.p);
      odd = c->node_odd.p;
      if (IBF_CCD_LEAF_RECORDS) {
        IBF_TRY(c->node_lbox.reserve(2 * (size_t)n));
        lbox = c->node_lbox.p;
      }
    }
    keys_sorted = c->keys_sorted.p;
    left = c->node_left.p, right = c->node_right.p, parent = c->node_parent.p, flag = c->node_flag.p;
    last = c->node_last.p;
    lo = c->node_lo.p, hi = c->node_hi.p;
    packed4 = c->node_packed.p;
  }
  PackedNode* packed = IBF_CCD_PACKED ? reinterpret_cast<PackedNode*>(packed4) : nullptr;
  if (!refit_only) {
    const int nparts = (int)std::min<int64_t>(grid_for(n), 148 * 2);
    IBF_TRY(c->dscratch.reserve(6 * (size_t)nparts + 8));
    IBF_TRY(c->keys.reserve(n));
    k_bounds<<<nparts, 256, 0, s>>>(n, c->box_lo.p, c->box_hi.p, c->dscratch.p);
    IBF_LAUNCH_CHECK();
    k_morton<<<grid_for(n), 256, 0, s>>>(n, c->box_lo.p, c->box_hi.p, c->dscratch.p, nparts, c->keys.p);
    IBF_LAUNCH_CHECK();
    size_t need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, c->keys.p, keys_sorted, (int)n, 0, 64, s);
    IBF_TRY(c->cub_tmp.reserve(need + 16));
    size_t have = c->cub_tmp.cap;
    IBF_CUDA(cub::DeviceRadixSort::SortKeys(c->cub_tmp.p, have, c->keys.p, keys_sorted, (int)n, 0, 64, s));
    if (n > 1) {
      k_build<<<grid_for(n - 1), 256, 0, s>>>((int)n, keys_sorted, left, right, parent, last, tfirst);
      IBF_LAUNCH_CHECK();
      if (tfirst) {
        IBF_CUDA(cudaMemsetAsync(tcounts, 0, 2 * sizeof(int), s));
        IBF_CUDA(cudaMemsetAsync(tucode, 0, n, s));
        IBF_CUDA(cudaMemsetAsync(troot, 0, n - 1, s));
        k_treelet_lists<<<grid_for(2 * n - 1), 256, 0, s>>>((int)n, tfirst, last, parent, kS, tucode, troot,
                                                             titems, tcounts);
        IBF_LAUNCH_CHECK();
        k_chunk_starts<<<grid_for(nchunks + 1), 256, 0, s>>>((int)n, kT, nchunks, tucode, tchunk);
        IBF_LAUNCH_CHECK();
      }
      if (odd) {
        k_depth_parity<<<grid_for(n - 1), 256, 0, s>>>((int)n, parent, odd);
        IBF_LAUNCH_CHECK();
      }
      if (lbox && prims) {
        k_leaf_ids<<<grid_for(n), 256, 0, s>>>((int)n, keys_sorted, prims, arity, lbox);
        IBF_LAUNCH_CHECK();
      }
    }
    if (cache) {
      cache->n = n;
      cache->uses = 0;
    }
  }
  if (cache) ++cache->uses;
  IBF_CUDA(cudaMemsetAsync(flag, 0, nn * sizeof(int), s));
  // algorithmic: per leaf the FP64 box and key in, the exact leaf record
  // out; per internal node one 64-byte record out
  {
  KernelClock kcr(KC_REFIT, s, (packed && n > 1) ? 96.0 * n + 64.0 * (n - 1) : 0.0, 0.0, (double)n);
  if (packed && n > 1 && tfirst) {
    if (refit_chunk_smem(kCap) > 48 * 1024) {
      static std::once_flag smem_once;
      std::call_once(smem_once, [] {
        cudaFuncSetAttribute(k_refit_chunks<kCap>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)refit_chunk_smem(kCap));
      });
    }
    k_refit_chunks<kCap><<<nchunks, kCap, refit_chunk_smem(kCap), s>>>(
        (int)n, keys_sorted, c->box_lo.p, c->box_hi.p, left, right, parent, last, tchunk, tucode, troot, packed,
        prims ? lbox : nullptr);
    IBF_LAUNCH_CHECK();
    k_refit_top<<<148 * 2, 256, 0, s>>>((int)n, left, right, parent, last, titems, tcounts, flag, packed);
  } else if (packed && n > 1) {
    k_refit_packed<<<grid_for(n), 256, 0, s>>>((int)n, keys_sorted, c->box_lo.p, c->box_hi.p, left, right, parent,
                                                last, flag, packed, prims ? lbox : nullptr);
  } else {
    if (cache && IBF_CCD_PACKED) {
      IBF_TRY(cache->lo.reserve(3 * nn));
      IBF_TRY(cache->hi.reserve(3 * nn));
      lo = cache->lo.p, hi = cache->hi.p;
    }
    k_refit<<<grid_for(n), 256, 0, s>>>((int)n, keys_sorted, c->box_lo.p, c->box_hi.p, left, right, parent, flag,
                                         lo, hi, nullptr);
  }
  IBF_LAUNCH_CHECK();
  }
  if (wide && packed && n > 1) {
    k_widen<<<grid_for(n - 1), 256, 0, s>>>((int)n, odd, packed, wide);
    IBF_LAUNCH_CHECK();
  }
  t.wide = (packed && n > 1) ? wide : nullptr;
  t.lbox = (packed && n > 1 && prims) ? lbox : nullptr;
  t.packed = n > 1 ? packed : nullptr;
  t.plo = c->box_lo.p;
  t.phi = c->box_hi.p;
  t.n = (int)n;
  t.keys = keys_sorted;
  t.left = left;
  t.right = right;
  t.lo = lo;
  t.hi = hi;
  return IBF_OK;
}

// One broad-phase pass (VF or EE): boxes, tree, traversal with optional
// prefilter, sort.  Result pairs in c->pairs_sorted[0..count).
static int broad_pass(ibf_ccd* c, int kind, const double* x0, const double* x1, double min_gap, bool filter,
                      int64_t* count, int64_t* n_candidates, cudaStream_t s) {
  Trace tr(kind == 0 ? "broad_pass VF" : (kind == 1 ? "broad_pass EE" : "broad_pass TT"));
  tr.mark("enter", s);
  const int64_t nt = (kind == 1) ? c->ne : c->nt;
  const int64_t nq = (kind == 0) ? c->nv : ((kind == 1) ? c->ne : c->nt);
  *count = 0;
  *n_candidates = 0;
  if (nt == 0 || nq == 0) return IBF_OK;
  IBF_TRY(c->box_lo.reserve(3 * nt));
  IBF_TRY(c->box_hi.reserve(3 * nt));
  IBF_TRY(c->qlo.reserve(3 * nq));
  IBF_TRY(c->qhi.reserve(3 * nq));
  if (kind == 2) {
    // static triangle boxes (intact/intersect.py:129-131), queried against themselves
    k_swept_boxes<3><<<grid_for(nt), 256, 0, s>>>(nt, c->tris.p, x0, x1, 0.0, c->box_lo.p, c->box_hi.p);
    IBF_LAUNCH_CHECK();
  } else if (kind == 0) {
    k_swept_boxes<3><<<grid_for(nt), 256, 0, s>>>(nt, c->tris.p, x0, x1, min_gap, c->box_lo.p, c->box_hi.p);
    IBF_LAUNCH_CHECK();
    k_swept_boxes<1><<<grid_for(nq), 256, 0, s>>>(nq, c->verts.p, x0, x1, 0.0, c->qlo.p, c->qhi.p);
    IBF_LAUNCH_CHECK();
  } else {
    k_swept_boxes<2><<<grid_for(nt), 256, 0, s>>>(nt, c->edges.p, x0, x1, 0.5 * min_gap, c->box_lo.p, c->box_hi.p);
    IBF_LAUNCH_CHECK();
  }
  tr.mark("boxes", s, nt);
  Tree tree;
  IBF_TRY(build_tree(c, nt, s, tree, (kind < 2 && IBF_CCD_REBUILD > 1) ? &c->tc[kind] : nullptr,
                     kind == 1 ? c->edges.p : c->tris.p, kind == 1 ? 2 : 3));
  tr.mark("tree", s);
  // VF queries (surface vertices) in Morton order of their boxes, so the 32
  // walks of a warp follow nearly the same path (EE and TT self-queries use
  // the tree's own sorted keys); recomputed when the triangle tree is rebuilt
  const unsigned long long* qorder = (kind == 0) ? nullptr : tree.keys;
  if (kind == 0 && IBF_CCD_VF_ORDER) {
    const bool fresh = !(IBF_CCD_REBUILD > 1) || c->tc[0].uses == 1 || c->vf_order_n != nq;
    if (fresh) {
      const int nparts = (int)std::min<int64_t>(grid_for(nq), 148 * 2);
      IBF_TRY(c->dscratch.reserve(6 * (size_t)nparts + 8));
      IBF_TRY(c->keys.reserve(nq));
      IBF_TRY(c->vf_order.reserve(nq));
      k_bounds<<<nparts, 256, 0, s>>>(nq, c->qlo.p, c->qhi.p, c->dscratch.p);
      IBF_LAUNCH_CHECK();
      k_morton<<<grid_for(nq), 256, 0, s>>>(nq, c->qlo.p, c->qhi.p, c->dscratch.p, nparts, c->keys.p);
      IBF_LAUNCH_CHECK();
      size_t need = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, need, c->keys.p, c->vf_order.p, (int)nq, 0, 64, s);
      IBF_TRY(c->cub_tmp.reserve(need + 16));
      size_t have = c->cub_tmp.cap;
      IBF_CUDA(cub::DeviceRadixSort::SortKeys(c->cub_tmp.p, have, c->keys.p, c->vf_order.p, (int)nq, 0, 64, s));
      c->vf_order_n = nq;
    }
    qorder = c->vf_order.p;
  }
  IBF_TRY(c->counters.reserve(4));
  IBF_TRY(c->host.reserve(64));
  if (c->pairs.cap < 4096) IBF_TRY(c->pairs.reserve(1 << 16));
  const bool split = filter && IBF_CCD_SPLIT;
  TraverseArgs a;
  for (int attempt = 0; attempt < 3; ++attempt) {
    IBF_CUDA(cudaMemsetAsync(c->counters.p, 0, 2 * sizeof(unsigned long long), s));
    IBF_CUDA(cudaMemsetAsync(c->counters.p + 3, 0, sizeof(unsigned long long), s));
    a.tree = tree;
    a.qorder = qorder;
    a.nq = nq;
    // self-queries (EE, TT) read the tree's own primitive boxes
    a.qlo = kind == 0 ? c->qlo.p : c->box_lo.p;
    a.qhi = kind == 0 ? c->qhi.p : c->box_hi.p;
    a.kind = kind;
    a.qprim = (kind == 0) ? c->verts.p : ((kind == 1) ? c->edges.p : c->tris.p);
    a.tprim = (kind == 1) ? c->edges.p : c->tris.p;
    a.x0 = x0;
    a.x1 = x1;
    a.min_gap = min_gap;
    a.filter = (filter && !split) ? 1 : 0;
    a.exact_leaf = (split && IBF_CCD_DEFER_EXACT) ? 0 : 1;
    a.out = c->pairs.p;
    a.cap = c->pairs.cap;
    a.counters = c->counters.p;
    unsigned long long* h = (unsigned long long*)c->host.p;
    {
      // algorithmic: 48 B per query box + 48 B per primitive box (each leaf
      // read once) + 16 B per candidate pair out (booked after the count)
      KernelClock kc(KC_TRAVERSE, s, 48.0 * (nq + tree.n), 0.0, 0.0);
      const bool packed = tree.packed != nullptr;
      if (packed && IBF_CCD_DYNAMIC) {
        // self-queries walk the tree's own leaves in sorted order
        const bool self = kind != 0 && a.qorder == tree.keys;
        auto kern = a.filter ? (self ? k_traverse_dyn<true, true> : k_traverse_dyn<true, false>)
                             : (self ? k_traverse_dyn<false, true> : k_traverse_dyn<false, false>);
        if (tree.wide)
          kern = a.filter ? (self ? k_traverse_wide<true, true> : k_traverse_wide<true, false>)
                          : (self ? k_traverse_wide<false, true> : k_traverse_wide<false, false>);
        int blocks_per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, 128, 0);
        blocks_per_sm = std::max(blocks_per_sm, 1);
        const int64_t want = div_up(nq, 128);
        kern<<<(int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)blocks_per_sm * sm_count())), 128, 0, s>>>(a);
      } else {
        auto kern = a.filter ? (packed ? k_traverse<true, true> : k_traverse<true, false>)
                             : (packed ? k_traverse<false, true> : k_traverse<false, false>);
        kern<<<grid_for(nq, 128), 128, 0, s>>>(a);
      }
      IBF_LAUNCH_CHECK();
      IBF_CUDA(cudaMemcpyAsync(h, c->counters.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
      IBF_CUDA(cudaStreamSynchronize(s));
      kc.bytes += 16.0 * (double)h[1];
      kc.units = (double)h[1];
    }
    *count = (int64_t)h[0];
    *n_candidates = (int64_t)h[1];
    if (h[0] <= c->pairs.cap) break;
    if (h[0] > (1ull << 30)) {
      set_error("broad phase: " + std::to_string(h[0]) + " pairs need narrow-phase work (" +
                std::to_string(h[1]) + " candidates for " + std::to_string(nq) +
                " queries): the step's motion is unbounded");
      return IBF_ERR_OOM;
    }
    IBF_TRY(c->pairs.reserve((size_t)h[0]));
  }
  tr.mark("traverse", s, *n_candidates);
  const unsigned long long* unsorted = c->pairs.p;
  if (split && *count) {
    const int64_t n_all = *count;
    IBF_TRY(c->pairs2.reserve(n_all));
    IBF_CUDA(cudaMemsetAsync(c->counters.p, 0, (a.exact_leaf ? 1 : 2) * sizeof(unsigned long long), s));
    a.out = c->pairs2.p;
    a.cap = c->pairs2.cap;
    unsigned long long* h = (unsigned long long*)c->host.p;
    {
      // algorithmic: 8 B per candidate in, 8 vertices x 24 B gathered, 8 B per survivor out
      KernelClock kc(KC_PREFILTER, s, 200.0 * (double)n_all, 0.0, (double)n_all);
      k_prefilter<<<grid_for(n_all, 256), 256, 0, s>>>(a, n_all, c->pairs.p);
      IBF_LAUNCH_CHECK();
      IBF_CUDA(cudaMemcpyAsync(h, c->counters.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
      IBF_CUDA(cudaStreamSynchronize(s));
      kc.bytes += 8.0 * (double)h[0];
    }
    *count = (int64_t)h[0];
    if (!a.exact_leaf) *n_candidates = (int64_t)h[1];   // the exact candidates (the walk counted float overlaps)
    unsorted = c->pairs2.p;
    tr.mark("prefilter", s, *count);
  }
  const int64_t cnt = *count;
  IBF_TRY(c->pairs_sorted.reserve(std::max<int64_t>(cnt, 1)));
  if (cnt) {
    size_t need = 0;
    // keys are (query << 32) | primitive, query < nq: only the bits that can be set
    int end_bit = 32;
    while (end_bit < 64 && (1LL << (end_bit - 32)) < nq) ++end_bit;
    cub::DeviceRadixSort::SortKeys(nullptr, need, unsorted, c->pairs_sorted.p, (int)cnt, 0, end_bit, s);
    IBF_TRY(c->cub_tmp.reserve(need + 16));
    size_t have = c->cub_tmp.cap;
    IBF_CUDA(cub::DeviceRadixSort::SortKeys(c->cub_tmp.p, have, unsorted, c->pairs_sorted.p, (int)cnt, 0, end_bit, s));
  }
  tr.mark("sort", s, cnt);
  tr.mark("exit", s);
  return IBF_OK;
}

}  // namespace ibf

using namespace ibf;

extern "C" int ibf_pair_eval(int kind, int64_t n, const double* pts, double* d, double* grad, double* weights,
                             uint8_t* degenerate, ibf_stream s) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)s);
  if (kind != 0 && kind != 1) {
    set_error("ibf_pair_eval: kind must be 0 (VF) or 1 (EE)");
    return IBF_ERR_BAD_ARG;
  }
  if (n <= 0) return IBF_OK;
  k_pair_eval<<<grid_for(n), 256, 0, (cudaStream_t)s>>>(kind, n, pts, d, grad, weights, degenerate);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

extern "C" int ibf_accd(int kind, int64_t n, const double* x0, const double* x1, double min_gap, double* toi,
                        ibf_stream s) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)s);
  if (kind != 0 && kind != 1) {
    set_error("ibf_accd: kind must be 0 (VF) or 1 (EE)");
    return IBF_ERR_BAD_ARG;
  }
  if (n <= 0) return IBF_OK;
  k_accd_batch<<<grid_for(n), 128, 0, (cudaStream_t)s>>>(kind, n, x0, x1, min_gap, toi);
  IBF_LAUNCH_CHECK();
  return IBF_OK;
}

extern "C" int ibf_ccd_create(int64_t n_tris, const int64_t* tris, int64_t n_edges, const int64_t* edges,
                              int64_t n_verts, const int64_t* verts, ibf_ccd** out) {
  if (n_tris < 0 || n_edges < 0 || n_verts < 0 || !out || n_tris >= (1LL << 31) || n_edges >= (1LL << 31)) {
    set_error("ibf_ccd_create: bad arguments");
    return IBF_ERR_BAD_ARG;
  }
  ibf_ccd* c = new ibf_ccd();
  c->nt = n_tris;
  c->ne = n_edges;
  c->nv = n_verts;
  std::vector<int> t(3 * n_tris), e(2 * n_edges), v(n_verts);
  for (int64_t k = 0; k < 3 * n_tris; ++k) t[k] = (int)tris[k];
  for (int64_t k = 0; k < 2 * n_edges; ++k) e[k] = (int)edges[k];
  for (int64_t k = 0; k < n_verts; ++k) v[k] = (int)verts[k];
  int st = c->tris.upload(t.data(), t.size());
  if (st == IBF_OK) st = c->edges.upload(e.data(), e.size());
  if (st == IBF_OK) st = c->verts.upload(v.data(), v.size());
  if (st == IBF_OK && cudaDeviceSynchronize() != cudaSuccess) st = IBF_ERR_CUDA;
  if (st != IBF_OK) {
    delete c;
    return st;
  }
  *out = c;
  return IBF_OK;
}

extern "C" void ibf_ccd_destroy(ibf_ccd* c) { delete c; }

// stored candidate quads (for ibf_ccd_get_candidates): reuse b_quad storage
static ibf::DevBuf<int>& cand_store(ibf_ccd* c) { return c->b_pos; }

extern "C" int ibf_ccd_candidates(ibf_ccd* c, const double* x0, const double* x1, double min_gap, int64_t* n_vf,
                                  int64_t* n_ee, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  int64_t cnt_vf = 0, cnt_ee = 0, all = 0;
  IBF_TRY(broad_pass(c, 0, x0, x1, min_gap, false, &cnt_vf, &all, s));
  DevBuf<int>& store = cand_store(c);
  IBF_TRY(store.reserve(4 * std::max<int64_t>(cnt_vf, 1)));
  if (cnt_vf) {
    k_pair_toi<<<grid_for(cnt_vf), 256, 0, s>>>(cnt_vf, 0, c->pairs_sorted.p, c->verts.p, c->tris.p, x0, x1, 0.0,
                                                 nullptr, store.p);
    IBF_LAUNCH_CHECK();
  }
  // keep VF quads aside while EE runs
  std::vector<int> vf_host(4 * cnt_vf);
  if (cnt_vf)
    IBF_CUDA(cudaMemcpyAsync(vf_host.data(), store.p, 4 * cnt_vf * sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_TRY(broad_pass(c, 1, x0, x1, min_gap, false, &cnt_ee, &all, s));
  IBF_TRY(store.reserve(4 * std::max<int64_t>(cnt_vf + cnt_ee, 1)));
  IBF_CUDA(cudaStreamSynchronize(s));
  if (cnt_vf) IBF_CUDA(cudaMemcpyAsync(store.p, vf_host.data(), 4 * cnt_vf * sizeof(int), cudaMemcpyHostToDevice, s));
  if (cnt_ee) {
    k_pair_toi<<<grid_for(cnt_ee), 256, 0, s>>>(cnt_ee, 1, c->pairs_sorted.p, c->edges.p, c->edges.p, x0, x1, 0.0,
                                                 nullptr, store.p + 4 * cnt_vf);
    IBF_LAUNCH_CHECK();
  }
  IBF_CUDA(cudaStreamSynchronize(s));
  c->n_vf = cnt_vf;
  c->n_ee = cnt_ee;
  *n_vf = cnt_vf;
  *n_ee = cnt_ee;
  return IBF_OK;
}

extern "C" int ibf_ccd_get_candidates(ibf_ccd* c, int64_t* vf_host, int64_t* ee_host, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  const int64_t tot = c->n_vf + c->n_ee;
  std::vector<int> q(4 * tot);
  if (tot) IBF_CUDA(cudaMemcpyAsync(q.data(), cand_store(c).p, 4 * tot * sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  for (int64_t k = 0; k < 4 * c->n_vf; ++k) vf_host[k] = q[k];
  for (int64_t k = 0; k < 4 * c->n_ee; ++k) ee_host[k] = q[4 * c->n_vf + k];
  return IBF_OK;
}

extern "C" int ibf_max_step_size(ibf_ccd* c, const double* x, const double* x_hat, double min_gap, double cap,
                                 double* alpha_host, int64_t* n_blocking_host, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  IBF_TRY(c->dscratch.reserve(8));
  IBF_TRY(c->host.reserve(64));
  c->t_ccd.begin(s);
  // survivors of both passes, kept in separate regions of b_* scratch
  int64_t cnt[2] = {0, 0}, all[2] = {0, 0};
  DevBuf<int>* quads = c->s_quad;
  DevBuf<double>* tois = c->s_toi;
  for (int kind = 0; kind < 2; ++kind) {
    IBF_TRY(broad_pass(c, kind, x, x_hat, min_gap, true, &cnt[kind], &all[kind], s));
    c->n_candidates += all[kind];
    if (cnt[kind]) {
      IBF_TRY(quads[kind].reserve(4 * cnt[kind]));
      IBF_TRY(tois[kind].reserve(cnt[kind]));
      // algorithmic: 4 vertices x (x, x_hat) 192 B + quad 16 B in, TOI 8 B out per pair
      KernelClock kc(KC_TOI, s, 216.0 * cnt[kind], 0.0, (double)cnt[kind]);
      k_pair_toi<<<grid_for(cnt[kind], 128), 128, 0, s>>>(
          cnt[kind], kind, c->pairs_sorted.p, kind == 0 ? c->verts.p : c->edges.p, kind == 0 ? c->tris.p : c->edges.p,
          x, x_hat, min_gap, tois[kind].p, quads[kind].p);
      IBF_LAUNCH_CHECK();
    }
  }
  // alpha = min(cap, min TOI over all candidates); non-survivors have TOI 1
  double base = cap;
  if ((all[0] + all[1]) > 0) base = std::min(base, 1.0);
  k_set<<<1, 1, 0, s>>>(c->dscratch.p, INFINITY);
  for (int kind = 0; kind < 2; ++kind)
    if (cnt[kind]) {
      k_min_toi<<<grid_for(cnt[kind]), 256, 0, s>>>(cnt[kind], tois[kind].p, c->dscratch.p);
      IBF_LAUNCH_CHECK();
    }
  // blocking pairs (TOI < 1), VF first then EE, sorted order within kind
  const int64_t tot = cnt[0] + cnt[1];
  IBF_TRY(c->b_kind.reserve(std::max<int64_t>(tot, 1)));
  IBF_TRY(c->b_quad.reserve(4 * std::max<int64_t>(tot, 1)));
  IBF_TRY(c->b_toi.reserve(std::max<int64_t>(tot, 1)));
  IBF_TRY(c->b_flag.reserve(tot + 2));
  DevBuf<int>& pos = c->s_pos;
  IBF_TRY(pos.reserve(tot + 2));
  int* hcount = (int*)c->host.p;
  int64_t nblock = 0;
  for (int kind = 0; kind < 2; ++kind) {
    const int64_t n = cnt[kind];
    if (!n) continue;
    k_block_flag<<<grid_for(n), 256, 0, s>>>(n, tois[kind].p, c->b_flag.p);
    IBF_LAUNCH_CHECK();
    IBF_CUDA(cudaMemsetAsync(c->b_flag.p + n, 0, sizeof(int), s));
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, c->b_flag.p, pos.p, (int)(n + 1), s);
    IBF_TRY(c->cub_tmp.reserve(need + 16));
    size_t have = c->cub_tmp.cap;
    IBF_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, have, c->b_flag.p, pos.p, (int)(n + 1), s));
    k_block_write<<<grid_for(n), 256, 0, s>>>(n, nblock, kind, c->b_flag.p, pos.p, quads[kind].p, tois[kind].p,
                                              c->b_kind.p, c->b_quad.p, c->b_toi.p);
    IBF_LAUNCH_CHECK();
    IBF_CUDA(cudaMemcpyAsync(hcount, pos.p + n, sizeof(int), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaStreamSynchronize(s));
    nblock += hcount[0];
  }
  double mt = INFINITY;
  IBF_CUDA(cudaMemcpyAsync(&mt, c->dscratch.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  c->t_ccd.end(s);
  IBF_CUDA(cudaStreamSynchronize(s));
  c->t_ccd.harvest();
  *alpha_host = std::min(base, mt);
  c->n_block = nblock;
  *n_blocking_host = nblock;
  return IBF_OK;
}

extern "C" int ibf_ccd_blocking(ibf_ccd* c, const int32_t** kinds, const int32_t** quads, const double** tois,
                                int64_t* n) {
  *kinds = c->b_kind.p;
  *quads = c->b_quad.p;
  *tois = c->b_toi.p;
  *n = c->n_block;
  return IBF_OK;
}

extern "C" int ibf_ccd_get_blocking(ibf_ccd* c, int64_t* kinds, int64_t* quads, double* tois, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  const int64_t n = c->n_block;
  if (!n) return IBF_OK;
  std::vector<int> k(n), q(4 * n);
  IBF_CUDA(cudaMemcpyAsync(k.data(), c->b_kind.p, n * sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(q.data(), c->b_quad.p, 4 * n * sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaMemcpyAsync(tois, c->b_toi.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  for (int64_t j = 0; j < n; ++j) {
    kinds[j] = k[j];
    for (int e = 0; e < 4; ++e) quads[4 * j + e] = q[4 * j + e];
  }
  return IBF_OK;
}

// ===================================================== penetration monitor
// GPU restatement of the reference's validation oracle (intact/intersect.py,
// SURVEY.md §8(f) f1) plus a nearest-pair monitor: certifies "penetration
// free" at C4 scale, where the numpy test is a Python loop.

namespace ibf {
namespace mon {

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 ld(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ D3 sub(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot(D3 a, D3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ D3 cross(D3 a, D3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double nrm(D3 a) { return sqrt(dot(a, a)); }

// inclusive segment pq vs triangle abc; coplanar segments miss (intersect.py:21-46)
__device__ bool segment_hits(D3 p, D3 q, D3 a, D3 b, D3 c) {
  const double eps = 1e-12;
  const D3 d = sub(q, p), e1 = sub(b, a), e2 = sub(c, a);
  const D3 h = cross(d, e2);
  const double det = dot(e1, h);
  const double scale = nrm(d) * nrm(e1) * nrm(e2);
  if (!(fabs(det) > eps * fmax(scale, 1e-300))) return false;
  const double f = 1.0 / det;
  const D3 s = sub(p, a);
  const double u = f * dot(s, h);
  const D3 qv = cross(s, e1);
  const double v = f * dot(d, qv);
  const double t = f * dot(e2, qv);
  return u >= -eps && v >= -eps && u + v <= 1.0 + eps && t >= -eps && t <= 1.0 + eps;
}

// all of T2's vertices strictly on one side of T1's plane (intersect.py:95-101)
__device__ bool one_side(const D3 T1[3], const D3 T2[3]) {
  const D3 n = cross(sub(T1[1], T1[0]), sub(T1[2], T1[0]));
  double amax = 0.0;
  for (int k = 0; k < 3; ++k) amax = fmax(amax, fmax(fabs(T2[k].x), fmax(fabs(T2[k].y), fabs(T2[k].z))));
  const double tol = 1e-12 * nrm(n) * (1.0 + amax);
  bool pos = true, neg = true;
  for (int k = 0; k < 3; ++k) {
    const double d = dot(sub(T2[k], T1[0]), n);
    pos = pos && d > tol;
    neg = neg && d < -tol;
  }
  return pos || neg;
}

__device__ bool coplanar_overlap(const D3 A3[3], const D3 B3[3]) {
  const D3 n = cross(sub(A3[1], A3[0]), sub(A3[2], A3[0]));
  const double an[3] = {fabs(n.x), fabs(n.y), fabs(n.z)};
  const int drop = (an[0] >= an[1] && an[0] >= an[2]) ? 0 : (an[1] >= an[2] ? 1 : 2);
  double A[3][2], B[3][2];
  for (int k = 0; k < 3; ++k) {
    const double va[3] = {A3[k].x, A3[k].y, A3[k].z}, vb[3] = {B3[k].x, B3[k].y, B3[k].z};
    int m = 0;
    for (int c = 0; c < 3; ++c)
      if (c != drop) {
        A[k][m] = va[c];
        B[k][m] = vb[c];
        ++m;
      }
  }
  auto crosses = [](const double* p, const double* q, const double* r, const double* s) {
    const double d1x = q[0] - p[0], d1y = q[1] - p[1], d2x = s[0] - r[0], d2y = s[1] - r[1];
    const double den = d1x * d2y - d1y * d2x;
    if (fabs(den) < 1e-300) return false;
    const double t = ((r[0] - p[0]) * d2y - (r[1] - p[1]) * d2x) / den;
    const double u = ((r[0] - p[0]) * d1y - (r[1] - p[1]) * d1x) / den;
    return -1e-12 <= t && t <= 1.0 + 1e-12 && -1e-12 <= u && u <= 1.0 + 1e-12;
  };
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (crosses(A[i], A[(i + 1) % 3], B[j], B[(j + 1) % 3])) return true;
  auto inside = [](const double* pt, double T[3][2]) {
    double sign = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double ex = T[(k + 1) % 3][0] - T[k][0], ey = T[(k + 1) % 3][1] - T[k][1];
      const double wx = pt[0] - T[k][0], wy = pt[1] - T[k][1];
      const double cr = ex * wy - ey * wx;
      if (sign == 0.0) sign = cr;
      else if (cr * sign < 0.0) return false;
    }
    return true;
  };
  return inside(A[0], B) || inside(B[0], A);
}

// intact/intersect.py:85-122 for one pair
__device__ bool tri_tri(const D3 A[3], const D3 B[3]) {
  if (one_side(A, B) || one_side(B, A)) return false;
  for (int i = 0; i < 3; ++i) {
    if (segment_hits(A[i], A[(i + 1) % 3], B[0], B[1], B[2])) return true;
    if (segment_hits(B[i], B[(i + 1) % 3], A[0], A[1], A[2])) return true;
  }
  const D3 n = cross(sub(A[1], A[0]), sub(A[2], A[0]));
  const double nn = nrm(n);
  if (nn < 1e-300) return false;
  double dmax = 0.0, span = 1.0;
  for (int k = 0; k < 3; ++k) {
    dmax = fmax(dmax, fabs(dot(sub(B[k], A[0]), n)) / nn);
    span = fmax(span, fmax(fmax(fabs(A[k].x), fabs(A[k].y)), fabs(A[k].z)));
    span = fmax(span, fmax(fmax(fabs(B[k].x), fabs(B[k].y)), fabs(B[k].z)));
  }
  return dmax < 1e-9 * span && coplanar_overlap(A, B);
}

}  // namespace mon

__global__ void k_tri_tri(int64_t n, const unsigned long long* __restrict__ pairs, const int* __restrict__ tris,
                          const double* __restrict__ x, int* __restrict__ hit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(pairs[i] >> 32), b = (int)(pairs[i] & 0xffffffffull);
    mon::D3 A[3], B[3];
    for (int k = 0; k < 3; ++k) {
      A[k] = mon::ld(x + 3 * (int64_t)tris[3 * a + k]);
      B[k] = mon::ld(x + 3 * (int64_t)tris[3 * b + k]);
    }
    hit[i] = mon::tri_tri(A, B) ? 1 : 0;
  }
}

__global__ void k_hit_write(int64_t n, const unsigned long long* __restrict__ pairs, const int* __restrict__ hit,
                            const int* __restrict__ pos, int64_t cap, long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!hit[i] || pos[i] >= cap) continue;
    out[2 * (int64_t)pos[i]] = (long long)(pairs[i] >> 32);
    out[2 * (int64_t)pos[i] + 1] = (long long)(pairs[i] & 0xffffffffull);
  }
}

// distances of broad-phase pairs; min via ordered bits (distances >= 0)
__global__ void k_pair_min_dist(int64_t n, int kind, const unsigned long long* __restrict__ pairs,
                                const int* __restrict__ qprim, const int* __restrict__ tprim,
                                const double* __restrict__ x, double* __restrict__ dist, double* __restrict__ dmin) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int qi = (int)(pairs[i] >> 32), pi = (int)(pairs[i] & 0xffffffffull);
    int q[4];
    if (kind == 0) {
      q[0] = qprim[qi]; q[1] = tprim[3 * pi]; q[2] = tprim[3 * pi + 1]; q[3] = tprim[3 * pi + 2];
    } else {
      q[0] = qprim[2 * qi]; q[1] = qprim[2 * qi + 1]; q[2] = tprim[2 * pi]; q[3] = tprim[2 * pi + 1];
    }
    V3 P[4];
    for (int k = 0; k < 4; ++k) P[k] = geo::ld3(x + 3 * (int64_t)q[k]);
    const double d = geo::pair_dist(kind, P);
    dist[i] = d;
    if (d == d) atomic_min_nonneg(dmin, d);
  }
}

__global__ void k_find_dist(int64_t n, const double* __restrict__ dist, const double* __restrict__ dmin,
                            unsigned long long* __restrict__ first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (dist[i] == *dmin) atomicMin(first, (unsigned long long)i);
}

}  // namespace ibf

extern "C" int ibf_static_intersection(ibf_ccd* c, const double* x, int64_t* n_hits, int64_t* pairs_host,
                                       int64_t cap, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  int64_t cnt = 0, all = 0;
  *n_hits = 0;
  IBF_TRY(broad_pass(c, 2, x, x, 0.0, false, &cnt, &all, s));
  if (!cnt) return IBF_OK;
  IBF_TRY(c->b_flag.reserve(cnt + 1));
  IBF_TRY(c->s_pos.reserve(cnt + 1));
  k_tri_tri<<<grid_for(cnt), 256, 0, s>>>(cnt, c->pairs_sorted.p, c->tris.p, x, c->b_flag.p);
  IBF_LAUNCH_CHECK();
  IBF_CUDA(cudaMemsetAsync(c->b_flag.p + cnt, 0, sizeof(int), s));
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, c->b_flag.p, c->s_pos.p, (int)(cnt + 1), s);
  IBF_TRY(c->cub_tmp.reserve(need + 16));
  size_t have = c->cub_tmp.cap;
  IBF_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, have, c->b_flag.p, c->s_pos.p, (int)(cnt + 1), s));
  int* h = (int*)c->host.p;
  IBF_CUDA(cudaMemcpyAsync(h, c->s_pos.p + cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  *n_hits = h[0];
  if (pairs_host && cap > 0 && h[0] > 0) {
    const int64_t k = std::min<int64_t>(cap, h[0]);
    DevBuf<long long> out;
    IBF_TRY(out.reserve(2 * k));
    k_hit_write<<<grid_for(cnt), 256, 0, s>>>(cnt, c->pairs_sorted.p, c->b_flag.p, c->s_pos.p, k, out.p);
    IBF_LAUNCH_CHECK();
    IBF_CUDA(cudaMemcpyAsync(pairs_host, out.p, 2 * k * sizeof(long long), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaStreamSynchronize(s));
  }
  return IBF_OK;
}

extern "C" int ibf_min_distance(ibf_ccd* c, const double* x, double radius, double* d_host, int64_t* pair_host,
                                ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  cudaStream_t s = (cudaStream_t)st;
  *d_host = INFINITY;
  if (pair_host)
    for (int k = 0; k < 5; ++k) pair_host[k] = -1;
  IBF_TRY(c->dscratch.reserve(8));
  IBF_TRY(c->counters.reserve(4));
  for (int kind = 0; kind < 2; ++kind) {
    int64_t cnt = 0, all = 0;
    IBF_TRY(broad_pass(c, kind, x, x, radius, false, &cnt, &all, s));
    if (!cnt) continue;
    IBF_TRY(c->pair_toi.reserve(cnt));
    k_set<<<1, 1, 0, s>>>(c->dscratch.p, INFINITY);
    IBF_LAUNCH_CHECK();
    const int* qprim = kind == 0 ? c->verts.p : c->edges.p;
    const int* tprim = kind == 0 ? c->tris.p : c->edges.p;
    k_pair_min_dist<<<grid_for(cnt), 256, 0, s>>>(cnt, kind, c->pairs_sorted.p, qprim, tprim, x, c->pair_toi.p,
                                                   c->dscratch.p);
    IBF_LAUNCH_CHECK();
    IBF_CUDA(cudaMemsetAsync(c->counters.p + 2, 0xff, sizeof(unsigned long long), s));
    k_find_dist<<<grid_for(cnt), 256, 0, s>>>(cnt, c->pair_toi.p, c->dscratch.p, c->counters.p + 2);
    IBF_LAUNCH_CHECK();
    double dm = INFINITY;
    unsigned long long idx = ~0ull, pr = 0;
    IBF_CUDA(cudaMemcpyAsync(&dm, c->dscratch.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaMemcpyAsync(&idx, c->counters.p + 2, sizeof(idx), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaStreamSynchronize(s));
    if (dm < *d_host && idx != ~0ull) {
      *d_host = dm;
      IBF_CUDA(cudaMemcpy(&pr, c->pairs_sorted.p + idx, sizeof(pr), cudaMemcpyDeviceToHost));
      if (pair_host) {
        const int qi = (int)(pr >> 32), pi = (int)(pr & 0xffffffffull);
        std::vector<int> qv(3), pv(3);
        if (kind == 0) {
          IBF_CUDA(cudaMemcpy(qv.data(), c->verts.p + qi, sizeof(int), cudaMemcpyDeviceToHost));
          IBF_CUDA(cudaMemcpy(pv.data(), c->tris.p + 3 * pi, 3 * sizeof(int), cudaMemcpyDeviceToHost));
          pair_host[1] = qv[0]; pair_host[2] = pv[0]; pair_host[3] = pv[1]; pair_host[4] = pv[2];
        } else {
          IBF_CUDA(cudaMemcpy(qv.data(), c->edges.p + 2 * qi, 2 * sizeof(int), cudaMemcpyDeviceToHost));
          IBF_CUDA(cudaMemcpy(pv.data(), c->edges.p + 2 * pi, 2 * sizeof(int), cudaMemcpyDeviceToHost));
          pair_host[1] = qv[0]; pair_host[2] = qv[1]; pair_host[3] = pv[0]; pair_host[4] = pv[1];
        }
        pair_host[0] = kind;
      }
    }
  }
  return IBF_OK;
}

namespace ibf {
int contacts_update_dev(ibf_contacts* c, int64_t nb, const int* bkind, const int* bquad, const double* btoi,
                        int64_t* admitted, int64_t* pruned, cudaStream_t s);
}

extern "C" int ibf_contacts_update(ibf_contacts* c, const ibf_ccd* blocking, int64_t* admitted, int64_t* pruned,
                                   ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  const int64_t nb = blocking ? blocking->n_block : 0;
  return contacts_update_dev(c, nb, nb ? blocking->b_kind.p : nullptr, nb ? blocking->b_quad.p : nullptr,
                             nb ? blocking->b_toi.p : nullptr, admitted, pruned, (cudaStream_t)st);
}
