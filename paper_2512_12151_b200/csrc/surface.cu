// Boundary surface of a tet mesh on the device.
//
// Replaces extract_surface_arrays (intact/mesh.py:106-124): a face is on the
// boundary iff its sorted vertex triple occurs once over all 4M tet faces;
// the boundary keeps the tets' face order and winding, the edges are the
// unique sorted (lo, hi) pairs of the boundary triangles in lexicographic
// order, and the vertices are the unique ids in ascending order — the three
// outputs of the reference, bit-exactly.
//
// Layout: faces f = 4 t + r (r = face opposite vertex r, intact/mesh.py
// _TET_FACES).  Triples are ordered by two stable radix passes, (b, c) as
// one 64-bit key and then a, so vertex ids may use the full int32 range.
// Edges sort as 64-bit (lo << 32 | hi) keys and are run-length encoded, which
// also gives the non-manifold count (edges on > 2 boundary faces) that the
// reference logs.  Integer work only: HBM-bound sorts and streams.

#include <cub/cub.cuh>

#include "common.cuh"

namespace ibf {
namespace {

__constant__ int c_tet_faces[12] = {1, 2, 3, 0, 3, 2, 0, 1, 3, 0, 2, 1};

__device__ __forceinline__ void face_verts(const long long* tets, long long f, int v[3]) {
  const long long t = f >> 2;
  const int r = (int)(f & 3);
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = (int)tets[4 * t + c_tet_faces[3 * r + k]];
}

__device__ __forceinline__ void sort3(int& a, int& b, int& c) {
  int t;
  if (a > b) { t = a; a = b; b = t; }
  if (b > c) { t = b; b = c; c = t; }
  if (a > b) { t = a; a = b; b = t; }
}

__global__ void k_check_ids(const long long* tets, long long n, int* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (tets[i] < 0 || tets[i] > 0x7fffffffLL) *bad = 1;
}

// key_bc = (b << 32) | c of the sorted triple, a, and the face id
__global__ void k_face_keys(const long long* tets, long long nf, unsigned long long* key_bc, unsigned* key_a,
                            int* idx) {
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < nf; f += (long long)gridDim.x * blockDim.x) {
    int v[3];
    face_verts(tets, f, v);
    sort3(v[0], v[1], v[2]);
    key_bc[f] = ((unsigned long long)(unsigned)v[1] << 32) | (unsigned)v[2];
    key_a[f] = (unsigned)v[0];
    idx[f] = (int)f;
  }
}

// a of the face at each (b, c)-sorted position, for the second stable pass
__global__ void k_gather_a(const unsigned* key_a, const int* idx, long long nf, unsigned* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf; i += (long long)gridDim.x * blockDim.x)
    out[i] = key_a[idx[i]];
}

__device__ __forceinline__ bool same_face(const long long* tets, int f, int g) {
  int u[3], v[3];
  face_verts(tets, f, u);
  face_verts(tets, g, v);
  sort3(u[0], u[1], u[2]);
  sort3(v[0], v[1], v[2]);
  return u[0] == v[0] && u[1] == v[1] && u[2] == v[2];
}

// flag[f] = 1 iff face f's triple occurs once (differs from both sorted neighbours)
__global__ void k_boundary_flags(const long long* tets, const int* idx, long long nf, unsigned char* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf; i += (long long)gridDim.x * blockDim.x) {
    const int f = idx[i];
    const bool lo = i > 0 && same_face(tets, f, idx[i - 1]);
    const bool hi = i + 1 < nf && same_face(tets, f, idx[i + 1]);
    flag[f] = (lo || hi) ? 0 : 1;
  }
}

__global__ void k_write_tris(const long long* tets, const int* bface, long long nt, long long* tris,
                             unsigned long long* ekeys, unsigned* vkeys) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nt; t += (long long)gridDim.x * blockDim.x) {
    int v[3];
    face_verts(tets, bface[t], v);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      tris[3 * t + k] = v[k];
      vkeys[3 * t + k] = (unsigned)v[k];
      // edges (0,1), (1,2), (2,0) as sorted pairs
      const int a = v[k], b = v[(k + 1) % 3];
      const unsigned lo = (unsigned)min(a, b), hi = (unsigned)max(a, b);
      ekeys[3 * t + k] = ((unsigned long long)lo << 32) | hi;
    }
  }
}

__global__ void k_write_edges(const unsigned long long* ukeys, const int* counts, const int* n_runs, long long* edges,
                              int* n_nonmanifold) {
  const long long n = *n_runs;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    edges[2 * i] = (long long)(ukeys[i] >> 32);
    edges[2 * i + 1] = (long long)(ukeys[i] & 0xffffffffULL);
    if (counts[i] > 2) atomicAdd(n_nonmanifold, 1);
  }
}

__global__ void k_widen(const unsigned* in, const int* n, long long* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < *n; i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i];
}

int grid_of(long long n) { return (int)std::max<long long>(1, std::min<long long>(div_up(n, 256), 16LL * sm_count())); }

}  // namespace
}  // namespace ibf

using namespace ibf;

struct ibf_surface {
  DevBuf<long long> tris, edges, verts;
  int64_t n_tris = 0, n_edges = 0, n_verts = 0, n_nonmanifold = 0;
};

static int extract(ibf_surface* h, int64_t m, const int64_t* tets_dev, cudaStream_t s) {
  const long long* tets = (const long long*)tets_dev;
  const long long nf = 4 * (long long)m;
  if (nf == 0) return IBF_OK;
  DevBuf<unsigned long long> kbc, kbc2;
  DevBuf<unsigned> ka, ka2, ka3;
  DevBuf<int> idx, idx2, idx3, small;
  DevBuf<unsigned char> flag;
  DevBuf<char> tmp;
  IBF_TRY(kbc.reserve(nf));
  IBF_TRY(kbc2.reserve(nf));
  IBF_TRY(ka.reserve(nf));
  IBF_TRY(ka2.reserve(nf));
  IBF_TRY(ka3.reserve(nf));
  IBF_TRY(idx.reserve(nf));
  IBF_TRY(idx2.reserve(nf));
  IBF_TRY(idx3.reserve(nf));
  IBF_TRY(flag.reserve(nf));
  IBF_TRY(small.reserve(4));
  IBF_CUDA(cudaMemsetAsync(small.p, 0, 4 * sizeof(int), s));
  k_check_ids<<<grid_of(4 * m), 256, 0, s>>>(tets, 4 * m, small.p);
  IBF_LAUNCH_CHECK();
  int host[4];
  IBF_CUDA(cudaMemcpyAsync(host, small.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  if (host[0]) {
    set_error("ibf_surface_extract: vertex id outside [0, 2^31)");
    return IBF_ERR_BAD_ARG;
  }
  auto cub_tmp = [&](size_t need) -> int {
    IBF_TRY(tmp.reserve(need + 16));
    return IBF_OK;
  };
  const int n = (int)nf;
  k_face_keys<<<grid_of(nf), 256, 0, s>>>(tets, nf, kbc.p, ka.p, idx.p);
  IBF_LAUNCH_CHECK();
  // pass 1: by (b, c); pass 2 (stable): by a
  size_t need = 0, have;
  cub::DeviceRadixSort::SortPairs(nullptr, need, kbc.p, kbc2.p, idx.p, idx2.p, n, 0, 64, s);
  IBF_TRY(cub_tmp(need));
  have = tmp.cap;
  IBF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, have, kbc.p, kbc2.p, idx.p, idx2.p, n, 0, 64, s));
  k_gather_a<<<grid_of(nf), 256, 0, s>>>(ka.p, idx2.p, nf, ka2.p);
  IBF_LAUNCH_CHECK();
  need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, ka2.p, ka3.p, idx2.p, idx3.p, n, 0, 32, s);
  IBF_TRY(cub_tmp(need));
  have = tmp.cap;
  IBF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, have, ka2.p, ka3.p, idx2.p, idx3.p, n, 0, 32, s));
  k_boundary_flags<<<grid_of(nf), 256, 0, s>>>(tets, idx3.p, nf, flag.p);
  IBF_LAUNCH_CHECK();
  // boundary face ids in ascending face order (reference: faces[counts[inverse] == 1])
  need = 0;
  cub::DeviceSelect::Flagged(nullptr, need, cub::CountingInputIterator<int>(0), flag.p, idx.p, small.p, n, s);
  IBF_TRY(cub_tmp(need));
  have = tmp.cap;
  IBF_CUDA(cub::DeviceSelect::Flagged(tmp.p, have, cub::CountingInputIterator<int>(0), flag.p, idx.p, small.p, n, s));
  IBF_CUDA(cudaMemcpyAsync(host, small.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  const long long nt = host[0];
  h->n_tris = nt;
  IBF_TRY(h->tris.reserve(3 * nt + 1));
  if (nt) {
    // edges: 3 nt 64-bit keys (kbc/kbc2), vertices: 3 nt ids (ka/ka2), run
    // counts (idx2); 3 nt exceeds the 4 m face count when most faces are
    // boundary (a lone tet: 12 > 4)
    IBF_TRY(kbc.reserve(3 * nt));
    IBF_TRY(kbc2.reserve(3 * nt));
    IBF_TRY(ka.reserve(3 * nt));
    IBF_TRY(ka2.reserve(3 * nt));
    IBF_TRY(idx2.reserve(3 * nt));
    k_write_tris<<<grid_of(nt), 256, 0, s>>>(tets, idx.p, nt, h->tris.p, kbc.p, ka.p);
    IBF_LAUNCH_CHECK();
    const int ne3 = (int)(3 * nt);
    need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, kbc.p, kbc2.p, ne3, 0, 64, s);
    IBF_TRY(cub_tmp(need));
    have = tmp.cap;
    IBF_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, have, kbc.p, kbc2.p, ne3, 0, 64, s));
    need = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, need, kbc2.p, kbc.p, idx2.p, small.p + 1, ne3, s);
    IBF_TRY(cub_tmp(need));
    have = tmp.cap;
    IBF_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, have, kbc2.p, kbc.p, idx2.p, small.p + 1, ne3, s));
    IBF_TRY(h->edges.reserve(2LL * ne3));
    k_write_edges<<<grid_of(ne3), 256, 0, s>>>(kbc.p, idx2.p, small.p + 1, h->edges.p, small.p + 2);
    IBF_LAUNCH_CHECK();
    need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, ka.p, ka2.p, ne3, 0, 32, s);
    IBF_TRY(cub_tmp(need));
    have = tmp.cap;
    IBF_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, have, ka.p, ka2.p, ne3, 0, 32, s));
    need = 0;
    cub::DeviceSelect::Unique(nullptr, need, ka2.p, ka.p, small.p + 3, ne3, s);
    IBF_TRY(cub_tmp(need));
    have = tmp.cap;
    IBF_CUDA(cub::DeviceSelect::Unique(tmp.p, have, ka2.p, ka.p, small.p + 3, ne3, s));
    IBF_TRY(h->verts.reserve(ne3));
    k_widen<<<grid_of(ne3), 256, 0, s>>>(ka.p, small.p + 3, h->verts.p);
    IBF_LAUNCH_CHECK();
    IBF_CUDA(cudaMemcpyAsync(host, small.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
    IBF_CUDA(cudaStreamSynchronize(s));
    h->n_edges = host[1];
    h->n_nonmanifold = host[2];
    h->n_verts = host[3];
  }
  return IBF_OK;
}

extern "C" int ibf_surface_extract(int64_t m, const int64_t* tets_dev, ibf_surface** out, int64_t* n_tris,
                                   int64_t* n_edges, int64_t* n_verts, int64_t* n_nonmanifold, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  if (!out || !n_tris || !n_edges || !n_verts || !n_nonmanifold || m < 0 || (m > 0 && !tets_dev)) {
    set_error("ibf_surface_extract: bad arguments");
    return IBF_ERR_BAD_ARG;
  }
  *out = nullptr;
  if (m > (int64_t)0x1fffffff / 4) {
    set_error("ibf_surface_extract: more than 2^27 tets");
    return IBF_ERR_BAD_ARG;
  }
  auto* h = new ibf_surface();
  const int st_ = extract(h, m, tets_dev, (cudaStream_t)st);
  if (st_ != IBF_OK) {
    delete h;
    return st_;
  }
  *out = h;
  *n_tris = h->n_tris;
  *n_edges = h->n_edges;
  *n_verts = h->n_verts;
  *n_nonmanifold = h->n_nonmanifold;
  return IBF_OK;
}

extern "C" int ibf_surface_get(const ibf_surface* h, int64_t* tris, int64_t* edges, int64_t* verts, ibf_stream st) {
  ::ibf::StreamScope ibf_scope_((cudaStream_t)st);
  if (!h) {
    set_error("ibf_surface_get: null handle");
    return IBF_ERR_BAD_ARG;
  }
  cudaStream_t s = (cudaStream_t)st;
  if (tris && h->n_tris)
    IBF_CUDA(cudaMemcpyAsync(tris, h->tris.p, 3 * h->n_tris * sizeof(int64_t), cudaMemcpyDefault, s));
  if (edges && h->n_edges)
    IBF_CUDA(cudaMemcpyAsync(edges, h->edges.p, 2 * h->n_edges * sizeof(int64_t), cudaMemcpyDefault, s));
  if (verts && h->n_verts)
    IBF_CUDA(cudaMemcpyAsync(verts, h->verts.p, h->n_verts * sizeof(int64_t), cudaMemcpyDefault, s));
  IBF_CUDA(cudaStreamSynchronize(s));
  return IBF_OK;
}

extern "C" void ibf_surface_destroy(ibf_surface* h) { delete h; }
