// Shared internals of libibf.so: status plumbing, device buffers, deterministic
// reductions.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/ibf.h"

namespace ibf {

void set_error(const std::string& msg);

#define IBF_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::ibf::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));         \
      return _e == cudaErrorMemoryAllocation ? IBF_ERR_OOM : IBF_ERR_CUDA;          \
    }                                                                               \
  } while (0)

#define IBF_TRY(call)                  \
  do {                                 \
    int _s = (call);                   \
    if (_s != IBF_OK) return _s;       \
  } while (0)

// every kernel launch of the library is followed by IBF_LAUNCH_CHECK, which
// also counts it (ibf_launch_count) for the bench's gpu_launches claim;
// atomic, since independent scenes may step concurrently on separate streams
extern std::atomic<unsigned long long> g_launches;
#define IBF_LAUNCH_CHECK()        \
  do {                            \
    ++::ibf::g_launches;          \
    IBF_CUDA(cudaGetLastError()); \
  } while (0)

// Device-time accumulator for one phase: events bracket the phase on its
// stream; harvest() adds the elapsed time once the stream has synchronised.
struct PhaseTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  bool pending = false;
  double ms = 0.0;
  long long count = 0;
  void begin(cudaStream_t s) {
    if (!a) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
    }
    harvest();
    cudaEventRecord(a, s);
  }
  void end(cudaStream_t s) {
    cudaEventRecord(b, s);
    pending = true;
  }
  void harvest() {
    if (!pending) return;
    float t = 0.0f;
    if (cudaEventElapsedTime(&t, a, b) == cudaSuccess) {
      ms += t;
      ++count;
      pending = false;
    }
  }
  void reset() {
    harvest();
    ms = 0.0;
    count = 0;
  }
};

// Per-kernel device clocks for the roofline lines of the bench
// (ibf_kernel_clocks): when switched on, a KernelClock scope brackets one
// launch with an event pair on its stream and books the launch's ALGORITHMIC
// bytes and flops (computed at the launch site from the
// sizes it processes).  Events are harvested when the clocks are read.  Off:
// one relaxed atomic load per launch.
enum KernelClockId {
  KC_ELEM = 0,      // k_elem: F, energy, PK1, SVD/eigen, 10 PSD blocks per tet
  KC_GATHER,        // k_gather_blocks: staging -> BSR slots
  KC_ROWS,          // k_vertex_rows: gradient rows, contact diagonal, Jacobi inverse
  KC_ENERGY,        // k_energy: incremental potential at up to 8 trial points
  KC_TRAVERSE,      // k_traverse: LBVH queries + fused ACCD prefilter
  KC_TOI,           // k_pair_toi: ACCD narrow phase on the survivors
  KC_PCG,           // k_pcg: one persistent PCG solve
  KC_PREFILTER,     // k_prefilter: ACCD prefilter over the broad-phase candidates
  KC_REFIT,         // LBVH refit: k_refit_treelets + k_refit_top (or k_refit_packed)
  KC_COUNT
};
extern std::atomic<bool> g_kclock_on;
struct KernelClock {
  int id;
  cudaStream_t s;
  cudaEvent_t b = nullptr;
  double bytes, flops, units;
  KernelClock(int id_, cudaStream_t s_, double bytes_, double flops_ = 0.0, double units_ = 0.0);
  ~KernelClock();
  KernelClock(const KernelClock&) = delete;
  KernelClock& operator=(const KernelClock&) = delete;
};

// Opt-in host-side phase trace (IBF_TRACE=1): synchronises the stream at
// each mark and prints the elapsed wall time per phase to stderr.  Off by
// default; a dev tool for finding host/device stalls, never on the timed path.
bool trace_enabled();
struct Trace {
  bool on;
  double last;
  std::string out;
  explicit Trace(const char* name);
  void mark(const char* what, cudaStream_t s, long long v = -1);
  ~Trace();
};

// Growable device buffer owned by a handle.  Never shrinks; growth only
// happens outside the timed hot loop once capacities settle.
// IBF_ALLOC_LOG=1: report (re)allocations slower than 1 ms (dev aid)
bool alloc_log();
double wall_now();
void alloc_report(const char* what, size_t bytes, double t0);

// Device memory of the handles' growable buffers comes from the device's
// stream-ordered pool, with the release threshold raised so freed blocks stay
// mapped for reuse.  Plain cudaMalloc / cudaFree inside the Newton loop (a
// buffer outgrowing its capacity mid-press) measured 2-800 ms per call on the
// B200 boxes, stalling the whole frame; the pool path is microseconds.
// Inside a C-ABI call that names a stream (StreamScope, set by every such
// entry point) both are ordered on that stream — a handle is used on one
// stream only (ibf.h), so nothing else can still be reading the old block and
// no device-wide sync is needed: one scene's buffer growth no longer stalls
// the scenes in flight on other streams.  Outside such a call (handle create /
// destroy) dev_alloc returns memory usable on any stream and dev_free waits
// for the device, like cudaMalloc / cudaFree.
int dev_alloc(void** p, size_t bytes);
void dev_free(void* p);

// The stream of the innermost C-ABI call on this thread (0: none).
extern thread_local cudaStream_t tl_stream;
struct StreamScope {
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(tl_stream) { tl_stream = s; }
  ~StreamScope() { tl_stream = prev; }
  StreamScope(const StreamScope&) = delete;
  StreamScope& operator=(const StreamScope&) = delete;
};

// Growable device buffer owned by a handle.  Never shrinks.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  int reserve(size_t n) {
    if (n <= cap) return IBF_OK;
    size_t want = n + n / 4 + 64;
    const double t0 = alloc_log() ? wall_now() : 0.0;
    if (p) dev_free(p);
    p = nullptr;
    cap = 0;
    IBF_TRY(dev_alloc((void**)&p, want * sizeof(T)));
    cap = want;
    if (t0 > 0.0) alloc_report("reserve", want * sizeof(T), t0);
    return IBF_OK;
  }
  // grow preserving contents (stream-ordered copy)
  int grow_keep(size_t n, size_t used, cudaStream_t s) {
    if (n <= cap) return IBF_OK;
    size_t want = n + n / 2 + 64;
    const double t0 = alloc_log() ? wall_now() : 0.0;
    T* q = nullptr;
    IBF_TRY(dev_alloc((void**)&q, want * sizeof(T)));
    if (p && used) IBF_CUDA(cudaMemcpyAsync(q, p, used * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p) {
      IBF_CUDA(cudaStreamSynchronize(s));
      dev_free(p);
    }
    p = q;
    cap = want;
    if (t0 > 0.0) alloc_report("grow_keep", want * sizeof(T), t0);
    return IBF_OK;
  }
  int upload(const T* host, size_t n, cudaStream_t s = 0) {
    IBF_TRY(reserve(n ? n : 1));
    if (n) IBF_CUDA(cudaMemcpyAsync(p, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
    return IBF_OK;
  }
  void release() {
    if (p) dev_free(p);
    p = nullptr;
    cap = 0;
  }
  ~DevBuf() { release(); }
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// Pinned host scratch for scalar readbacks.
struct HostScratch {
  void* p = nullptr;
  size_t cap = 0;
  int reserve(size_t bytes) {
    if (bytes <= cap) return IBF_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    IBF_CUDA(cudaMallocHost(&p, bytes));
    cap = bytes;
    return IBF_OK;
  }
  ~HostScratch() {
    if (p) cudaFreeHost(p);
  }
};

int sm_count();
inline int64_t div_up(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------ device side

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum (fixed shuffle tree); result valid in every thread.
// smem must hold blockDim.x/32 doubles; callers separate consecutive uses with
// a __syncthreads (done at the end here).
__device__ __forceinline__ double block_sum(double v, double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  double r = (lane < nw) ? smem[lane] : 0.0;
  r = warp_sum(r);
  __syncthreads();
  return r;
}

__device__ __forceinline__ double block_max(double v, double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  double r = (lane < nw) ? smem[lane] : -INFINITY;
  r = warp_max(r);
  __syncthreads();
  return r;
}

// Sum of n partials in a fixed order by one warp (lane-strided, then tree).
__device__ __forceinline__ double warp_sum_array(const double* a, int n) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  for (int i = lane; i < n; i += 32) v += a[i];
  return warp_sum(v);
}

// atomicMin / atomicMax on non-negative doubles through their ordered bits.
__device__ __forceinline__ void atomic_min_nonneg(double* addr, double v) {
  atomicMin(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

}  // namespace ibf
