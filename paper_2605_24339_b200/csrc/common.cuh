// Shared device helpers for the GMCP B200 kernels.
//
// Vector algebra mirrors the reference's IEEE operation order (Eigen eager,
// left-to-right reductions: see oracle/eigen_shim/Eigen/Core). Translation
// units that must be bit-exact with the reference (sampler, broadphase, step
// filter) are compiled with -fmad=false so no FMA contraction changes a
// rounding; the energy/gradient/Hessian units allow FMA (1e-9 tolerance).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/gmcp_types.h"

namespace gmcp_b200 {

// ---------------------------------------------------------------------------
// errors

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StatusError : std::runtime_error {
  StatusError(int c, const std::string& m, int64_t b = -1) : std::runtime_error(m), code(c), bad(b) {}
  int code;
  int64_t bad;
};

#define GMCP_CUDA(call)                                                                      \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw ::gmcp_b200::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// Device memory comes from the device's stream-ordered pool with an
// unbounded release threshold: freed blocks stay cached in the process, so
// the buffers a rebuild regrows or a scratch DBuf re-creates are served
// without new driver mappings (plain cudaMalloc of fresh memory measured
// 10-300 ms on the box, in the batched Newton loop's rebuilds). A free first
// synchronizes the device (as cudaFree does), so no kernel still reads it.
inline void* dev_alloc(size_t bytes) {
  static std::atomic<bool> configured[64] = {};
  int dev = 0;
  GMCP_CUDA(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && !configured[dev].load(std::memory_order_acquire)) {
    cudaMemPool_t pool;  // idempotent: racing threads set the same attribute
    GMCP_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = ~0ull;
    GMCP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    configured[dev].store(true, std::memory_order_release);
  }
  void* p = nullptr;
  GMCP_CUDA(cudaMallocAsync(&p, bytes, 0));
  GMCP_CUDA(cudaStreamSynchronize(0));
  return p;
}
inline void dev_free(void* p) {
  if (!p) return;
  cudaDeviceSynchronize();
  cudaFreeAsync(p, 0);
}

// Device buffer (grow-only).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { dev_free(p); }
  void resize(size_t m) {
    if (m > cap) {
      static const bool trace = std::getenv("GMCP_TRACE_ALLOC") != nullptr;
      const auto t0 = std::chrono::steady_clock::now();
      dev_free(p);
      p = nullptr;
      const size_t old = cap;
      // 1.5x headroom, then doubling: per-rebuild sizes that drift by a few
      // percent (re-sampled scenes) never regrow a buffer inside a solve
      cap = std::max(m + m / 2 + 16, 2 * cap);
      p = static_cast<T*>(dev_alloc(cap * sizeof(T)));
      if (trace)
        std::fprintf(stderr, "[gmcp alloc] %zu -> %zu B in %.2f ms\n", old * sizeof(T), cap * sizeof(T),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    n = m;
  }
  void upload(const T* h, size_t m, cudaStream_t s) {
    resize(m);
    if (m) GMCP_CUDA(cudaMemcpyAsync(p, h, m * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
  void download(T* h, size_t m, cudaStream_t s) const {
    if (m) GMCP_CUDA(cudaMemcpyAsync(h, p, m * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  std::vector<T> to_host(cudaStream_t s) const {
    std::vector<T> v(n);
    download(v.data(), n, s);
    GMCP_CUDA(cudaStreamSynchronize(s));
    return v;
  }
  void zero(cudaStream_t s) {
    if (n) GMCP_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(cap, o.cap);
  }
};

// NVTX range over a host stage (K-stages of the pipeline, the solver phases):
// visible in Nsight Systems / ncu --nvtx; no cost without an attached tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------------------
// Per-context binding. Every C-ABI entry binds its context's device and CUB
// temp storage to the calling thread for the duration of the call (RAII), so
// contexts on different devices (or several on one device) may be driven
// from different host threads: nothing device-side is process-global.

struct CubScratch {
  DBuf<unsigned char> tmp;
  void* get(size_t bytes) {
    tmp.resize(bytes > 0 ? bytes : 1);
    return tmp.p;
  }
};

CubScratch*& bound_scratch();  // thread-local; defined in capi.cpp

class DeviceBind {
 public:
  DeviceBind(int device, CubScratch* s) : prev_s_(bound_scratch()) {
    GMCP_CUDA(cudaGetDevice(&prev_dev_));
    if (prev_dev_ != device) GMCP_CUDA(cudaSetDevice(device));
    bound_scratch() = s;
    dev_ = device;
  }
  ~DeviceBind() {
    bound_scratch() = prev_s_;
    if (prev_dev_ != dev_) cudaSetDevice(prev_dev_);
  }
  DeviceBind(const DeviceBind&) = delete;
  DeviceBind& operator=(const DeviceBind&) = delete;

 private:
  int prev_dev_ = 0, dev_ = 0;
  CubScratch* prev_s_;
};

// ---------------------------------------------------------------------------
// vector algebra (reference evaluation order)

struct d3 {
  double x, y, z;
};
struct d2 {
  double x, y;
};

__host__ __device__ __forceinline__ d3 mk3(double a, double b, double c) { return d3{a, b, c}; }
__device__ __forceinline__ d3 ld3(const double* __restrict__ x, int v) {
  const double* p = x + 3 * (int64_t)v;
  return d3{__ldg(p), __ldg(p + 1), __ldg(p + 2)};
}
// one 256-bit read-only load of a 32-byte aligned group of four doubles
__device__ __forceinline__ void ldg4(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ d3 ld3nc(const double* x, int v) {
  const double* p = x + 3 * (int64_t)v;
  return d3{p[0], p[1], p[2]};
}
__host__ __device__ __forceinline__ d3 operator+(d3 a, d3 b) { return d3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ __forceinline__ d3 operator-(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ __forceinline__ d3 operator*(double s, d3 a) { return d3{s * a.x, s * a.y, s * a.z}; }
__host__ __device__ __forceinline__ d3 operator/(d3 a, double s) { return d3{a.x / s, a.y / s, a.z / s}; }
__host__ __device__ __forceinline__ double dot(d3 a, d3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__host__ __device__ __forceinline__ double norm(d3 a) { return sqrt(dot(a, a)); }
__host__ __device__ __forceinline__ d3 cross(d3 a, d3 b) {
  return d3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__host__ __device__ __forceinline__ d3 unit(d3 a) {
  const double z = dot(a, a);
  return z > 0 ? a / sqrt(z) : a;
}
__host__ __device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }
__host__ __device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }

__host__ __device__ __forceinline__ d2 operator+(d2 a, d2 b) { return d2{a.x + b.x, a.y + b.y}; }
__host__ __device__ __forceinline__ d2 operator-(d2 a, d2 b) { return d2{a.x - b.x, a.y - b.y}; }
__host__ __device__ __forceinline__ d2 operator*(double s, d2 a) { return d2{s * a.x, s * a.y}; }
__host__ __device__ __forceinline__ double norm2(d2 a) { return sqrt(a.x * a.x + a.y * a.y); }
__host__ __device__ __forceinline__ double cross2(d2 a, d2 b) { return a.x * b.y - a.y * b.x; }

// barrier.hpp:55-66 (callers check g > 0, eps > 0)
__device__ __forceinline__ void barrier_eval(double g, double eps, double& B, double& dB, double& ddB) {
  B = dB = ddB = 0;
  if (g >= eps) return;
  const double d = g - eps;
  const double ln = log(g / eps);
  B = -d * d * ln;
  dB = -2.0 * d * ln - d * d / g;
  ddB = -2.0 * ln - 4.0 * d / g + d * d / (g * g);
}

// ---------------------------------------------------------------------------
// device sample set (reference order, structure of arrays)

struct DevSamples {
  int64_t n = 0;
  const int8_t* type = nullptr;
  const int32_t* slave = nullptr;   // [n][3]
  const int32_t* master = nullptr;  // [n][3] (-1 padded)
  const double* beta_s = nullptr;   // [n][3]
  const double* wm = nullptr;       // [n][3] master interpolation weights (face beta_m; edge 1-eta, eta)
  const double* coef = nullptr;     // (kappa_type * weight) * gamma
  const double* eps = nullptr;
  const double* gamma = nullptr;
};

__device__ __forceinline__ int n_master(int8_t t) { return t == GMCP_FACE ? 3 : (t == GMCP_EDGE ? 2 : 1); }

// Warp-level deterministic reductions (fixed butterfly order).
// Programmatic dependent launch (sm_90+): a kernel launched with
// launch_pdl may become resident while the previous kernel on the stream is
// still running; it must execute pdl_wait() before reading that kernel's
// results. A primary that calls pdl_trigger() lets its dependents launch at
// once (their blocks take SM slots as the primary's blocks retire).
#ifndef GMCP_PDL
#define GMCP_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if GMCP_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if GMCP_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <class... P, class... A>
void launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, cudaStream_t s, A&&... args) {
#if GMCP_PDL
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  GMCP_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...));
#else
  kernel<<<grid, block, 0, s>>>(std::forward<A>(args)...);
#endif
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kRedBlocks = 592;  // fixed grid for deterministic reductions (4 x 148 SMs)
constexpr int kRedThreads = 256;

}  // namespace gmcp_b200
