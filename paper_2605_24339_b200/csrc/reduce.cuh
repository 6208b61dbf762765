// Deterministic reductions shared by the contact kernels: fixed grid, fixed
// per-thread order, fixed butterfly / block order -> bitwise reproducible.
#pragma once

#include "ctx.hpp"

namespace gmcp_b200 {
namespace {

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NT / 32; ++i) r += sh[i];
  return r;  // valid in thread 0
}

// Sums `parts` (n values, one per block of a fixed grid) in index order.
__global__ void k_sum_parts(const double* __restrict__ parts, int n, int stride, double* __restrict__ out) {
  __shared__ double sh[kRedThreads / 32];
  pdl_wait();  // no-op unless launched with launch_pdl
  for (int c = 0; c < stride; ++c) {
    double v = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += parts[(int64_t)i * stride + c];
    const double r = block_sum<kRedThreads>(v, sh);
    if (threadIdx.x == 0) out[c] = r;
  }
}


// status words: [0] first infeasible sample, [1] first degenerate, [2] spare
// (all ~0 = none), [3] = 0; memsets, no pageable host copy
inline void reset_red(Ctx& c) {
  c.red_u.resize(4);
  GMCP_CUDA(cudaMemsetAsync(c.red_u.p, 0xff, 3 * sizeof(unsigned long long), c.stream));
  GMCP_CUDA(cudaMemsetAsync(c.red_u.p + 3, 0, sizeof(unsigned long long), c.stream));
}

}  // namespace
}  // namespace gmcp_b200
