// Per-sample kinematics on the device (contact_energy.hpp:26-73) and the gap
// of contact_sampling.hpp:350-372, in the reference's operation order.
#pragma once

#include <cstring>

#include "common.cuh"

namespace gmcp_b200 {

struct Kin {
  double g;
  d3 n, xs;
  int nv;
  d3 dg[6];  // slave 0..2, master 3..5
};

// Loads the master interpolation weights / ids of sample i.
__device__ __forceinline__ void load_master(const DevSamples& S, int64_t i, int& nm, double w[3], int mid[3]) {
  nm = n_master(S.type[i]);
  w[0] = S.wm[3 * i];
  w[1] = S.wm[3 * i + 1];
  w[2] = S.wm[3 * i + 2];
  mid[0] = S.master[3 * i];
  mid[1] = S.master[3 * i + 1];
  mid[2] = S.master[3 * i + 2];
}

// sample_kinematics. Returns false for a degenerate slave triangle (cn == 0).
template <bool WithGradient>
__device__ __forceinline__ bool kinematics(const DevSamples& S, int64_t i, const double* __restrict__ x, Kin& k) {
  const d3 a0 = ld3(x, S.slave[3 * i]), a1 = ld3(x, S.slave[3 * i + 1]), a2 = ld3(x, S.slave[3 * i + 2]);
  const d3 e1 = a1 - a0, e2 = a2 - a0;
  const d3 c = cross(e1, e2);
  const double cn = norm(c);
  if (!(cn > 0)) return false;
  k.n = c / cn;
  const double b0 = S.beta_s[3 * i], b1 = S.beta_s[3 * i + 1], b2 = S.beta_s[3 * i + 2];
  k.xs = (b0 * a0 + b1 * a1) + b2 * a2;
  int nm, mid[3];
  double w[3];
  load_master(S, i, nm, w, mid);
  d3 xm = mk3(0, 0, 0);
  for (int j = 0; j < nm; ++j) xm = xm + w[j] * ld3(x, mid[j]);
  const d3 d = xm - k.xs;
  k.g = dot(k.n, d);
  k.nv = 3 + nm;
  if (WithGradient) {
    const d3 r = (d - k.g * k.n) / cn;
    k.dg[0] = (-b0) * k.n + cross(r, e2 - e1);
    k.dg[1] = (-b1) * k.n + cross(e2, r);
    k.dg[2] = (-b2) * k.n + cross(r, e1);
    for (int j = 0; j < nm; ++j) k.dg[3 + j] = w[j] * k.n;
  }
  return true;
}

// sample_gap with triangle_normal's degenerate-area cutoff (geometry.hpp:14-21).
// Returns false when triangle_normal would throw.
__device__ __forceinline__ bool sample_gap(const DevSamples& S, int64_t i, const double* __restrict__ x, double& g) {
  const d3 a0 = ld3(x, S.slave[3 * i]), a1 = ld3(x, S.slave[3 * i + 1]), a2 = ld3(x, S.slave[3 * i + 2]);
  const d3 cr = cross(a1 - a0, a2 - a0);
  const d3 lo = mk3(dmin(dmin(a0.x, a1.x), a2.x), dmin(dmin(a0.y, a1.y), a2.y), dmin(dmin(a0.z, a1.z), a2.z));
  const d3 hi = mk3(dmax(dmax(a0.x, a1.x), a2.x), dmax(dmax(a0.y, a1.y), a2.y), dmax(dmax(a0.z, a1.z), a2.z));
  const double diag2 = norm(hi - lo);
  if (0.5 * norm(cr) <= 1e-12 * diag2 * diag2) return false;
  const d3 n = unit(cr);
  const d3 xs = (S.beta_s[3 * i] * a0 + S.beta_s[3 * i + 1] * a1) + S.beta_s[3 * i + 2] * a2;
  int nm, mid[3];
  double w[3];
  load_master(S, i, nm, w, mid);
  d3 xm;
  if (nm == 3)
    xm = (w[0] * ld3(x, mid[0]) + w[1] * ld3(x, mid[1])) + w[2] * ld3(x, mid[2]);
  else if (nm == 2)
    xm = w[0] * ld3(x, mid[0]) + w[1] * ld3(x, mid[1]);
  else
    xm = ld3(x, mid[0]);
  g = dot(n, xm - xs);
  return true;
}

// Order-preserving map double -> uint64 for atomicMin/atomicMax.
__device__ __forceinline__ unsigned long long ord_bits(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double from_ord_bits(unsigned long long b) {
  b = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d;
  memcpy(&d, &b, sizeof d);
  return d;
#endif
}
inline unsigned long long ord_bits_host(double v) {
  unsigned long long b;
  memcpy(&b, &v, sizeof b);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

}  // namespace gmcp_b200
