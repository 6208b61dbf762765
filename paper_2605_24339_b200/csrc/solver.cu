// Device-resident quasi-static solver: the reference's System::solve
// (proj/include/gmcp/solver.hpp:125-228) with the LDL^T direct solve replaced
// by a block-Jacobi preconditioned CG over 3x3 BCSR (K9), the linear elastic
// operator (elasticity.hpp:39-141) as a constant BCSR (K11), and the contact
// terms from the per-pair contexts (K6-K10). Positions, step, gradient and
// every Krylov vector stay on the device for the whole run; the host reads
// only scalars (residual, alpha, energy decrease, convergence) per iteration.
#include <algorithm>
#include <atomic>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

#include "../../include/gmcp_solver.h"
#include "ctx.hpp"
#include "kin.cuh"
#include "cubutil.cuh"
#include <cooperative_groups.h>
#include "coarse.cuh"

namespace gmcp_b200 {

namespace {

constexpr int kMaxPairs = 4;
constexpr int kThreads = 256;
constexpr int kBlocks = 592;  // fixed grid: deterministic reductions
#ifndef GMCP_PAIR_JACOBI
#define GMCP_PAIR_JACOBI 1  // vertex-pair 6x6 block-Jacobi for the single-system PCG
#endif

// ---------------------------------------------------------------------------
// deterministic single-kernel reductions: per-block partials + "last block"
// sums them in block order.

struct RedSlot {
  double* parts;          // [kBlocks * width]
  unsigned int* counter;  // arrival counter (reset by the last block)
};

template <int W, int NT = kThreads>
__device__ __forceinline__ bool block_reduce_last(double (&v)[W], RedSlot rs, double (&out)[W]) {
  __shared__ double sh[W][NT / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < W; ++q) {
    double t = warp_sum(v[q]);
    if (lane == 0) sh[q][wid] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < W; ++q) {
      double t = 0;
      for (int i = 0; i < NT / 32; ++i) t += sh[q][i];
      rs.parts[blockIdx.x * W + q] = t;
    }
    __threadfence();
    last = atomicAdd(rs.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
#pragma unroll
  for (int q = 0; q < W; ++q) {
    double t = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += NT) t += __ldcg(rs.parts + i * W + q);
    t = warp_sum(t);
    if (lane == 0) sh[q][wid] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < W; ++q) {
      double t = 0;
      for (int i = 0; i < NT / 32; ++i) t += sh[q][i];
      out[q] = t;
    }
    *rs.counter = 0;
  }
  return true;  // out valid in thread 0 of the last block
}

// ---------------------------------------------------------------------------
// BCSR descriptor (3x3 blocks, rows = vertices)

struct Bcsr {
  const int32_t* rowptr = nullptr;
  const int32_t* cols = nullptr;
  const double* vals = nullptr;
  int bs = 9;       // value (block k, entry q) at vals[k * bs + q * cs]:
  int64_t cs = 1;   // AoS (9, 1) or component-major (1, nnzb)
};
struct MatSet {
  Bcsr el;
  Bcsr c[kMaxPairs];
  int np = 0;
  double shift = 0;  // regularization added to every diagonal entry (solver.hpp:352-356)
  // symmetric-half copy of el for the PCG SpMV (single systems): the nh
  // blocks on and above the diagonal, compacted: entries 0-7 of stored block i
  // at hv[8 i] (two 32-byte loads), entry 8 at hv[8 nh + i]. hix[k] (union
  // block k) = i of the stored block on/above the diagonal, ~i of the stored
  // block whose transpose it is (below the diagonal); nh = hn. The SpMV reads
  // (column, hix) pairs interleaved: hix[2 k] = column, hix[2 k + 1] = index.
  const int32_t* hix = nullptr;
  int64_t hn = 0;
  const double* hv = nullptr;
};

__device__ __forceinline__ d3 bmv(const double* b, d3 p) {
  return d3{b[0] * p.x + b[1] * p.y + b[2] * p.z, b[3] * p.x + b[4] * p.y + b[5] * p.z,
            b[6] * p.x + b[7] * p.y + b[8] * p.z};
}

// y_v = sum_j A_vj p_j for one row, lanes stride the row's blocks, then a
// fixed butterfly -> deterministic.
__device__ __forceinline__ d3 row_mv(const Bcsr& A, int v, const double* __restrict__ p, int lane) {
  d3 acc = mk3(0, 0, 0);
  const int a = A.rowptr[v], b = A.rowptr[v + 1];
  for (int k = a + lane; k < b; k += 32) acc = acc + bmv(A.vals + 9 * (int64_t)k, ld3(p, A.cols[k]));
  return acc;
}

// K9 -- preconditioned CG, two kernels per iteration. The SpMV forms the new
// search direction on the fly from double-buffered p (p_new = z + beta p_old
// for every row it touches, written only for its own rows), so the separate
// p-update pass disappears while the arithmetic stays standard PCG:
//   p = z + beta p, q = A p, alpha = rz / (p.q), x += alpha p, r -= alpha q,
//   z = Minv r, beta = rz_new / rz.
// scal: [0] rz [1] pq [2] alpha [3] beta [4] rr [5] bb

// lanes per BCSR row in the SpMV: 4 for large systems (beats 2, 8, 16 on C3),
// 8 below kSmallRows rows, where the iteration is latency-bound
constexpr int kSmallRows = 32768;
constexpr double kRegularization = 1e-8;  // SolverSettings::regularization (solver.hpp:40)
// Stagnation = the solve failed (a singular step: e.g. a body held only by
// contact that is not yet engaged, with a load along the free mode). The
// reference's LDL^T fails at once there and retries regularized
// (solver.hpp:352-361); CG instead plateaus at the inconsistent part of the
// rhs. A solve whose best rr over the last kStagWindow iterations did not
// halve the best rr before that window, while still above 1e-8 bb, is
// declared failed, so the regularized retry starts after ~2k iterations
// rather than pcg_max_iters. Converging solves shrink rr by orders of
// magnitude per window and never trip it.
constexpr int kStagWindow = 1024;
constexpr int kStagWindowCoarse = 256;
constexpr int kDriftWindow = 256;
constexpr double kDriftFail = 1e6;  // 100x the largest true/tolerance ratio refinement accepts (kRefineMaxDrift)
// an unshifted solve whose true residual is this far above the rhs at a drift
// check diverges along an unconstrained mode (singular system) -> fail now (a
// regularized solve may pass through large residuals on its way down: exempt)
constexpr double kDivergeRel = 10.0;
constexpr double kAcceptRelInf = 1e-6;  // solver.hpp:349-356 acceptance of a linear solve
// scaled coarse pivots below this drop their rigid mode: low enough to keep a
// floating body's regularized rigid mode (pivot ~ shift / aggregate stiffness)
constexpr double kCoarseDropDefault = 1e-13;
constexpr double kSceneCoarseDrop = 1e-8;  // per-scene inverses: ill-conditioned rigid modes drop earlier
constexpr double kCoarseStale = 1.25;   // refresh the coarse inverse when a solve needs 25% more iterations

// A_vj x for block k, read through the read-only path (either layout)
__device__ __forceinline__ d3 bmv_ro(const Bcsr& A, int64_t k, d3 p) {
  const double* b = A.vals + k * A.bs;
  const int64_t c = A.cs;
  const double b0 = __ldg(b), b1 = __ldg(b + c), b2 = __ldg(b + 2 * c), b3 = __ldg(b + 3 * c), b4 = __ldg(b + 4 * c);
  const double b5 = __ldg(b + 5 * c), b6 = __ldg(b + 6 * c), b7 = __ldg(b + 7 * c), b8 = __ldg(b + 8 * c);
  return d3{b0 * p.x + b1 * p.y + b2 * p.z, b3 * p.x + b4 * p.y + b5 * p.z, b6 * p.x + b7 * p.y + b8 * p.z};
}

// y_v = sum_j A_vj (z_j + beta p_j) over one row by kRowLanes lanes, two
// blocks in flight per lane (fixed order: deterministic)
// block k of the symmetric-half operand times p: H_vj for j >= v, else the
// transpose of the stored block (j, v)
__device__ __forceinline__ d3 half_bmv(int raw, const double* __restrict__ hv, int64_t nh, d3 p) {
  const bool lower = raw < 0;
  const int64_t idx = lower ? ~raw : raw;
  double b0, u1, u2, u3, b4, u5, u6, u7;
  ldg4(hv + 8 * idx, b0, u1, u2, u3);
  ldg4(hv + 8 * idx + 4, b4, u5, u6, u7);
  const double b8 = __ldg(hv + 8 * nh + idx);
  const double b1 = lower ? u3 : u1, b3 = lower ? u1 : u3, b2 = lower ? u6 : u2, b6 = lower ? u2 : u6;
  const double b5 = lower ? u7 : u5, b7 = lower ? u5 : u7;
  return d3{b0 * p.x + b1 * p.y + b2 * p.z, b3 * p.x + b4 * p.y + b5 * p.z, b6 * p.x + b7 * p.y + b8 * p.z};
}

// row_mv8 over the symmetric-half operand (MatSet::hv / hix)
template <int kRowLanes, bool kOne = false>
__device__ __forceinline__ d3 row_mv8_half(const Bcsr& A, const int32_t* __restrict__ hix,
                                           const double* __restrict__ hv, int64_t nh, int v,
                                           const double* __restrict__ z, const double* __restrict__ p, double beta,
                                           int sub) {
  d3 acc0 = mk3(0, 0, 0), acc1 = mk3(0, 0, 0);
  const int a = __ldg(A.rowptr + v), b = __ldg(A.rowptr + v + 1);
  const int2* ch = reinterpret_cast<const int2*>(hix);
  int k = a + sub;
  for (; k + kRowLanes < b; k += 2 * kRowLanes) {
    const int2 c0 = __ldg(ch + k), c1 = __ldg(ch + k + kRowLanes);
    const d3 x0 = kOne ? ld3(p, c0.x) : ld3(z, c0.x) + beta * ld3(p, c0.x);
    const d3 x1 = kOne ? ld3(p, c1.x) : ld3(z, c1.x) + beta * ld3(p, c1.x);
    acc0 = acc0 + half_bmv(c0.y, hv, nh, x0);
    acc1 = acc1 + half_bmv(c1.y, hv, nh, x1);
  }
  if (k < b) {
    const int2 c0 = __ldg(ch + k);
    acc0 = acc0 + half_bmv(c0.y, hv, nh, kOne ? ld3(p, c0.x) : ld3(z, c0.x) + beta * ld3(p, c0.x));
  }
  return acc0 + acc1;
}

template <int kRowLanes>
__device__ __forceinline__ d3 row_mv8(const Bcsr& A, int v, const double* __restrict__ z,
                                      const double* __restrict__ p, double beta, int sub) {
  d3 acc0 = mk3(0, 0, 0), acc1 = mk3(0, 0, 0);
  const int a = __ldg(A.rowptr + v), b = __ldg(A.rowptr + v + 1);
  int k = a + sub;
  for (; k + kRowLanes < b; k += 2 * kRowLanes) {
    const int j0 = __ldg(A.cols + k), j1 = __ldg(A.cols + k + kRowLanes);
    const d3 x0 = ld3(z, j0) + beta * ld3(p, j0);
    const d3 x1 = ld3(z, j1) + beta * ld3(p, j1);
    acc0 = acc0 + bmv_ro(A, k, x0);
    acc1 = acc1 + bmv_ro(A, k + kRowLanes, x1);
  }
  if (k < b) {
    const int j = __ldg(A.cols + k);
    acc0 = acc0 + bmv_ro(A, k, ld3(z, j) + beta * ld3(p, j));
  }
  return acc0 + acc1;
}

// K9a: p_new = z + beta p_old (own rows), q = mask .* (H p_new), pq -> alpha (last block).
inline bool pupdate_on() {  // GMCP_PUPDATE=0: p_new formed inside the SpMV on every system
  static const bool on = !std::getenv("GMCP_PUPDATE") || std::atoi(std::getenv("GMCP_PUPDATE")) != 0;
  return on;
}

// p_new = z + beta p_old, streamed (the SpMV then gathers one vector, not two)
__global__ void __launch_bounds__(kThreads) k_pupdate(int64_t n, const double* __restrict__ z,
                                                      const double* __restrict__ p_old, double* __restrict__ p_new,
                                                      const double* __restrict__ scal) {
  const double beta = scal[3];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p_new[i] = z[i] + beta * p_old[i];
}

template <int kRowLanes, bool kHalf = false, bool kPre = false>
__global__ void __launch_bounds__(kThreads) k_spmv_cg(int nv, MatSet M, const double* __restrict__ mask,
                                                      const double* __restrict__ z, const double* __restrict__ p_old,
                                                      double* __restrict__ p_new, double* __restrict__ q,
                                                      double* scal, RedSlot rs) {
  const int lane = threadIdx.x & 31, sub = lane & (kRowLanes - 1);
  const double beta = scal[3];
  double dots[1] = {0};
  const int rows_per_block = kThreads / kRowLanes;
  // the loop bound is uniform per warp (all lanes reach the shuffles)
  for (int v0 = blockIdx.x * rows_per_block + (threadIdx.x >> 5) * (32 / kRowLanes); v0 < nv;
       v0 += gridDim.x * rows_per_block) {
    const int v = v0 + (lane / kRowLanes);
    d3 acc = mk3(0, 0, 0);
    if (v < nv) {
      if (kPre) {  // p_new formed by k_pupdate: one gathered vector
        acc = row_mv8_half<kRowLanes, true>(M.el, M.hix, M.hv, M.hn, v, nullptr, p_new, 0.0, sub);
      } else if (kHalf) {
        acc = row_mv8_half<kRowLanes>(M.el, M.hix, M.hv, M.hn, v, z, p_old, beta, sub);
      } else {
        acc = row_mv8<kRowLanes>(M.el, v, z, p_old, beta, sub);
        for (int k = 0; k < M.np; ++k) acc = acc + row_mv8<kRowLanes>(M.c[k], v, z, p_old, beta, sub);
      }
    }
#pragma unroll
    for (int o = kRowLanes / 2; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    }
    if (sub == 0 && v < nv) {
      const d3 m = ld3(mask, v);
      const d3 pv = kPre ? ld3(p_new, v) : ld3(z, v) + beta * ld3(p_old, v);
      if (M.shift != 0) acc = acc + M.shift * pv;
      const d3 y = mk3(m.x * acc.x, m.y * acc.y, m.z * acc.z);
      q[3 * v] = y.x;
      q[3 * v + 1] = y.y;
      q[3 * v + 2] = y.z;
      if (!kPre) {
        p_new[3 * v] = pv.x;
        p_new[3 * v + 1] = pv.y;
        p_new[3 * v + 2] = pv.z;
      }
      dots[0] += dot(pv, y);
    }
  }
  double out[1];
  if (block_reduce_last<1>(dots, rs, out) && threadIdx.x == 0) {
    scal[1] = out[0];                                // pq
    scal[2] = out[0] != 0 ? scal[0] / out[0] : 0.0;  // alpha = rz / pq
    if (!(out[0] > 0)) scal[8] += 1.0;               // p.Hp <= 0: H not positive definite on p
  }
}

// K9b: x += alpha p, r -= alpha q, z = Minv r; rz_new, rr -> beta (last block).
template <bool kCoarse>
__global__ void __launch_bounds__(kThreads) k_update_cg(int nv, const double* __restrict__ p,
                                                        const double* __restrict__ q, double* __restrict__ x,
                                                        double* __restrict__ r, double* __restrict__ z,
                                                        const double* __restrict__ minv, double* scal, RedSlot rs) {
  const double a = scal[2];
  double dots[2] = {0, 0};
  // per-warp transpose of the 24-byte-per-thread results: coalesced stores
  __shared__ double stg[kThreads / 32][3][96];
  const int lane = threadIdx.x & 31;
  double(*st)[96] = stg[threadIdx.x >> 5];
  for (int v = blockIdx.x * kThreads + threadIdx.x; v - lane < nv; v += gridDim.x * kThreads) {
    const bool in = v < nv;
    const int vv = in ? v : nv - 1;
    const d3 xv = ld3nc(x, vv) + a * ld3nc(p, vv);
    const d3 rv = ld3nc(r, vv) - a * ld3nc(q, vv);
    const d3 zv = bmv(minv + 9 * (int64_t)vv, rv);
    const double xa[3] = {xv.x, xv.y, xv.z}, ra[3] = {rv.x, rv.y, rv.z}, za[3] = {zv.x, zv.y, zv.z};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      st[0][3 * lane + c] = xa[c];
      st[1][3 * lane + c] = ra[c];
      st[2][3 * lane + c] = za[c];
    }
    __syncwarp();
    const int64_t base = 3 * (int64_t)(v - lane);
    const int64_t lim = 3 * (int64_t)nv - base;  // valid entries of this warp's slice
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int o = 32 * j + lane;
      if (o < lim) {
        x[base + o] = st[0][o];
        r[base + o] = st[1][o];
        z[base + o] = st[2][o];
      }
    }
    __syncwarp();
    if (in) {
      dots[0] += dot(rv, zv);
      dots[1] += dot(rv, rv);
    }
  }
  double out[2];
  if (block_reduce_last<2>(dots, rs, out) && threadIdx.x == 0) {
    if (kCoarse) {  // r.z completed by the coarse solve (k_coarse_apply)
      scal[6] = out[0];
    } else {
      const double rz_old = scal[0];
      scal[3] = rz_old != 0 ? out[0] / rz_old : 0.0;  // beta
      scal[0] = out[0];                                // rz
    }
    scal[4] = out[1];  // rr
  }
}

// Vertex-pair block-Jacobi (6x6): M = blockdiag over the pairs of the masked
// merged operator restricted to {v, partner}; unpaired vertices keep the 3x3
// block. Row v of M^-1 is stored as minv2[v] = [ (M^-1)_vv | (M^-1)_vp ]
// (3x6), so z_v = (M^-1)_vv r_v + (M^-1)_vp r_p. Both vertices of a pair
// invert the same 6x6 in the same (lower id first) order.
__device__ __forceinline__ bool get_block(const Bcsr& A, int v, int w, double* d) {
  int lo = A.rowptr[v], hi = A.rowptr[v + 1];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A.cols[mid] < w) lo = mid + 1; else hi = mid;
  }
  if (!(lo < A.rowptr[v + 1] && A.cols[lo] == w)) return false;
  const double* b = A.vals + (int64_t)lo * A.bs;
  for (int q = 0; q < 9; ++q) d[q] = b[q * A.cs];
  return true;
}
__device__ __forceinline__ void add_block(const MatSet& M, int v, int w, double* d) {
  double t[9];
  if (get_block(M.el, v, w, t))
    for (int q = 0; q < 9; ++q) d[q] += t[q];
  for (int k = 0; k < M.np; ++k)
    if (get_block(M.c[k], v, w, t))
      for (int q = 0; q < 9; ++q) d[q] += t[q];
}
__global__ void k_pair_jacobi(int nv, MatSet M, const double* __restrict__ mask, const int32_t* __restrict__ pair,
                              double* __restrict__ minv2, const int32_t* __restrict__ vscene = nullptr,
                              const double* __restrict__ shift_s = nullptr) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    if (shift_s) M.shift = shift_s[vscene[v]];  // batched scenes: the scene's own shift (pairs lie in one scene)
    const int pv = pair[v];
    const int a = pv < 0 ? v : min(v, pv), b = pv < 0 ? v : max(v, pv);
    const int n = pv < 0 ? 3 : 6;
    double G[6][6];
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) G[i][j] = (i == j && i >= n) ? 1.0 : 0.0;
    const int ids[2] = {a, b};
    for (int I = 0; I < n / 3; ++I)
      for (int J = 0; J < n / 3; ++J) {
        double d[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        add_block(M, ids[I], ids[J], d);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double g = d[3 * i + j] + (I == J && i == j ? M.shift : 0.0);
            const double mi = mask[3 * ids[I] + i], mj = mask[3 * ids[J] + j];
            if (mi == 0 || mj == 0) g = (I == J && i == j) ? 1.0 : 0.0;
            G[3 * I + i][3 * J + j] = g;
          }
      }
    // Gauss-Jordan inverse (SPD: no pivoting), in place. A pivot below 1e-12 x
    // the largest diagonal entry (singular or nearly singular pair block)
    // makes both vertices of the pair fall back to their own 3x3 block inverse
    // (k_block_jacobi's rule), so M^-1 keeps the stiffness scaling.
    double gmax = 0;
    for (int i = 0; i < n; ++i) gmax = fmax(gmax, fabs(G[i][i]));
    const double thr = 1e-12 * gmax;
    double Inv[6][6];
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) Inv[i][j] = (i == j) ? 1.0 : 0.0;
    bool ok = true;
    for (int c = 0; c < 6; ++c) {
      ok = ok && G[c][c] > thr;
      const double ip = G[c][c] > thr ? 1.0 / G[c][c] : 0.0;
      for (int j = 0; j < 6; ++j) {
        G[c][j] *= ip;
        Inv[c][j] *= ip;
      }
      for (int i = 0; i < 6; ++i)
        if (i != c) {
          const double f = G[i][c];
          for (int j = 0; j < 6; ++j) {
            G[i][j] -= f * G[c][j];
            Inv[i][j] -= f * Inv[c][j];
          }
        }
    }
    const int me = (v == a) ? 0 : 3, ot = 3 - me;
    double* o = minv2 + 18 * (int64_t)v;
    if (ok) {  // symmetrized: the partner stores the transpose of this cross block
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          o[3 * i + j] = 0.5 * (Inv[me + i][me + j] + Inv[me + j][me + i]);
          o[9 + 3 * i + j] = pv < 0 ? 0.0 : 0.5 * (Inv[me + i][ot + j] + Inv[ot + j][me + i]);
        }
    } else {  // own masked 3x3 block (k_block_jacobi)
      double D[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      add_block(M, v, v, D);
      D[0] += M.shift;
      D[4] += M.shift;
      D[8] += M.shift;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          if (mask[3 * v + i] == 0 || mask[3 * v + j] == 0) D[3 * i + j] = (i == j) ? 1.0 : 0.0;
      const double c00 = D[4] * D[8] - D[5] * D[7], c01 = D[2] * D[7] - D[1] * D[8], c02 = D[1] * D[5] - D[2] * D[4];
      const double c10 = D[5] * D[6] - D[3] * D[8], c11 = D[0] * D[8] - D[2] * D[6], c12 = D[2] * D[3] - D[0] * D[5];
      const double c20 = D[3] * D[7] - D[4] * D[6], c21 = D[1] * D[6] - D[0] * D[7], c22 = D[0] * D[4] - D[1] * D[3];
      const double det = D[0] * c00 + D[1] * c10 + D[2] * c20;
      for (int q = 0; q < 18; ++q) o[q] = 0;
      if (det != 0 && isfinite(det)) {
        const double id = 1.0 / det;
        o[0] = c00 * id; o[1] = c01 * id; o[2] = c02 * id;
        o[3] = c10 * id; o[4] = c11 * id; o[5] = c12 * id;
        o[6] = c20 * id; o[7] = c21 * id; o[8] = c22 * id;
      } else {
        for (int q = 0; q < 3; ++q) o[4 * q] = D[4 * q] != 0 ? 1.0 / D[4 * q] : 1.0;
      }
    }
  }
}

__device__ __forceinline__ d3 pair_apply(const double* __restrict__ minv2, int v, d3 rv, d3 rp) {
  const double* m = minv2 + 18 * (int64_t)v;
  return bmv(m, rv) + bmv(m + 9, rp);
}

// K9b with the pair preconditioner: r ping-pongs (r_in -> r_out) so a thread
// can form its partner's new residual r_p = r_in[p] - alpha q[p] itself.
template <bool kCoarse>
__global__ void __launch_bounds__(kThreads) k_update_cg_pair(int nv, const double* __restrict__ p,
                                                             const double* __restrict__ q, double* __restrict__ x,
                                                             const double* __restrict__ r_in,
                                                             double* __restrict__ r_out, double* __restrict__ z,
                                                             const double* __restrict__ minv2,
                                                             const int32_t* __restrict__ pair, double* scal,
                                                             RedSlot rs) {
  const double a = scal[2];
  double dots[2] = {0, 0};
  __shared__ double stg[kThreads / 32][3][96];
  const int lane = threadIdx.x & 31;
  double(*st)[96] = stg[threadIdx.x >> 5];
  for (int v = blockIdx.x * kThreads + threadIdx.x; v - lane < nv; v += gridDim.x * kThreads) {
    const bool in = v < nv;
    const int vv = in ? v : nv - 1;
    const d3 xv = ld3nc(x, vv) + a * ld3nc(p, vv);
    const d3 rv = ld3nc(r_in, vv) - a * ld3nc(q, vv);
    const int pp = pair[vv];
    const d3 rp = pp < 0 ? mk3(0, 0, 0) : ld3nc(r_in, pp) - a * ld3nc(q, pp);
    const d3 zv = pair_apply(minv2, vv, rv, rp);
    const double xa[3] = {xv.x, xv.y, xv.z}, ra[3] = {rv.x, rv.y, rv.z}, za[3] = {zv.x, zv.y, zv.z};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      st[0][3 * lane + c] = xa[c];
      st[1][3 * lane + c] = ra[c];
      st[2][3 * lane + c] = za[c];
    }
    __syncwarp();
    const int64_t base = 3 * (int64_t)(v - lane);
    const int64_t lim = 3 * (int64_t)nv - base;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int o = 32 * j + lane;
      if (o < lim) {
        x[base + o] = st[0][o];
        r_out[base + o] = st[1][o];
        z[base + o] = st[2][o];
      }
    }
    __syncwarp();
    if (in) {
      dots[0] += dot(rv, zv);
      dots[1] += dot(rv, rv);
    }
  }
  double out[2];
  if (block_reduce_last<2>(dots, rs, out) && threadIdx.x == 0) {
    if (kCoarse) {  // r.z completed by the coarse solve (k_coarse_apply)
      scal[6] = out[0];
    } else {
      const double rz_old = scal[0];
      scal[3] = rz_old != 0 ? out[0] / rz_old : 0.0;  // beta
      scal[0] = out[0];                                // rz
    }
    scal[4] = out[1];  // rr
  }
}

// PCG init with the pair preconditioner (z = M^-1 r, r = -mask .* grad)
template <bool kCoarse>
__global__ void __launch_bounds__(kThreads) k_pcg_init_pair(int nv, const double* __restrict__ grad,
                                                            const double* __restrict__ mask,
                                                            const double* __restrict__ minv2,
                                                            const int32_t* __restrict__ pair,
                                                            double* __restrict__ x, double* __restrict__ r,
                                                            double* __restrict__ z, double* __restrict__ p,
                                                            double* scal, RedSlot rs) {
  double dots[2] = {0, 0};
  for (int v = blockIdx.x * kThreads + threadIdx.x; v < nv; v += gridDim.x * kThreads) {
    const d3 m = ld3(mask, v), g = ld3(grad, v);
    const d3 rv = mk3(-m.x * g.x, -m.y * g.y, -m.z * g.z);
    const int pp = pair[v];
    d3 rp = mk3(0, 0, 0);
    if (pp >= 0) {
      const d3 mp = ld3(mask, pp), gp = ld3(grad, pp);
      rp = mk3(-mp.x * gp.x, -mp.y * gp.y, -mp.z * gp.z);
    }
    const d3 zv = pair_apply(minv2, v, rv, rp);
    const double ra[3] = {rv.x, rv.y, rv.z}, za[3] = {zv.x, zv.y, zv.z};
    for (int k = 0; k < 3; ++k) {
      x[3 * v + k] = 0;
      p[3 * v + k] = 0;
      r[3 * v + k] = ra[k];
      z[3 * v + k] = za[k];
    }
    dots[0] += dot(rv, zv);
    dots[1] += dot(rv, rv);
  }
  double out[2];
  if (block_reduce_last<2>(dots, rs, out) && threadIdx.x == 0) {
    scal[kCoarse ? 6 : 0] = out[0];
    scal[3] = 0;
    scal[4] = out[1];
    scal[5] = out[1];
    scal[8] = 0;
  }
}

// PCG init: x = p = 0, r = b = -mask.*grad, z = Minv r; rz, rr, bb; beta = 0.
template <bool kCoarse>
__global__ void __launch_bounds__(kThreads) k_pcg_init(int nv, const double* __restrict__ grad,
                                                       const double* __restrict__ mask, const double* __restrict__ minv,
                                                       double* __restrict__ x, double* __restrict__ r,
                                                       double* __restrict__ z, double* __restrict__ p, double* scal,
                                                       RedSlot rs) {
  double dots[2] = {0, 0};
  for (int v = blockIdx.x * kThreads + threadIdx.x; v < nv; v += gridDim.x * kThreads) {
    const d3 m = ld3(mask, v), g = ld3(grad, v);
    const d3 rv = mk3(-m.x * g.x, -m.y * g.y, -m.z * g.z);
    const d3 zv = bmv(minv + 9 * (int64_t)v, rv);
    const double ra[3] = {rv.x, rv.y, rv.z}, za[3] = {zv.x, zv.y, zv.z};
    for (int k = 0; k < 3; ++k) {
      x[3 * v + k] = 0;
      p[3 * v + k] = 0;
      r[3 * v + k] = ra[k];
      z[3 * v + k] = za[k];
    }
    dots[0] += dot(rv, zv);
    dots[1] += dot(rv, rv);
  }
  double out[2];
  if (block_reduce_last<2>(dots, rs, out) && threadIdx.x == 0) {
    scal[kCoarse ? 6 : 0] = out[0];  // rz (smoother part when the coarse solve completes it)
    scal[3] = 0;                     // beta: first direction p = z
    scal[4] = out[1];                // rr
    scal[5] = out[1];                // bb
    scal[8] = 0;                     // non-positive curvature count
  }
}

// ---------------------------------------------------------------------------
// Two-level PCG iteration kernels (coarse.cuh). With the coarse space on, one
// PCG iteration is three kernels: the SpMV (k_spmv_cg), the update fused with
// the restriction (k_update_agg), and the coarse solve fused with the
// prolongation (k_coarse_prolong). Both fused kernels run one CTA per
// aggregate over its vertex list, so the per-aggregate sums are CTA-local
// fixed-order reductions (deterministic), and every z entry is completed by
// the CTA that owns its vertex.

// CTA sum of W values in warp order (thread 0 holds the result): thread q
// sums value q over the warps, so the W sums run side by side
template <int W, int NT>
__device__ __forceinline__ void cta_sum(double (&v)[W], double (&sh)[NT / 32][W]) {
  __shared__ double tot[W];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < W; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < W; ++q) sh[wid][q] = v[q];
  __syncthreads();
  if (threadIdx.x < W) {
    double t = 0;
    for (int w = 0; w < NT / 32; ++w) t += sh[w][threadIdx.x];
    tot[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < W; ++q) v[q] = tot[q];
}

// x += alpha p, r = r_in - alpha q, z = M1^-1 r (pair or 3x3 block-Jacobi);
// s_a = S P^T r over the aggregate; r.z (smoother part) and r.r by the last block.
constexpr int kAggThreads = 1024;  // one CTA per aggregate: all of its vertices in flight at once
template <bool kPair>
__global__ void __launch_bounds__(kAggThreads) k_update_agg(
    const int32_t* __restrict__ agg_off, const int32_t* __restrict__ agg_verts, const double* __restrict__ dvec,
    const double* __restrict__ mask, const double* __restrict__ scale, const double* __restrict__ p,
    const double* __restrict__ q, double* __restrict__ x, const double* r_in, double* r_out,
    double* __restrict__ z, const double* __restrict__ minv, const int32_t* __restrict__ pair,
    double* __restrict__ s, double* scal, RedSlot rs) {
  __shared__ double sh[kAggThreads / 32][8];
  const int a = blockIdx.x;
  const double al = scal[2];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // t(3), w(3), rz, rr
  const int e1 = agg_off[a + 1];
  for (int e = agg_off[a] + threadIdx.x; e < e1; e += kAggThreads) {
    const int v = agg_verts[e];
    const d3 xv = ld3nc(x, v) + al * ld3nc(p, v);
    const d3 rv = ld3nc(r_in, v) - al * ld3nc(q, v);
    d3 zv;
    if (kPair) {
      const int pp = pair[v];
      const d3 rp = pp < 0 ? mk3(0, 0, 0) : ld3nc(r_in, pp) - al * ld3nc(q, pp);
      zv = pair_apply(minv, v, rv, rp);
    } else {
      zv = bmv(minv + 9 * (int64_t)v, rv);
    }
    x[3 * v] = xv.x;
    x[3 * v + 1] = xv.y;
    x[3 * v + 2] = xv.z;
    r_out[3 * v] = rv.x;
    r_out[3 * v + 1] = rv.y;
    r_out[3 * v + 2] = rv.z;
    z[3 * v] = zv.x;
    z[3 * v + 1] = zv.y;
    z[3 * v + 2] = zv.z;
    const d3 m = ld3(mask, v);
    const d3 mr = mk3(m.x * rv.x, m.y * rv.y, m.z * rv.z);
    const d3 w = cross(ld3(dvec, v), mr);
    acc[0] += mr.x;
    acc[1] += mr.y;
    acc[2] += mr.z;
    acc[3] += w.x;
    acc[4] += w.y;
    acc[5] += w.z;
    acc[6] += dot(rv, zv);
    acc[7] += dot(rv, rv);
  }
  cta_sum<8, kAggThreads>(acc, sh);
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) s[6 * a + k] = acc[k] * scale[6 * a + k];
  double d[2] = {threadIdx.x == 0 ? acc[6] : 0.0, threadIdx.x == 0 ? acc[7] : 0.0};
  double out[2];
  if (block_reduce_last<2, kAggThreads>(d, rs, out) && threadIdx.x == 0) {
    scal[6] = out[0];  // r.z of the smoother; k_coarse_prolong completes it
    scal[4] = out[1];  // rr
  }
}

// y_a = S (Ainv s')_a for the CTA's aggregate (6 rows, one warp each, loads
// unrolled), z_v += Phi_v y_a over its vertices, and s.y -> rz = r.M1^-1 r +
// s.y, beta (last block). kInit: first direction (beta = 0).
template <bool kInit>
__global__ void __launch_bounds__(kAggThreads) k_coarse_prolong(
    int n_pad, const double* __restrict__ Ainv, const double* __restrict__ scale, const double* __restrict__ s,
    const int32_t* __restrict__ agg_off, const int32_t* __restrict__ agg_verts, const double* __restrict__ dvec,
    const double* __restrict__ mask, double* __restrict__ z, double* scal, RedSlot rs) {
  __shared__ double ya[6], sy[6];
  __shared__ double part[kAggThreads / 32][6];
  const int a = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  {  // the aggregate's 6 coarse rows dotted with s by the whole CTA: every
     // thread loads its column slice of each row at once (one L2 round trip),
     // warp sums, then the 32 warp partials in warp order (deterministic)
    double acc[6] = {0, 0, 0, 0, 0, 0};
    const double* rows = Ainv + (int64_t)(6 * a) * n_pad;
    for (int j = threadIdx.x; j < n_pad; j += kAggThreads) {
      const double sj = __ldg(s + j);
#pragma unroll
      for (int r = 0; r < 6; ++r) acc[r] += __ldg(rows + (int64_t)r * n_pad + j) * sj;
    }
#pragma unroll
    for (int r = 0; r < 6; ++r) acc[r] = warp_sum(acc[r]);
    if (lane == 0)
#pragma unroll
      for (int r = 0; r < 6; ++r) part[wid][r] = acc[r];
    __syncthreads();
    if (threadIdx.x < 6) {
      const int r = threadIdx.x, i = 6 * a + r;
      double t = 0;
      for (int w = 0; w < kAggThreads / 32; ++w) t += part[w][r];
      ya[r] = scale[i] * t;
      sy[r] = s[i] * t;
    }
  }
  __syncthreads();
  const d3 t = mk3(ya[0], ya[1], ya[2]), om = mk3(ya[3], ya[4], ya[5]);
  const int e1 = agg_off[a + 1];
  for (int e = agg_off[a] + threadIdx.x; e < e1; e += kAggThreads) {
    const int v = agg_verts[e];
    const d3 u = t + cross(om, ld3(dvec, v));
    const d3 m = ld3(mask, v);
    z[3 * v] += m.x * u.x;
    z[3 * v + 1] += m.y * u.y;
    z[3 * v + 2] += m.z * u.z;
  }
  double d[1] = {threadIdx.x == 0 ? ((sy[0] + sy[1]) + (sy[2] + sy[3])) + (sy[4] + sy[5]) : 0.0};
  double out[1];
  if (block_reduce_last<1, kAggThreads>(d, rs, out) && threadIdx.x == 0) {
    const double rz = scal[6] + out[0];
    if (kInit) {
      scal[0] = rz;
      scal[3] = 0;
    } else {
      const double rz_old = scal[0];
      scal[3] = rz_old != 0 ? rz / rz_old : 0.0;
      scal[0] = rz;
    }
  }
}

// ---------------------------------------------------------------------------
// Small systems (C1, C4, the patch test): the whole two-level PCG iteration
// loop in ONE cooperative launch. The three-kernel iteration is latency-bound
// there (~27 us for 1,253 vertices); here it is three grid barriers:
//   A  p = z + beta p_old (own rows) and q = mask .* (H + shift) p, p.q partial
//   B  per aggregate (CTA-owned): x += alpha p, r = r_in - alpha q, z = M1^-1 r
//      (vertex pairs), restriction s_a, r.z and r.r partials
//   C  per aggregate: its 6 coarse rows of y = S Ac^+ s', z += Phi y, s.y partial
// then every thread sums the per-CTA partials in CTA order (the same values in
// every CTA: deterministic) and takes the same convergence / stagnation /
// failure decisions. Vectors written inside the kernel are read with ld.cg
// (L2): the L1s are not coherent across SMs. The drift check of pcg_core runs
// every kDriftWindow iterations on the true residual.
constexpr int kCoopThreads = 256, kCoopMaxCtas = 64;
constexpr int kCoopMaxRows = 16384;  // systems up to this many vertices run k_pcg_coop
struct CoopArgs {
  MatSet M;
  int nv;
  const double* mask;
  const double* grad;  // rhs = -mask .* grad (the drift check)
  const double* minv2;
  const int32_t* pair;
  const int32_t* agg_off;
  const int32_t* agg_verts;
  const double* dvec;
  const double* scale;
  const double* inv;
  int n_agg, n_pad;
  double* x;
  double* r0;
  double* r1;
  double* z;
  double* p0;
  double* p1;
  double* q;
  double* s;
  double* part;  // [4][kCoopMaxCtas]
  double* scal;  // in: [0] rz [4] rr [5] bb; out: [0] rz [4] rr [9] status [10] iterations
  double tol2;
  int maxit;
  int drift_check;
  double drift_tol;  // kDriftFail * tol
};
__device__ __forceinline__ d3 ldcg3(const double* p, int v) {
  return mk3(__ldcg(p + 3 * (int64_t)v), __ldcg(p + 3 * (int64_t)v + 1), __ldcg(p + 3 * (int64_t)v + 2));
}
// CTA sum of W values (thread 0 of the CTA holds them), fixed order
template <int W>
__device__ __forceinline__ void coop_cta_sum(double (&v)[W], double (*sh)[W]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < W; ++q) v[q] = warp_sum(v[q]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < W; ++q) sh[wid][q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < W; ++q) {
      double t = 0;
      for (int w = 0; w < kCoopThreads / 32; ++w) t += sh[w][q];
      v[q] = t;
    }
}
__global__ void __launch_bounds__(kCoopThreads) k_pcg_coop(CoopArgs A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[kCoopThreads / 32][8];
  __shared__ double ya[6];
  const int G = gridDim.x, b = blockIdx.x, t = threadIdx.x, lane = t & 31, sub = lane & 7;
  const int gt = b * kCoopThreads + t, nthreads = G * kCoopThreads;
  const MatSet& M = A.M;
  double rz = __ldcg(A.scal), rr = __ldcg(A.scal + 4);
  const double bb = __ldcg(A.scal + 5), target = A.tol2 * bb;
  double beta = 0;
  int it = 0, status = 0;
  double win_min = INFINITY, prev_min = INFINITY;
  while (rr > target && it < A.maxit) {
    double* p_old = (it & 1) ? A.p1 : A.p0;
    double* p_new = (it & 1) ? A.p0 : A.p1;
    const double* r_in = (it & 1) ? A.r1 : A.r0;
    double* r_out = (it & 1) ? A.r0 : A.r1;
    // A: SpMV, 8 lanes per row, rows grid-strided
    double pq = 0;
    for (int v0 = gt >> 3; v0 - (lane >> 3) < A.nv; v0 += nthreads >> 3) {  // warp-uniform bound
      const int v = v0;
      d3 acc0 = mk3(0, 0, 0), acc1 = mk3(0, 0, 0);
      if (v < A.nv) {
        const Bcsr& E = M.el;
        if (M.hv) {
          const int a0 = __ldg(E.rowptr + v), a1 = __ldg(E.rowptr + v + 1);
          const int2* ch = reinterpret_cast<const int2*>(M.hix);
          for (int k = a0 + sub; k < a1; k += 8) {
            const int2 c = __ldg(ch + k);
            acc0 = acc0 + half_bmv(c.y, M.hv, M.hn, ldcg3(A.z, c.x) + beta * ldcg3(p_old, c.x));
          }
        } else {
          const int a0 = __ldg(E.rowptr + v), a1 = __ldg(E.rowptr + v + 1);
          for (int k = a0 + sub; k < a1; k += 8) {
            const int j = __ldg(E.cols + k);
            acc0 = acc0 + bmv_ro(E, k, ldcg3(A.z, j) + beta * ldcg3(p_old, j));
          }
        }
      }
      d3 acc = acc0 + acc1;
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
      }
      if (sub == 0 && v < A.nv) {
        const d3 m = ld3(A.mask, v);
        const d3 pv = ldcg3(A.z, v) + beta * ldcg3(p_old, v);
        if (M.shift != 0) acc = acc + M.shift * pv;
        const d3 y = mk3(m.x * acc.x, m.y * acc.y, m.z * acc.z);
        __stcg(A.q + 3 * (int64_t)v, y.x);
        __stcg(A.q + 3 * (int64_t)v + 1, y.y);
        __stcg(A.q + 3 * (int64_t)v + 2, y.z);
        __stcg(p_new + 3 * (int64_t)v, pv.x);
        __stcg(p_new + 3 * (int64_t)v + 1, pv.y);
        __stcg(p_new + 3 * (int64_t)v + 2, pv.z);
        pq += dot(pv, y);
      }
    }
    {
      double v1[1] = {pq};
      coop_cta_sum<1>(v1, reinterpret_cast<double(*)[1]>(sh));
      if (t == 0) __stcg(A.part + b, v1[0]);
    }
    grid.sync();
    pq = 0;
    for (int i = 0; i < G; ++i) pq += __ldcg(A.part + i);
    const double alpha = pq != 0 ? rz / pq : 0.0;
    // B: per aggregate: update, smoother, restriction
    double rzs = 0, rrs = 0;
    for (int a = b; a < A.n_agg; a += G) {
      double acc[6] = {0, 0, 0, 0, 0, 0};
      const int e1 = __ldg(A.agg_off + a + 1);
      for (int e = __ldg(A.agg_off + a) + t; e < e1; e += kCoopThreads) {
        const int v = __ldg(A.agg_verts + e);
        const d3 xv = ldcg3(A.x, v) + alpha * ldcg3(p_new, v);
        const d3 rv = ldcg3(r_in, v) - alpha * ldcg3(A.q, v);
        const int pp = __ldg(A.pair + v);
        const d3 rp = pp < 0 ? mk3(0, 0, 0) : ldcg3(r_in, pp) - alpha * ldcg3(A.q, pp);
        const d3 zv = pair_apply(A.minv2, v, rv, rp);
        __stcg(A.x + 3 * (int64_t)v, xv.x);
        __stcg(A.x + 3 * (int64_t)v + 1, xv.y);
        __stcg(A.x + 3 * (int64_t)v + 2, xv.z);
        __stcg(r_out + 3 * (int64_t)v, rv.x);
        __stcg(r_out + 3 * (int64_t)v + 1, rv.y);
        __stcg(r_out + 3 * (int64_t)v + 2, rv.z);
        __stcg(A.z + 3 * (int64_t)v, zv.x);
        __stcg(A.z + 3 * (int64_t)v + 1, zv.y);
        __stcg(A.z + 3 * (int64_t)v + 2, zv.z);
        const d3 m = ld3(A.mask, v);
        const d3 mr = mk3(m.x * rv.x, m.y * rv.y, m.z * rv.z);
        const d3 w = cross(ld3(A.dvec, v), mr);
        acc[0] += mr.x;
        acc[1] += mr.y;
        acc[2] += mr.z;
        acc[3] += w.x;
        acc[4] += w.y;
        acc[5] += w.z;
        rzs += dot(rv, zv);
        rrs += dot(rv, rv);
      }
      coop_cta_sum<6>(acc, reinterpret_cast<double(*)[6]>(sh));
      if (t == 0)
        for (int k = 0; k < 6; ++k) __stcg(A.s + 6 * a + k, acc[k] * __ldg(A.scale + 6 * a + k));
    }
    {
      double v2[2] = {rzs, rrs};
      coop_cta_sum<2>(v2, reinterpret_cast<double(*)[2]>(sh));
      if (t == 0) {
        __stcg(A.part + kCoopMaxCtas + b, v2[0]);
        __stcg(A.part + 2 * kCoopMaxCtas + b, v2[1]);
      }
    }
    grid.sync();
    // C: coarse rows of the CTA's aggregates, prolongation, s.y
    double sy = 0;
    for (int a = b; a < A.n_agg; a += G) {
      double acc[6] = {0, 0, 0, 0, 0, 0};
      const double* rows = A.inv + (int64_t)(6 * a) * A.n_pad;
      for (int j = t; j < A.n_pad; j += kCoopThreads) {
        const double sj = __ldcg(A.s + j);
#pragma unroll
        for (int k = 0; k < 6; ++k) acc[k] += __ldg(rows + (int64_t)k * A.n_pad + j) * sj;
      }
      coop_cta_sum<6>(acc, reinterpret_cast<double(*)[6]>(sh));
      if (t == 0) {
        double syl = 0;
        for (int k = 0; k < 6; ++k) {
          const int i = 6 * a + k;
          ya[k] = __ldg(A.scale + i) * acc[k];
          syl += __ldcg(A.s + i) * acc[k];
        }
        sy += syl;
      }
      __syncthreads();
      const d3 tt = mk3(ya[0], ya[1], ya[2]), om = mk3(ya[3], ya[4], ya[5]);
      const int e1 = __ldg(A.agg_off + a + 1);
      for (int e = __ldg(A.agg_off + a) + t; e < e1; e += kCoopThreads) {
        const int v = __ldg(A.agg_verts + e);
        const d3 u = tt + cross(om, ld3(A.dvec, v));
        const d3 m = ld3(A.mask, v);
        const d3 zv = ldcg3(A.z, v);
        __stcg(A.z + 3 * (int64_t)v, zv.x + m.x * u.x);
        __stcg(A.z + 3 * (int64_t)v + 1, zv.y + m.y * u.y);
        __stcg(A.z + 3 * (int64_t)v + 2, zv.z + m.z * u.z);
      }
      __syncthreads();
    }
    if (t == 0) __stcg(A.part + 3 * kCoopMaxCtas + b, sy);
    grid.sync();
    double rzn = 0, rrn = 0, syt = 0;
    for (int i = 0; i < G; ++i) {
      rzn += __ldcg(A.part + kCoopMaxCtas + i);
      rrn += __ldcg(A.part + 2 * kCoopMaxCtas + i);
      syt += __ldcg(A.part + 3 * kCoopMaxCtas + i);
    }
    rzn += syt;
    beta = rz != 0 ? rzn / rz : 0.0;
    rz = rzn;
    rr = rrn;
    ++it;
    if (!isfinite(rr) || !(rz > 0)) {
      status = 1;
      break;
    }
    if (A.drift_check && it % kDriftWindow == 0) {  // true residual ||mask .* (grad + (H + shift) x)||
      double tr = 0;
      for (int v0 = gt >> 3; v0 - (lane >> 3) < A.nv; v0 += nthreads >> 3) {
        const int v = v0;
        d3 acc = mk3(0, 0, 0);
        if (v < A.nv) {
          const Bcsr& E = M.el;
          const int a0 = __ldg(E.rowptr + v), a1 = __ldg(E.rowptr + v + 1);
          for (int k = a0 + sub; k < a1; k += 8) acc = acc + bmv_ro(E, k, ldcg3(A.x, __ldg(E.cols + k)));
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
          acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
        }
        if (sub == 0 && v < A.nv) {
          const d3 m = ld3(A.mask, v), gg = ld3(A.grad, v), xv = ldcg3(A.x, v);
          if (M.shift != 0) acc = acc + M.shift * xv;
          const d3 e = mk3(m.x * (acc.x + gg.x), m.y * (acc.y + gg.y), m.z * (acc.z + gg.z));
          tr += dot(e, e);
        }
      }
      double v1[1] = {tr};
      coop_cta_sum<1>(v1, reinterpret_cast<double(*)[1]>(sh));
      if (t == 0) __stcg(A.part + b, v1[0]);
      grid.sync();
      tr = 0;
      for (int i = 0; i < G; ++i) tr += __ldcg(A.part + i);
      const double true_rel = sqrt(tr / bb), rec_rel = sqrt(rr / bb);
      if (true_rel - rec_rel > A.drift_tol || (M.shift == 0 && true_rel > kDivergeRel)) {
        status = 2;
        break;
      }
      grid.sync();  // part reused by the next phase A
    }
    win_min = fmin(win_min, rr);
    if (it % kStagWindowCoarse == 0) {
      if (it >= 2 * kStagWindowCoarse && !(win_min < 0.5 * prev_min) && rr > 1e-8 * bb) break;  // stagnated
      prev_min = fmin(prev_min, win_min);
      win_min = INFINITY;
    }
  }
  if (b == 0 && t == 0) {
    A.scal[0] = rz;
    A.scal[4] = rr;
    A.scal[9] = (double)status;
    A.scal[10] = (double)it;
  }
}

// Block-Jacobi: Minv_v = inverse of the masked 3x3 diagonal block.
// diagonal block of row v copied to d[9] (either layout); false if absent
__device__ __forceinline__ bool get_diag(const Bcsr& A, int v, double* d) {
  int lo = A.rowptr[v], hi = A.rowptr[v + 1];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A.cols[mid] < v) lo = mid + 1; else hi = mid;
  }
  if (!(lo < A.rowptr[v + 1] && A.cols[lo] == v)) return false;
  const double* b = A.vals + (int64_t)lo * A.bs;
  for (int q = 0; q < 9; ++q) d[q] = b[q * A.cs];
  return true;
}

__global__ void k_block_jacobi(int nv, MatSet M, const double* __restrict__ mask, double* __restrict__ minv) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    double D[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    get_diag(M.el, v, D);
    for (int k = 0; k < M.np; ++k) {
      double c[9];
      if (get_diag(M.c[k], v, c))
        for (int q = 0; q < 9; ++q) D[q] += c[q];
    }
    D[0] += M.shift;
    D[4] += M.shift;
    D[8] += M.shift;
    const double m[3] = {mask[3 * v], mask[3 * v + 1], mask[3 * v + 2]};
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        if (m[a] == 0 || m[b] == 0) D[3 * a + b] = (a == b) ? 1.0 : 0.0;
      }
    const double c00 = D[4] * D[8] - D[5] * D[7], c01 = D[2] * D[7] - D[1] * D[8], c02 = D[1] * D[5] - D[2] * D[4];
    const double c10 = D[5] * D[6] - D[3] * D[8], c11 = D[0] * D[8] - D[2] * D[6], c12 = D[2] * D[3] - D[0] * D[5];
    const double c20 = D[3] * D[7] - D[4] * D[6], c21 = D[1] * D[6] - D[0] * D[7], c22 = D[0] * D[4] - D[1] * D[3];
    const double det = D[0] * c00 + D[1] * c10 + D[2] * c20;
    double* o = minv + 9 * (int64_t)v;
    if (det != 0 && isfinite(det)) {
      const double id = 1.0 / det;
      o[0] = c00 * id; o[1] = c01 * id; o[2] = c02 * id;
      o[3] = c10 * id; o[4] = c11 * id; o[5] = c12 * id;
      o[6] = c20 * id; o[7] = c21 * id; o[8] = c22 * id;
    } else {  // point Jacobi fallback
      for (int q = 0; q < 9; ++q) o[q] = 0;
      for (int a = 0; a < 3; ++a) o[4 * a] = D[4 * a] != 0 ? 1.0 / D[4 * a] : 1.0;
    }
  }
}

// True residual of an accepted solve (solver.hpp:349-356 accepts a solve iff
// ||M s - rhs||_inf <= 1e-6 ||rhs||_inf): res = mask .* (H dx + shift dx) + mask .* grad
// (rhs = -mask .* grad). Sums of res^2 and rhs^2 by the fixed-order block
// reduction -> out[0..1]; max |res|, max |rhs| as ordered bits -> red[0..1].
__global__ void __launch_bounds__(kThreads) k_true_resid(int nv, MatSet M, const double* __restrict__ mask,
                                                         const double* __restrict__ dx,
                                                         const double* __restrict__ grad, double* __restrict__ rvec,
                                                         double* out, unsigned long long* red, RedSlot rs) {
  const int lane = threadIdx.x & 31;
  double d[2] = {0, 0};
  unsigned long long mr = 0, mb = 0;
  const int nw = gridDim.x * (kThreads / 32);
  for (int v = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); v < nv; v += nw) {
    d3 acc = mk3(0, 0, 0);
    const Bcsr* mats[1 + kMaxPairs] = {&M.el, &M.c[0], &M.c[1], &M.c[2], &M.c[3]};
    for (int m = 0; m <= M.np; ++m) {
      const Bcsr& A = *mats[m];
      for (int k = A.rowptr[v] + lane; k < A.rowptr[v + 1]; k += 32) acc = acc + bmv_ro(A, k, ld3(dx, A.cols[k]));
    }
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    acc.z = warp_sum(acc.z);
    if (lane == 0) {
      const d3 m = ld3(mask, v), g = ld3(grad, v), dv = ld3(dx, v);
      const double y[3] = {acc.x + M.shift * dv.x, acc.y + M.shift * dv.y, acc.z + M.shift * dv.z};
      const double ma[3] = {m.x, m.y, m.z}, ga[3] = {g.x, g.y, g.z};
      for (int a = 0; a < 3; ++a) {
        const double r = ma[a] * y[a] + ma[a] * ga[a], b = ma[a] * ga[a];
        rvec[3 * v + a] = r;
        d[0] += r * r;
        d[1] += b * b;
        const unsigned long long br = ord_bits(fabs(r)), bb = ord_bits(fabs(b));
        mr = br > mr ? br : mr;
        mb = bb > mb ? bb : mb;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
  }
  if (lane == 0) {
    atomicMax(red, mr);
    atomicMax(red + 1, mb);
  }
  double o2[2];
  if (block_reduce_last<2>(d, rs, o2) && threadIdx.x == 0) {
    out[0] = o2[0];
    out[1] = o2[1];
  }
}

// Sum of the free-dof diagonal entries of H (elastic + contact) -> out[0]
// (solver.hpp:333-336, the regularization scale).
__global__ void __launch_bounds__(kThreads) k_diag_sum(int nv, MatSet M, const double* __restrict__ mask,
                                                       double* out, RedSlot rs) {
  double acc[1] = {0};
  for (int v = blockIdx.x * kThreads + threadIdx.x; v < nv; v += gridDim.x * kThreads) {
    double d[3] = {0, 0, 0};
    double e[9];
    if (get_diag(M.el, v, e))
      for (int a = 0; a < 3; ++a) d[a] = e[4 * a];
    for (int k = 0; k < M.np; ++k) {
      double c[9];
      if (get_diag(M.c[k], v, c))
        for (int a = 0; a < 3; ++a) d[a] += c[4 * a];
    }
    for (int a = 0; a < 3; ++a)
      if (mask[3 * v + a] != 0) acc[0] += d[a];
  }
  double o[1];
  if (block_reduce_last<1>(acc, rs, o) && threadIdx.x == 0) out[0] = o[0];
}

// Elastic gradient K_el (x - rest) -> grad = g_el + sum_pairs g_c - lambda f_ext.
// Also residual = max |grad_d| over free dofs (order-free max).
__global__ void k_grad_total(int nv, Bcsr K, const double* __restrict__ x, const double* __restrict__ rest,
                             const double* __restrict__ fext, double lambda, const double* const* __restrict__ gc,
                             int np, const double* __restrict__ mask, double* __restrict__ gel,
                             double* __restrict__ grad, unsigned long long* red) {
  const int lane = threadIdx.x & 31;
  unsigned long long best = 0;
  const int nw = gridDim.x * (blockDim.x / 32);
  for (int v = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); v < nv; v += nw) {
    d3 acc = mk3(0, 0, 0);
    for (int k = K.rowptr[v] + lane; k < K.rowptr[v + 1]; k += 32) {
      const int j = K.cols[k];
      acc = acc + bmv(K.vals + 9 * (int64_t)k, ld3(x, j) - ld3(rest, j));
    }
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    acc.z = warp_sum(acc.z);
    if (lane == 0) {
      gel[3 * v] = acc.x;
      gel[3 * v + 1] = acc.y;
      gel[3 * v + 2] = acc.z;
      double g[3] = {acc.x, acc.y, acc.z};
      for (int k = 0; k < np; ++k)
        for (int a = 0; a < 3; ++a) g[a] += gc[k][3 * v + a];
      for (int a = 0; a < 3; ++a) {
        g[a] -= lambda * fext[3 * v + a];
        grad[3 * v + a] = g[a];
        if (mask[3 * v + a] != 0) {
          const unsigned long long b = ord_bits(fabs(g[a]));
          best = b > best ? b : best;
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0) atomicMax(red, best);
}

// Scalars for the line search: out = [g_el.dx, dx.K dx, f.dx] (K dx via SpMV).
__global__ void __launch_bounds__(kThreads) k_ls_coeffs(int nv, Bcsr K, const double* __restrict__ dx,
                                                        const double* __restrict__ gel,
                                                        const double* __restrict__ fext, double* out, RedSlot rs) {
  const int lane = threadIdx.x & 31;
  double d[3] = {0, 0, 0};
  const int nw = gridDim.x * (kThreads / 32);
  for (int v = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); v < nv; v += nw) {
    d3 acc = row_mv(K, v, dx, lane);
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    acc.z = warp_sum(acc.z);
    if (lane == 0) {
      const d3 dv = ld3(dx, v);
      d[0] += dot(ld3(gel, v), dv);
      d[1] += dot(dv, acc);
      d[2] += dot(ld3(fext, v), dv);
    }
  }
  double o[3];
  if (block_reduce_last<3>(d, rs, o) && threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) out[q] = o[q];
}

// Elastic energy 0.5 u.(K u) and external work f.u, u = x - rest.
__global__ void __launch_bounds__(kThreads) k_energy_el(int nv, const double* __restrict__ gel,
                                                        const double* __restrict__ x, const double* __restrict__ rest,
                                                        const double* __restrict__ fext, double* out, RedSlot rs) {
  double d[2] = {0, 0};
  for (int v = blockIdx.x * kThreads + threadIdx.x; v < nv; v += gridDim.x * kThreads) {
    const d3 u = ld3(x, v) - ld3(rest, v);
    d[0] += dot(ld3(gel, v), u);
    d[1] += dot(ld3(fext, v), u);
  }
  double o[2];
  if (block_reduce_last<2>(d, rs, o) && threadIdx.x == 0) {
    out[0] = 0.5 * o[0];
    out[1] = o[1];
  }
}

__global__ void k_add_into(int64_t n, const double* __restrict__ a, double* y) {  // y += a
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a[i] + y[i];
}
__global__ void k_axpy_to(int64_t n, const double* __restrict__ x, double a, const double* __restrict__ dx,
                          double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] + a * dx[i];
}

// max |x_v - ref_v| over a vertex list (pair_motion, solver.hpp:279-290)
__global__ void k_motion(int64_t n, const int32_t* __restrict__ verts, const double* __restrict__ x,
                         const double* __restrict__ ref, unsigned long long* red) {
  unsigned long long best = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int v = verts[i];
    const unsigned long long b = ord_bits(norm(ld3(x, v) - ld3(ref, v)));
    best = b > best ? b : best;
  }
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(red, best);
}

// Merged values: H_k = K_el[src0] + sum_p K_c,p[src1+p] (fixed order).
struct ValPtrs {
  const double* v[1 + kMaxPairs];
};
__global__ void k_merge(int64_t nnzb, int ns, const int32_t* __restrict__ src, ValPtrs V, double* __restrict__ out,
                        const int32_t* __restrict__ hix, double* __restrict__ hv, int64_t nh) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnzb; k += (int64_t)gridDim.x * blockDim.x) {
    double acc[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] = 0.0;
    for (int s = 0; s < ns; ++s) {
      const int32_t i = src[(int64_t)ns * k + s];
      if (i >= 0) {
        const double* b = V.v[s] + 9 * (int64_t)i;
#pragma unroll
        for (int q = 0; q < 9; ++q) acc[q] += b[q];
      }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) out[q * nnzb + k] = acc[q];  // component-major (coalesced SpMV loads)
    if (hv && hix[2 * k + 1] >= 0) {  // on/above the diagonal: the compact symmetric-half copy
      const int64_t i = hix[2 * k + 1];
#pragma unroll
      for (int q = 0; q < 8; ++q) hv[8 * i + q] = acc[q];
      hv[8 * nh + i] = acc[8];
    }
  }
}

// Symmetric-half numbering (MatSet::hix). k_half_count: per row, the blocks on
// and above the diagonal (columns are sorted); after the scan hoff[v] is the
// compact index of row v's first such block. k_half_index: (column, hix) of
// every union block; block (v, c), c < v, points at the stored (c, v), found by binary
// search in row c. A missing mirror (non-symmetric pattern) sets *bad.
__global__ void k_half_count(int nv, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                             int32_t* __restrict__ cnt) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    int c = 0;
    for (int k = rowptr[v]; k < rowptr[v + 1]; ++k) c += cols[k] >= v;
    cnt[v] = c;
  }
}
__global__ void k_half_index(int nv, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                             const int32_t* __restrict__ hoff, int32_t* __restrict__ hix, int* bad) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    int up = hoff[v];
    for (int k = rowptr[v]; k < rowptr[v + 1]; ++k) {
      const int c = cols[k];
      hix[2 * k] = c;
      if (c >= v) {
        hix[2 * k + 1] = up++;
        continue;
      }
      int lo = rowptr[c], hi = rowptr[c + 1];
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cols[mid] < v) lo = mid + 1;
        else hi = mid;
      }
      if (lo < rowptr[c + 1] && cols[lo] == v) {
        int before = 0;  // blocks of row c below its diagonal precede the stored ones
        for (int t = rowptr[c]; t < lo; ++t) before += cols[t] >= c;
        hix[2 * k + 1] = ~(hoff[c] + before);
      } else {
        hix[2 * k + 1] = 0;
        atomicExch(bad, 1);
      }
    }
  }
}

int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

}  // namespace

// ===========================================================================

struct Body {
  std::vector<double> verts;  // rest (local)
  std::vector<int32_t> tets;
  double E, nu, lambda, mu;
  int32_t offset, nv;
  std::vector<double> vol;   // per tet
  std::vector<double> grads; // per tet [4][3]
};

struct PairRt {
  std::unique_ptr<Ctx> c;
  gmcp_barrier_params params;
  DBuf<double> ref_pos;      // positions at sampling time
  DBuf<int32_t> motion_verts;  // slave.verts ++ master.verts
  std::vector<int64_t> scene_soff;  // batched: sample offsets per scene after the last load step
};

struct SystemImpl {
  int device = 0;
  CubScratch cub;  // CUB temp storage (bound per C-ABI call)
  cudaStream_t stream = nullptr;
  // batched independent scenes: contiguous vertex ranges per scene
  int32_t n_scenes = 1;
  std::vector<int32_t> vscene;       // scene of each vertex (empty: one scene)
  std::vector<int64_t> scene_voff;   // [S+1] vertex offsets
  std::vector<int64_t> scene_iters;  // Newton iterations per scene (last solve)
  std::vector<gmcp_step_stats> scene_stats;  // [load step][scene] StepStats of the last batched solve
  int32_t scene_stats_steps = 0;              // load steps completed
  int64_t n_dof = 0;
  int64_t launches = 0;
  std::vector<Body> bodies;
  std::vector<double> rest, f_ext, dirichlet;
  std::vector<uint8_t> fixed;
  std::vector<std::unique_ptr<PairRt>> pairs;
  // device
  DBuf<double> x, dx, xtry, rest_d, fext_d, mask_d, grad, gel, r, z, p, q, w, minv, scal, parts, lsco, eel;
  DBuf<double> minv2, r2;   // vertex-pair block-Jacobi: [v][3x6] rows, r ping-pong
  DBuf<int32_t> pair_d;      // vertex-pair partner (-1: none), from the elastic matrix
  bool has_pairs = false;
  // preconditioner of the single-system PCG (runtime: GMCP_PAIR_JACOBI, GMCP_COARSE, GMCP_COARSE_AGGS)
  bool use_pair = true, use_coarse = true;
  int coarse_aggs = 128;
  CoarseSpace cs;            // two-level coarse space (coarse.cuh)
  int64_t load_step = 0;     // current load step (coarse refresh policy)
  bool coarse_refresh_always = false;  // GMCP_COARSE_REFRESH=1: new coarse inverse every solve
  double coarse_drop = kCoarseDropDefault;  // GMCP_COARSE_DROP
  int coarse_scene_aggs = 24;          // batched scenes: aggregates per scene (GMCP_COARSE_SCENE_AGGS)
  int64_t u_gen = 0;         // union pattern generation (coarse pair lists follow it)
  DBuf<unsigned int> counter;
  DBuf<unsigned long long> redu;
  DBuf<int32_t> k_rowptr, k_cols;
  DBuf<double> k_vals;
  // merged Newton matrix H = K_el + sum_pairs K_c on the union pattern (PCG operand);
  // u_src[(1 + np) * k + s]: block index of union block k in the elastic (s = 0) /
  // pair s-1 matrix, or -1. Pattern rebuilt when a pair is re-sampled.
  DBuf<int32_t> u_rowptr, u_cols, u_src;
  DBuf<double> u_vals;
  DBuf<int32_t> u_hix, u_hoff;  // symmetric-half PCG operand (MatSet::hix / hv): single systems
  int64_t u_hn = 0;
  DBuf<double> u_half;
  bool u_half_ok = false;
  bool use_half = true;      // GMCP_HALF_SPMV=0 turns it off
  int64_t u_nnzb = 0;
  bool u_valid = false;
  struct UnionTmp {  // build_union scratch, reused across rebuilds
    DBuf<unsigned long long> keys, keys2, ukeys;
    DBuf<int64_t> vals, vals2;
    DBuf<int32_t> ucnt, uoff, nuniq, rowcnt;
    DBuf<int> bad;
  } utmp;
  DBuf<const double*> gc_ptrs;
  bool el_built = false;
  int64_t el_nnzb = 0;
  std::vector<double> x_host;
  // stats of the last solve
  int64_t pcg_iters_total = 0;
  // true residual of every linear solve since the last reset (gmcp_system_linear_stats):
  // ||H dx - rhs||_2 / ||rhs||_2 and the inf-norm ratio the reference's acceptance test uses
  double last_true_rel2 = 0, last_true_relinf = 0, true_rel2_max = 0, true_relinf_max = 0;
  int64_t n_linear_solves = 0, refinements = 0;
  int64_t drift_fails = 0;       // PCG solves failed early on a true/recursive residual gap (pcg_core)
  DBuf<double> coop_part;        // per-CTA partial sums of k_pcg_coop
  double last_solve_shift = -1;  // shift / pattern generation of the last pcg_core call (refinement passes)
  int64_t last_solve_ops = -1;
  int64_t coarse_fallbacks = 0;  // batched: scene solves re-run with block-Jacobi after a failed two-level solve
  DBuf<double> rt, xacc;  // true residual vector, accumulated solution (residual replacement)
  // optional host capture of the last linear system (gmcp_system_capture_linear_system)
  bool capture = false;
  std::vector<int32_t> cap_rowptr, cap_cols;
  std::vector<double> cap_vals, cap_mask, cap_grad, cap_dx;
  double cap_shift = 0;
  // Newton-iteration timing (gmcp_system_time_newton): stop after iter_limit
  int64_t iter_limit = 0;
  std::vector<double> iter_ms;
  std::vector<int64_t> iter_pcg;
  std::vector<int64_t> iter_active;  // batched: scenes iterated per loop pass
  // PCG chunk graphs timed with CUDA events on the solve stream (since the
  // last reset): device ms and iterations, for the PCG roofline in bench.py
  double pcg_ev_ms = 0;
  int64_t pcg_ev_iters = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // instantiated PCG chunk graph and the launch parameters it was captured with
  struct PcgKey {
    MatSet M;
    int nv, lanes, gsp, gup;
    const void* ptrs[14];
  } pcg_key;
  cudaGraphExec_t pcg_exec = nullptr;

  int nv() const { return (int)(n_dof / 3); }
  void sync() { GMCP_CUDA(cudaStreamSynchronize(stream)); }
  RedSlot slot(int off) {
    return RedSlot{parts.p, counter.p + off};
  }
};

namespace {

// elasticity.hpp:20-31
void make_material(double E, double nu, double& lambda, double& mu) {
  if (!(E > 0)) throw StatusError(GMCP_ERR_CONFIG, "material: Young's modulus must be positive");
  if (!(nu > -1.0) || nu >= 0.5 - 1e-6)
    throw StatusError(GMCP_ERR_CONFIG, "material: Poisson ratio must lie in (-1, 0.5 - 1e-6)");
  lambda = E * nu / ((1 + nu) * (1 - 2 * nu));
  mu = E / (2 * (1 + nu));
}

// elasticity.hpp:39-61 (rest shape-function gradients)
void build_operators(Body& b) {
  const int64_t nt = (int64_t)b.tets.size() / 4;
  b.vol.resize(nt);
  b.grads.resize(12 * nt);
  for (int64_t t = 0; t < nt; ++t) {
    const int32_t* tt = &b.tets[4 * t];
    double D[3][3];
    for (int i = 0; i < 3; ++i)
      for (int r = 0; r < 3; ++r) D[r][i] = b.verts[3 * tt[i + 1] + r] - b.verts[3 * tt[0] + r];
    const double det = D[0][0] * (D[1][1] * D[2][2] - D[2][1] * D[1][2]) -
                       D[1][0] * (D[0][1] * D[2][2] - D[2][1] * D[0][2]) +
                       D[2][0] * (D[0][1] * D[1][2] - D[1][1] * D[0][2]);
    b.vol[t] = det / 6.0;
    if (!(b.vol[t] > 0))
      throw StatusError(GMCP_ERR_DEGENERATE, "build_element_operators: non-positive tet volume at tet " +
                                                 std::to_string(t));
    double G[3][3];  // inverse of D
    G[0][0] = (D[1][1] * D[2][2] - D[1][2] * D[2][1]) / det;
    G[0][1] = (D[0][2] * D[2][1] - D[0][1] * D[2][2]) / det;
    G[0][2] = (D[0][1] * D[1][2] - D[0][2] * D[1][1]) / det;
    G[1][0] = (D[1][2] * D[2][0] - D[1][0] * D[2][2]) / det;
    G[1][1] = (D[0][0] * D[2][2] - D[0][2] * D[2][0]) / det;
    G[1][2] = (D[0][2] * D[1][0] - D[0][0] * D[1][2]) / det;
    G[2][0] = (D[1][0] * D[2][1] - D[1][1] * D[2][0]) / det;
    G[2][1] = (D[0][1] * D[2][0] - D[0][0] * D[2][1]) / det;
    G[2][2] = (D[0][0] * D[1][1] - D[0][1] * D[1][0]) / det;
    double* g = &b.grads[12 * t];
    for (int k = 0; k < 3; ++k) g[k] = 0;
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) {
        g[3 * (i + 1) + k] = G[i][k];
        g[k] -= G[i][k];
      }
  }
}

// Constant elastic BCSR (elasticity.hpp:124-141), blocks summed in tet order.
// Host-side set-up work over independent items (bodies) on up to 32 threads;
// every item is computed by exactly one thread, so results do not depend on
// the thread count.
template <class F>
void parallel_for(int64_t n, F&& f) {
  const int nt = (int)std::min<int64_t>(n, std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
  if (nt <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex m;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&]() {
      try {
        for (int64_t i; (i = next.fetch_add(1)) < n;) f(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(m);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// Vertex pairs of the 6x6 block-Jacobi (single systems and the per-scene CTA
// PCG) from an AoS BCSR of the operand's constant part: greedy matching of the
// strongest normalized couplings |K_vw|_F^2 / (|K_vv|_F |K_ww|_F) (ties by index).
void build_pairing(SystemImpl& S, int nv, const int32_t* rowptr, const int32_t* cols, const double* vals) {
#if GMCP_PAIR_JACOBI
  S.has_pairs = false;
  if (S.use_pair) {
    // vertex ranges matched independently: the bodies when no block couples two
    // of them (the elastic operator), else the whole system. Greedy matching
    // in descending score (ties in (row, block) order) on disjoint components
    // equals the global greedy matching, so each range sorts its own edges.
    std::vector<std::pair<int32_t, int32_t>> ranges;
    for (const Body& b : S.bodies) ranges.push_back({b.offset, b.offset + b.nv});
    std::atomic<bool> split{!ranges.empty()};
    parallel_for((int64_t)ranges.size(), [&](int64_t r) {
      for (int v = ranges[r].first; v < ranges[r].second; ++v)
        for (int k = rowptr[v]; k < rowptr[v + 1]; ++k)
          if (cols[k] < ranges[r].first || cols[k] >= ranges[r].second) {
            split = false;
            return;
          }
    });
    if (!split) ranges.assign(1, {0, nv});
    std::vector<double> dn(nv, 0.0);
    parallel_for((int64_t)ranges.size(), [&](int64_t r) {
      for (int v = ranges[r].first; v < ranges[r].second; ++v)
        for (int k = rowptr[v]; k < rowptr[v + 1]; ++k)
          if (cols[k] == v)
            for (int q = 0; q < 9; ++q) dn[v] += vals[9 * (size_t)k + q] * vals[9 * (size_t)k + q];
    });
    std::vector<int32_t> mate(nv, -1);
    parallel_for((int64_t)ranges.size(), [&](int64_t r) {
      struct Edge { double s; int32_t a, b; };
      std::vector<Edge> edges;
      for (int v = ranges[r].first; v < ranges[r].second; ++v)
        for (int k = rowptr[v]; k < rowptr[v + 1]; ++k) {
          const int w = cols[k];
          if (w <= v || !(dn[v] > 0) || !(dn[w] > 0)) continue;
          double f = 0;
          for (int q = 0; q < 9; ++q) f += vals[9 * (size_t)k + q] * vals[9 * (size_t)k + q];
          edges.push_back({f / std::sqrt(dn[v] * dn[w]), v, w});
        }
      std::stable_sort(edges.begin(), edges.end(), [](const Edge& x, const Edge& y) { return x.s > y.s; });
      for (const Edge& e : edges)
        if (mate[e.a] < 0 && mate[e.b] < 0) {
          mate[e.a] = e.b;
          mate[e.b] = e.a;
        }
    });
    S.pair_d.upload(mate, S.stream);
    S.has_pairs = true;
  }
#else
  S.has_pairs = false;
#endif
}

void build_elastic(SystemImpl& S) {
  const int nv = S.nv();
  // per body (bodies are independent; one thread each): its rows, columns
  // ascending, blocks summed over its tets in tet order
  struct BodyCsr {
    std::vector<int32_t> len, cols;
    std::vector<double> vals;
  };
  std::vector<BodyCsr> part(S.bodies.size());
  parallel_for((int64_t)S.bodies.size(), [&](int64_t bi_) {
    const Body& b = S.bodies[bi_];
    std::vector<std::vector<std::pair<int32_t, std::array<double, 9>>>> rows(b.nv);
    const int64_t nt = (int64_t)b.tets.size() / 4;
    for (int64_t t = 0; t < nt; ++t) {
      const double* g = &b.grads[12 * t];
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
          const double* gi = g + 3 * i;
          const double* gj = g + 3 * j;
          const double gg = gi[0] * gj[0] + gi[1] * gj[1] + gi[2] * gj[2];
          std::array<double, 9> blk;
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
              blk[3 * r + c] = b.vol[t] * (b.lambda * gi[r] * gj[c] + b.mu * gj[r] * gi[c] + (r == c ? b.mu * gg : 0.0));
          const int32_t li = b.tets[4 * t + i], bj = b.offset + b.tets[4 * t + j];
          auto& row = rows[li];
          auto it = std::find_if(row.begin(), row.end(), [&](const auto& e) { return e.first == bj; });
          if (it == row.end()) {
            row.push_back({bj, blk});
          } else {
            for (int q = 0; q < 9; ++q) it->second[q] += blk[q];
          }
        }
    }
    BodyCsr& P = part[bi_];
    P.len.resize(b.nv);
    size_t tot = 0;
    for (const auto& row : rows) tot += row.size();
    P.cols.reserve(tot);
    P.vals.reserve(9 * tot);
    for (int v = 0; v < b.nv; ++v) {
      auto& row = rows[v];
      std::sort(row.begin(), row.end(), [](const auto& a, const auto& c) { return a.first < c.first; });
      P.len[v] = (int32_t)row.size();
      for (const auto& e : row) {
        P.cols.push_back(e.first);
        P.vals.insert(P.vals.end(), e.second.begin(), e.second.end());
      }
    }
  });
  std::vector<int32_t> rowptr(nv + 1, 0);
  std::vector<int64_t> boff(S.bodies.size() + 1, 0);
  for (size_t bi_ = 0; bi_ < S.bodies.size(); ++bi_) {
    const Body& b = S.bodies[bi_];
    for (int v = 0; v < b.nv; ++v) rowptr[b.offset + v + 1] = part[bi_].len[v];
  }
  for (int v = 0; v < nv; ++v) rowptr[v + 1] += rowptr[v];
  const int64_t nnzb = rowptr[nv];
  // uninitialized host arrays (every entry is copied below): no 1.4 GB memset at C5
  std::unique_ptr<int32_t[]> cols(new int32_t[std::max<int64_t>(nnzb, 1)]);
  std::unique_ptr<double[]> vals(new double[std::max<int64_t>(9 * nnzb, 1)]);
  parallel_for((int64_t)S.bodies.size(), [&](int64_t bi_) {
    const Body& b = S.bodies[bi_];
    const int64_t o = rowptr[b.offset];
    std::copy(part[bi_].cols.begin(), part[bi_].cols.end(), cols.get() + o);
    std::copy(part[bi_].vals.begin(), part[bi_].vals.end(), vals.get() + 9 * o);
  });
  S.k_rowptr.upload(rowptr, S.stream);
  S.k_cols.upload(cols.get(), nnzb, S.stream);
  S.k_vals.upload(vals.get(), 9 * nnzb, S.stream);
  S.el_nnzb = nnzb;
  build_pairing(S, nv, rowptr.data(), cols.get(), vals.get());
  S.sync();  // the uploads read the host arrays
  S.el_built = true;
}

// The PCG operand: the merged matrix (one BCSR) when pairs exist.
MatSet mats(SystemImpl& S) {
  MatSet M;
  if (S.pairs.empty() || !S.u_valid) {
    M.el = Bcsr{S.k_rowptr.p, S.k_cols.p, S.k_vals.p};
    M.np = (int)S.pairs.size();
    for (int k = 0; k < M.np; ++k) {
      const AssemblyPlan& P = S.pairs[k]->c->plan;
      M.c[k] = Bcsr{P.rowptr.p, P.cols.p, P.vals.p};
    }
    return M;
  }
  M.el = Bcsr{S.u_rowptr.p, S.u_cols.p, S.u_vals.p, 1, S.u_nnzb};
  M.np = 0;
  if (S.u_half_ok) {
    M.hix = S.u_hix.p;
    M.hv = S.u_half.p;
    M.hn = S.u_hn;
  }
  return M;
}

// Union pattern of the elastic and every pair's contact BCSR, on the device
// (per rebuild): every block of every source is emitted as ((row, col) key,
// source << 32 | block) in source order, stably radix-sorted by key and
// run-length encoded; u_src then lists each union block's source blocks.
__global__ void k_union_emit(int nv, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                             int64_t source, int64_t base, unsigned long long* __restrict__ keys,
                             int64_t* __restrict__ vals) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x)
    for (int k = rowptr[v]; k < rowptr[v + 1]; ++k) {
      keys[base + k] = ((unsigned long long)(uint32_t)v << 32) | (unsigned long long)(uint32_t)cols[k];
      vals[base + k] = (source << 32) | k;
    }
}
__global__ void k_union_fill(int64_t nu, int ns, const unsigned long long* __restrict__ ukeys,
                             const int32_t* __restrict__ uoff, const int32_t* __restrict__ ucnt,
                             const int64_t* __restrict__ vals, int32_t* __restrict__ ucols, int32_t* __restrict__ src,
                             int32_t* __restrict__ rowcnt) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nu; k += (int64_t)gridDim.x * blockDim.x) {
    ucols[k] = (int32_t)(ukeys[k] & 0xffffffffull);
    atomicAdd(&rowcnt[(int64_t)(ukeys[k] >> 32)], 1);  // integer counts: order-free
    for (int e = uoff[k]; e < uoff[k] + ucnt[k]; ++e)
      src[(int64_t)ns * k + (vals[e] >> 32)] = (int32_t)(vals[e] & 0xffffffffll);
  }
}

void build_union(SystemImpl& S) {
  const int nv = S.nv(), np = (int)S.pairs.size(), ns = 1 + np;
  std::vector<const int32_t*> rp{S.k_rowptr.p}, cl{S.k_cols.p};
  std::vector<int64_t> nb{S.el_nnzb};
  for (auto& pr : S.pairs) {
    rp.push_back(pr->c->plan.rowptr.p);
    cl.push_back(pr->c->plan.cols.p);
    nb.push_back(pr->c->plan.nnzb);
  }
  int64_t total = 0;
  for (int64_t v : nb) total += v;
  auto& T = S.utmp;
  auto& keys = T.keys;
  auto& keys2 = T.keys2;
  auto& ukeys = T.ukeys;
  auto& vals = T.vals;
  auto& vals2 = T.vals2;
  auto& ucnt = T.ucnt;
  auto& uoff = T.uoff;
  auto& nuniq = T.nuniq;
  auto& rowcnt = T.rowcnt;
  keys.resize(std::max<int64_t>(total, 1));
  keys2.resize(std::max<int64_t>(total, 1));
  ukeys.resize(std::max<int64_t>(total, 1));
  vals.resize(std::max<int64_t>(total, 1));
  vals2.resize(std::max<int64_t>(total, 1));
  ucnt.resize(total + 1);
  uoff.resize(total + 1);
  nuniq.resize(1);
  int64_t base = 0;
  for (int q = 0; q < ns; ++q) {
    if (nb[q]) {
      k_union_emit<<<grid_for(nv, 256), 256, 0, S.stream>>>(nv, rp[q], cl[q], q, base, keys.p, vals.p);
      ++S.launches;
    }
    base += nb[q];
  }
  int rb = 1;
  while ((1ll << rb) < nv) ++rb;
  sort_pairs(keys.p, keys2.p, vals.p, vals2.p, total, S.stream, 32 + rb);
  run_length_encode(keys2.p, ukeys.p, ucnt.p, nuniq.p, total, S.stream);
  int32_t nu = 0;
  GMCP_CUDA(cudaMemcpyAsync(&nu, nuniq.p, sizeof nu, cudaMemcpyDeviceToHost, S.stream));
  S.sync();
  GMCP_CUDA(cudaMemsetAsync(ucnt.p + nu, 0, sizeof(int32_t), S.stream));
  exclusive_scan(ucnt.p, uoff.p, (int64_t)nu + 1, S.stream);
  S.u_nnzb = nu;
  S.u_cols.resize(std::max<int64_t>(nu, 1));
  S.u_src.resize(std::max<int64_t>((int64_t)ns * nu, 1));
  GMCP_CUDA(cudaMemsetAsync(S.u_src.p, 0xff, std::max<int64_t>((int64_t)ns * nu, 1) * sizeof(int32_t), S.stream));
  rowcnt.resize(nv + 1);
  rowcnt.zero(S.stream);
  k_union_fill<<<grid_for(nu, 256), 256, 0, S.stream>>>(nu, ns, ukeys.p, uoff.p, ucnt.p, vals2.p, S.u_cols.p, S.u_src.p,
                                                        rowcnt.p);
  ++S.launches;
  S.u_rowptr.resize(nv + 1);
  exclusive_scan(rowcnt.p, S.u_rowptr.p, (int64_t)nv + 1, S.stream);
  S.u_vals.resize(std::max<int64_t>(9 * S.u_nnzb, 1));
  S.u_half_ok = false;
  if (S.use_half && S.n_scenes == 1 && nu > 0) {
    S.u_hix.resize(2 * (int64_t)nu);
    S.u_hoff.resize(nv + 1);
    DBuf<int>& bad = T.bad;
    bad.resize(1);
    bad.zero(S.stream);
    rowcnt.zero(S.stream);
    k_half_count<<<grid_for(nv, 128), 128, 0, S.stream>>>(nv, S.u_rowptr.p, S.u_cols.p, rowcnt.p);
    exclusive_scan(rowcnt.p, S.u_hoff.p, (int64_t)nv + 1, S.stream);
    k_half_index<<<grid_for(nv, 128), 128, 0, S.stream>>>(nv, S.u_rowptr.p, S.u_cols.p, S.u_hoff.p, S.u_hix.p,
                                                         bad.p);
    S.launches += 2;
    int hb = 0, hn = 0;
    GMCP_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof hb, cudaMemcpyDeviceToHost, S.stream));
    GMCP_CUDA(cudaMemcpyAsync(&hn, S.u_hoff.p + nv, sizeof hn, cudaMemcpyDeviceToHost, S.stream));
    S.sync();
    S.u_hn = hn;
    S.u_half.resize(9 * (int64_t)hn);
    S.u_half_ok = hb == 0;
  }
  S.sync();
  S.u_valid = true;
  ++S.u_gen;
}

// solver.hpp:256-269
double derived_newton_tol(const SystemImpl& S) {
  double scale = 0;
  for (double f : S.f_ext) scale = std::max(scale, std::abs(f));
  double vol_sum = 0, e_max = 0;
  long n_elem = 0;
  for (const Body& b : S.bodies) {
    for (double v : b.vol) vol_sum += v;
    n_elem += (long)b.vol.size();
    e_max = std::max(e_max, b.E);
  }
  const double h = std::cbrt(6.0 * vol_sum / std::max<long>(n_elem, 1));
  scale = std::max(scale, 1e-6 * e_max * h * h);
  return 1e-6 * std::max(scale, 1e-6);
}

void rebuild_pair(SystemImpl& S, PairRt& pr, const double* eps_ref_dev) {
  const NvtxRange nvtx_("gmcp:rebuild pair");
  Ctx& c = *pr.c;
  S.u_valid = false;
  int64_t counts[3];
  static const bool trace = std::getenv("GMCP_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  double tms[3];
  auto lap = [&](int k) {
    if (!trace) return;
    S.sync();
    const auto t1 = std::chrono::steady_clock::now();
    tms[k] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    t0 = t1;
  };
  const int64_t l0 = c.launches;
  run_broadphase(c, pr.params.detection_radius, counts);
  lap(0);
  run_sampler(c, eps_ref_dev);
  lap(1);
  c.plan.valid = false;
  build_assembly_plan(c);
  lap(2);
  if (trace)
    std::fprintf(stderr, "[gmcp rebuild pair] broadphase %.2f sampler %.2f plan %.2f ms, %lld launches\n", tms[0],
                 tms[1], tms[2], (long long)(c.launches - l0));
  pr.ref_pos.resize(S.n_dof);
  GMCP_CUDA(cudaMemcpyAsync(pr.ref_pos.p, S.x.p, S.n_dof * sizeof(double), cudaMemcpyDeviceToDevice, S.stream));
}

// Returns {feasible, contact energy sum, min gap} at positions xp.
struct CE {
  bool feasible;
  double energy, min_gap;
};
CE contact_energy_at(SystemImpl& S, double* xp) {
  CE o{true, 0.0, 1.7976931348623157e308};
  for (auto& pr : S.pairs) {
    Ctx& c = *pr->c;
    double* saved = c.x_ext;
    c.x_ext = xp;
    const EnergyOut e = run_energy(c, false);
    c.x_ext = saved;
    if (e.first_degenerate >= 0 && (e.first_bad < 0 || e.first_degenerate < e.first_bad))
      throw StatusError(GMCP_ERR_DEGENERATE, "contact sample on a degenerate slave triangle");
    o.min_gap = std::min(o.min_gap, e.min_gap);
    if (e.first_bad >= 0) {
      o.feasible = false;
      return o;
    }
    o.energy += e.energy;
  }
  return o;
}

// Elastic + external energy at S.x (gel must hold K (x - rest)).
void elastic_terms(SystemImpl& S, double& e_el, double& work) {
  k_energy_el<<<kBlocks, kThreads, 0, S.stream>>>(S.nv(), S.gel.p, S.x.p, S.rest_d.p, S.fext_d.p, S.eel.p, S.slot(0));
  ++S.launches;
  double h[2];
  GMCP_CUDA(cudaMemcpyAsync(h, S.eel.p, sizeof h, cudaMemcpyDeviceToHost, S.stream));
  S.sync();
  e_el = h[0];
  work = h[1];
}

// grad = K u + sum contact grads - lambda f ; returns residual (max |grad| free)
double assemble(SystemImpl& S, double lambda) {
  const NvtxRange nvtx_("gmcp:assemble");
  std::vector<const double*> gp;
  for (auto& pr : S.pairs) {
    int64_t bad = -1;
    run_assembly(*pr->c, 1, &bad);
    gp.push_back(pr->c->grad.p);
  }
  if (!S.pairs.empty()) {  // merged PCG operand
    if (!S.u_valid) build_union(S);
    ValPtrs V{};
    V.v[0] = S.k_vals.p;
    for (size_t p = 0; p < S.pairs.size(); ++p) V.v[1 + p] = S.pairs[p]->c->plan.vals.p;
    k_merge<<<grid_for(S.u_nnzb, 256), 256, 0, S.stream>>>(S.u_nnzb, 1 + (int)S.pairs.size(), S.u_src.p, V,
                                                            S.u_vals.p, S.u_half_ok ? S.u_hix.p : nullptr,
                                                            S.u_half_ok ? S.u_half.p : nullptr, S.u_hn);
    ++S.launches;
  }
  S.gc_ptrs.resize(std::max<size_t>(gp.size(), 1));
  if (!gp.empty())
    GMCP_CUDA(cudaMemcpyAsync(S.gc_ptrs.p, gp.data(), gp.size() * sizeof(double*), cudaMemcpyHostToDevice, S.stream));
  GMCP_CUDA(cudaMemsetAsync(S.redu.p, 0, sizeof(unsigned long long), S.stream));
  k_grad_total<<<grid_for((int64_t)S.nv() * 32, 256), 256, 0, S.stream>>>(
      S.nv(), Bcsr{S.k_rowptr.p, S.k_cols.p, S.k_vals.p}, S.x.p, S.rest_d.p, S.fext_d.p, lambda, S.gc_ptrs.p,
      (int)gp.size(), S.mask_d.p, S.gel.p, S.grad.p, S.redu.p);
  ++S.launches;
  unsigned long long u;
  GMCP_CUDA(cudaMemcpyAsync(&u, S.redu.p, sizeof u, cudaMemcpyDeviceToHost, S.stream));
  S.sync();
  return from_ord_bits(u);
}

// Coarse space of the two-level preconditioner (coarse.cuh), host side, per
// solve set-up: each body's rest bounding box is cut into a grid of roughly
// cubic cells, ~coarse_aggs cells over the system in proportion to the bodies'
// vertex counts (a thin body gets one cell through its thickness); the
// vertices of one cell form an aggregate (empty cells form none).
void build_coarse(SystemImpl& S, const std::vector<double>& mask) {
  CoarseSpace& C = S.cs;
  C.enabled = false;
  const bool scenes = S.n_scenes > 1;
  if (!S.use_coarse) return;
  const int nv = S.nv();
  std::vector<int32_t> agg(nv, -1);
  int n_agg = 0;
  // batched scenes: a per-scene coarse space of ~coarse_scene_aggs aggregates
  // (each body lies in one scene; bodies come in scene order)
  std::vector<int64_t> scene_nv(std::max(S.n_scenes, 1), 0);
  if (scenes)
    for (const Body& b : S.bodies) scene_nv[S.vscene[b.offset]] += b.nv;
  std::vector<int32_t> body_first_agg;
  for (const Body& b : S.bodies) {
    body_first_agg.push_back(n_agg);
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int v = 0; v < b.nv; ++v)
      for (int k = 0; k < 3; ++k) {
        lo[k] = std::min(lo[k], b.verts[3 * v + k]);
        hi[k] = std::max(hi[k], b.verts[3 * v + k]);
      }
    const double kb = scenes ? std::max(1.0, (double)S.coarse_scene_aggs * b.nv / std::max<int64_t>(1, scene_nv[S.vscene[b.offset]]))
                             : std::max(1.0, (double)S.coarse_aggs * b.nv / std::max(1, nv));
    double L[3];
    for (int k = 0; k < 3; ++k) L[k] = std::max(hi[k] - lo[k], 1e-12 * std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], 1e-300}));
    // cell size h with prod max(1, round(L/h)) ~ kb (bisection on log h)
    auto cells = [&](double h, int* g) {
      double p = 1;
      for (int k = 0; k < 3; ++k) {
        const double c = std::min(std::max(1.0, std::floor(L[k] / h + 0.5)), 4095.0);
        g[k] = (int)c;
        p *= c;
      }
      return p;
    };
    const double lmax = std::max({L[0], L[1], L[2]});
    double hl = lmax * 1e-6, hh = lmax * 2;
    int g[3];
    for (int it = 0; it < 200; ++it) {
      const double hm = std::sqrt(hl * hh);
      if (cells(hm, g) > kb) hl = hm; else hh = hm;
    }
    cells(hh, g);
    std::map<int64_t, int32_t> id;
    for (int v = 0; v < b.nv; ++v) {
      int64_t key = 0;
      for (int k = 0; k < 3; ++k) {
        const int c = std::min(g[k] - 1, std::max(0, (int)((b.verts[3 * v + k] - lo[k]) / L[k] * g[k])));
        key = key * 4096 + c;
      }
      auto it = id.find(key);
      if (it == id.end()) it = id.emplace(key, 0).first;
      agg[b.offset + v] = (int32_t)key;  // replaced by a dense id below
    }
    int32_t next = n_agg;
    for (auto& kv : id) kv.second = next++;  // cells in (x, y, z) order
    for (int v = 0; v < b.nv; ++v) agg[b.offset + v] = id[agg[b.offset + v]];
    n_agg = next;
  }
  for (int v = 0; v < nv; ++v)
    if (agg[v] < 0) return;  // a vertex outside every body: no coarse space
  std::vector<double> cen(3 * (size_t)n_agg, 0.0), dvec(3 * (size_t)nv), gram(36 * (size_t)n_agg, 0.0);
  std::vector<int32_t> off(n_agg + 1, 0), verts(nv);
  for (int v = 0; v < nv; ++v) ++off[agg[v] + 1];
  for (int a = 0; a < n_agg; ++a) off[a + 1] += off[a];
  {
    std::vector<int32_t> fill(off.begin(), off.end() - 1);
    for (int v = 0; v < nv; ++v) verts[fill[agg[v]]++] = v;  // ascending within an aggregate
  }
  for (int a = 0; a < n_agg; ++a) {
    for (int e = off[a]; e < off[a + 1]; ++e)
      for (int k = 0; k < 3; ++k) cen[3 * a + k] += S.rest[3 * (size_t)verts[e] + k];
    for (int k = 0; k < 3; ++k) cen[3 * a + k] /= std::max(1, off[a + 1] - off[a]);
  }
  for (int v = 0; v < nv; ++v) {
    const int a = agg[v];
    const double d[3] = {S.rest[3 * (size_t)v] - cen[3 * a], S.rest[3 * (size_t)v + 1] - cen[3 * a + 1],
                         S.rest[3 * (size_t)v + 2] - cen[3 * a + 2]};
    for (int k = 0; k < 3; ++k) dvec[3 * (size_t)v + k] = d[k];
    // Phi_v = M [I | -[d]x] (3 x 6)
    const double cx[3][3] = {{0, -d[2], d[1]}, {d[2], 0, -d[0]}, {-d[1], d[0], 0}};
    double Phi[3][6];
    for (int i = 0; i < 3; ++i) {
      const double m = mask[3 * (size_t)v + i];
      for (int j = 0; j < 3; ++j) {
        Phi[i][j] = m * (i == j ? 1.0 : 0.0);
        Phi[i][3 + j] = -m * cx[i][j];
      }
    }
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j)
        for (int q = 0; q < 3; ++q) gram[36 * (size_t)a + 6 * i + j] += Phi[q][i] * Phi[q][j];
  }
  C.n_agg = n_agg;
  C.n_pad = ((6 * n_agg + kGJ - 1) / kGJ) * kGJ;
  C.agg.upload(agg, S.stream);
  C.dvec.upload(dvec, S.stream);
  C.agg_off.upload(off, S.stream);
  C.agg_verts.upload(verts, S.stream);
  C.gram.upload(gram, S.stream);
  static const bool trace = std::getenv("GMCP_TRACE") != nullptr;
  if (scenes) {  // per-scene dense blocks: scene s owns aggregates [sa[s], sa[s+1]), its
                 // (6 n_s)^2 coarse matrix at c_off[s]
    const int NS = S.n_scenes;
    std::vector<int32_t> sa(NS + 1, 0), agg_scene(n_agg);
    for (size_t bi = 0; bi < S.bodies.size(); ++bi) {
      const int sc = S.vscene[S.bodies[bi].offset];
      const int a1 = bi + 1 < S.bodies.size() ? body_first_agg[bi + 1] : n_agg;
      for (int a = body_first_agg[bi]; a < a1; ++a) agg_scene[a] = sc;
      sa[sc + 1] = a1;
    }
    for (int sc = 0; sc < NS; ++sc) sa[sc + 1] = std::max(sa[sc + 1], sa[sc]);
    std::vector<int64_t> coff(NS + 1, 0);
    int max_c = 0;
    for (int sc = 0; sc < NS; ++sc) {
      const int64_t d = 6 * (int64_t)(sa[sc + 1] - sa[sc]);
      coff[sc + 1] = coff[sc] + d * d;
      max_c = std::max(max_c, (int)d);
    }
    if (max_c > kSceneCoarseMax) return;  // too large for the per-scene CTA kernel: no coarse space
    C.scene_agg.upload(sa, S.stream);
    C.agg_scene.upload(agg_scene, S.stream);
    C.scene_coff.upload(coff, S.stream);
    C.A.resize(std::max<int64_t>(coff[NS], 1));
    C.scale.resize(6 * (size_t)n_agg);
    C.n_scene_c = max_c;
    C.pat_gen = -2;
    C.enabled = true;
    if (trace)
      std::fprintf(stderr, "[gmcp] per-scene coarse spaces: %d aggregates over %d scenes (max %d coarse dofs/scene)\n",
                   n_agg, NS, max_c);
    return;
  }
  if (trace) std::fprintf(stderr, "[gmcp] coarse space: %d aggregates, %d coarse dofs (padded)\n", n_agg, C.n_pad);
  const size_t n2 = (size_t)C.n_pad * C.n_pad;
  C.A.resize(n2);
  C.B.resize(n2);
  C.scale.resize(C.n_pad);
  C.s.resize(C.n_pad);
  C.y.resize(C.n_pad);
  C.s.zero(S.stream);
  C.y.zero(S.stream);
  C.pat_gen = -2;  // pair lists rebuilt at the first solve
  C.enabled = true;
}

// Coarse operator of this solve's operand (single merged BCSR M.el) and its
// scaled pseudo-inverse. Pair lists are rebuilt when the pattern changed.
void coarse_setup_impl(SystemImpl& S, const MatSet& M);
void coarse_setup(SystemImpl& S, const MatSet& M) {
  const NvtxRange nvtx_("gmcp:coarse setup");
  static const bool trace = std::getenv("GMCP_TRACE") != nullptr;
  if (!trace) return coarse_setup_impl(S, M);
  const auto t0 = std::chrono::steady_clock::now();
  coarse_setup_impl(S, M);
  S.sync();
  std::fprintf(stderr, "[gmcp] coarse setup %.3f ms (%d aggregate pairs, %d coarse dofs)\n",
               std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), S.cs.n_pairs,
               S.cs.n_pad);
}
// aggregate-pair block lists of the operand's pattern (rebuilt when it changed)
void coarse_pair_lists(SystemImpl& S, const MatSet& M) {
  CoarseSpace& C = S.cs;
  const int nv = S.nv();
  const Bcsr& A = M.el;
  int64_t nnzb = 0;
  GMCP_CUDA(cudaMemcpyAsync(&nnzb, &A.rowptr[nv], sizeof(int32_t), cudaMemcpyDeviceToHost, S.stream));
  S.sync();
  nnzb = (int64_t)(int32_t)nnzb;
  const int64_t gen = S.u_valid ? S.u_gen : -1;
  if (C.pat_rowptr != A.rowptr || C.pat_cols != A.cols || C.pat_nnzb != nnzb || C.pat_gen != gen) {
    const int64_t m = std::max<int64_t>(nnzb, 1);
    C.u_row.resize(m);
    C.blk.resize(m);
    C.blk2.resize(m);
    C.key.resize(m);
    C.key2.resize(m);
    C.ukey.resize(m);
    C.pcnt.resize(m + 1);
    C.poff.resize(m + 1);
    C.npair.resize(1);
    k_block_rows<<<grid_for(nv, 256), 256, 0, S.stream>>>(nv, A.rowptr, C.u_row.p);
    k_pair_keys<<<grid_for(nnzb, 256), 256, 0, S.stream>>>(nnzb, C.u_row.p, A.cols, C.agg.p, C.n_agg, C.key.p,
                                                           C.blk.p);
    S.launches += 2;
    int kb = 1;
    while ((1ull << kb) <= (unsigned long long)C.n_agg * C.n_agg) ++kb;
    sort_pairs(C.key.p, C.key2.p, C.blk.p, C.blk2.p, nnzb, S.stream, kb);
    run_length_encode(C.key2.p, C.ukey.p, C.pcnt.p, C.npair.p, nnzb, S.stream);
    int32_t np = 0;
    unsigned long long last = 0;
    GMCP_CUDA(cudaMemcpyAsync(&np, C.npair.p, sizeof np, cudaMemcpyDeviceToHost, S.stream));
    S.sync();
    if (np > 0) {
      GMCP_CUDA(cudaMemcpyAsync(&last, C.ukey.p + np - 1, sizeof last, cudaMemcpyDeviceToHost, S.stream));
      S.sync();
      if (last == (unsigned long long)C.n_agg * C.n_agg) --np;  // lower-tile blocks (sentinel key)
    }
    GMCP_CUDA(cudaMemsetAsync(C.pcnt.p + np, 0, sizeof(int32_t), S.stream));
    exclusive_scan(C.pcnt.p, C.poff.p, (int64_t)np + 1, S.stream);
    C.n_pairs = np;
    C.pat_rowptr = A.rowptr;
    C.pat_cols = A.cols;
    C.pat_nnzb = nnzb;
    C.pat_gen = gen;
  }
}

void coarse_setup_impl(SystemImpl& S, const MatSet& M) {
  CoarseSpace& C = S.cs;
  const Bcsr& A = M.el;
  coarse_pair_lists(S, M);
  const int n_pad = C.n_pad;
  GMCP_CUDA(cudaMemsetAsync(C.A.p, 0, (size_t)n_pad * n_pad * sizeof(double), S.stream));
  if (C.n_pairs > 0)
    k_coarse_assemble<<<C.n_pairs, 256, 0, S.stream>>>(
        C.n_pairs, C.n_agg, n_pad, C.ukey.p, C.poff.p, C.pcnt.p, C.blk2.p, C.u_row.p, A.cols, A.vals, A.bs, A.cs,
        S.mask_d.p, C.dvec.p, C.gram.p, M.shift, C.A.p);
  k_coarse_scale<<<grid_for(n_pad, 256), 256, 0, S.stream>>>(n_pad, C.A.p, C.scale.p);
  k_coarse_apply_scale<<<grid_for((int64_t)n_pad * n_pad, 256), 256, 0, S.stream>>>(n_pad, C.A.p, C.scale.p);
  S.launches += 3;
  const int nt = n_pad / kGJ;
  double* X = C.A.p;
  double* Y = C.B.p;
  static const bool trace = std::getenv("GMCP_TRACE") != nullptr;
  cudaEvent_t te[3];
  if (trace) {
    for (auto& e : te) GMCP_CUDA(cudaEventCreate(&e));
    GMCP_CUDA(cudaEventRecord(te[0], S.stream));
  }
  GMCP_CUDA(cudaMemsetAsync(S.redu.p + 4, 0, sizeof(unsigned long long), S.stream));
  C.piv.resize(2 * kGJ * kGJ);
  // one cooperative launch when every CTA's tiles fit in shared memory
  static const bool persistent = !std::getenv("GMCP_GJ_PERSISTENT") || std::atoi(std::getenv("GMCP_GJ_PERSISTENT")) != 0;
  int sms = 0;
  GMCP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, S.device));
  const int G = std::min(sms, nt * nt);
  const size_t gsmem = (size_t)((nt * nt + G - 1) / G + 1 + 3 * kGJGroups) * kGJ * (kGJ + 1) * sizeof(double);
  if (persistent && gsmem <= 200 * 1024) {
    GMCP_CUDA(cudaFuncSetAttribute(k_gj_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
    int occ = 0;
    GMCP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gj_persistent, kGJPThreads, gsmem));
    if (occ >= 1) {
      C.gj_rowp.resize(2 * (size_t)nt * kGJ * kGJ);
      C.gj_colp.resize(2 * (size_t)nt * kGJ * kGJ);
      int np_ = n_pad;
      double thr = S.coarse_drop;
      unsigned long long* dr = S.redu.p + 4;
      void* args[] = {&np_, &X, &C.gj_rowp.p, &C.gj_colp.p, &C.piv.p, &thr, &dr};
      if (trace) GMCP_CUDA(cudaEventRecord(te[1], S.stream));
      const cudaError_t le =
          cudaLaunchCooperativeKernel((const void*)k_gj_persistent, G, kGJPThreads, args, gsmem, S.stream);
      if (le != cudaSuccess) {  // e.g. the SMs are shared and the grid cannot be co-resident: per-step launches
        (void)cudaGetLastError();
        goto per_step;
      }
      ++S.launches;
      C.inv = X;
      if (trace) {
        GMCP_CUDA(cudaEventRecord(te[2], S.stream));
        GMCP_CUDA(cudaEventSynchronize(te[2]));
        float a = 0, b = 0;
        GMCP_CUDA(cudaEventElapsedTime(&a, te[0], te[1]));
        GMCP_CUDA(cudaEventElapsedTime(&b, te[1], te[2]));
        std::fprintf(stderr, "[gmcp] Gauss-Jordan (one cooperative launch, %d CTAs): %.3f ms\n", G, b);
        for (auto& e : te) cudaEventDestroy(e);
      }
      return;
    }
  }
per_step:
  k_gj_pivot0<<<1, kGJThreads, 0, S.stream>>>(n_pad, X, C.piv.p, S.coarse_drop, S.redu.p + 4);
  ++S.launches;
  for (int k = 0; k < nt; ++k) {
    k_gj_step<<<dim3(nt, nt), kGJThreads, 0, S.stream>>>(n_pad, k, X, Y, C.piv.p + (k & 1) * kGJ * kGJ,
                                                  C.piv.p + ((k + 1) & 1) * kGJ * kGJ, S.coarse_drop, S.redu.p + 4);
    ++S.launches;
    std::swap(X, Y);
    if (trace && k == 0) GMCP_CUDA(cudaEventRecord(te[1], S.stream));
  }
  C.inv = X;
  if (trace) {
    GMCP_CUDA(cudaEventRecord(te[2], S.stream));
    GMCP_CUDA(cudaEventSynchronize(te[2]));
    float a = 0, b = 0;
    GMCP_CUDA(cudaEventElapsedTime(&a, te[0], te[1]));
    GMCP_CUDA(cudaEventElapsedTime(&b, te[1], te[2]));
    std::fprintf(stderr, "[gmcp] Gauss-Jordan: pivot 0 + step 0 %.3f ms, steps 1..%d %.3f ms\n", a, nt - 1, b);
    for (auto& e : te) cudaEventDestroy(e);
  }
}

// Batched scenes: every scene's coarse operator (its own shift) and its
// scaled pseudo-inverse, per batched PCG call.
void coarse_setup_scenes(SystemImpl& S, const MatSet& M, const double* shift_dev) {
  const NvtxRange nvtx_("gmcp:coarse setup (scenes)");
  CoarseSpace& C = S.cs;
  const Bcsr& A = M.el;
  coarse_pair_lists(S, M);
  const int NS = S.n_scenes;
  GMCP_CUDA(cudaMemsetAsync(C.A.p, 0, C.A.n * sizeof(double), S.stream));
  if (C.n_pairs > 0)
    k_coarse_assemble<<<C.n_pairs, 256, 0, S.stream>>>(
        C.n_pairs, C.n_agg, 0, C.ukey.p, C.poff.p, C.pcnt.p, C.blk2.p, C.u_row.p, A.cols, A.vals, A.bs, A.cs,
        S.mask_d.p, C.dvec.p, C.gram.p, 0.0, C.A.p, C.agg_scene.p, C.scene_agg.p, C.scene_coff.p, shift_dev);
  k_scene_coarse_inv<<<NS, 256, 0, S.stream>>>(C.scene_agg.p, C.scene_coff.p, C.A.p, C.scale.p, kSceneCoarseDrop);
  S.launches += 2;
}

// ||H dx - rhs|| of the solve just finished (recomputed, not the recursive
// residual PCG stops on); optionally copies the linear system to the host.
void true_residual(SystemImpl& S, const MatSet& M) {
  const int nv = S.nv();
  GMCP_CUDA(cudaMemsetAsync(S.redu.p + 2, 0, 2 * sizeof(unsigned long long), S.stream));
  k_true_resid<<<kBlocks, kThreads, 0, S.stream>>>(nv, M, S.mask_d.p, S.dx.p, S.grad.p, S.rt.p, S.scal.p + 12,
                                                   S.redu.p + 2, S.slot(5));
  ++S.launches;
  double sums[2];
  unsigned long long mx[2];
  GMCP_CUDA(cudaMemcpyAsync(sums, S.scal.p + 12, sizeof sums, cudaMemcpyDeviceToHost, S.stream));
  GMCP_CUDA(cudaMemcpyAsync(mx, S.redu.p + 2, sizeof mx, cudaMemcpyDeviceToHost, S.stream));
  S.sync();
  S.last_true_rel2 = sums[1] > 0 ? std::sqrt(sums[0] / sums[1]) : 0.0;
  const double bi = from_ord_bits(mx[1]);
  S.last_true_relinf = bi > 0 ? from_ord_bits(mx[0]) / bi : 0.0;
  if (S.capture) {  // the operand as one AoS BCSR (all sources summed per block) + mask, grad, dx
    S.cap_shift = M.shift;
    const Bcsr* src[1 + kMaxPairs] = {&M.el, &M.c[0], &M.c[1], &M.c[2], &M.c[3]};
    std::vector<std::vector<int32_t>> rp(1 + M.np), cl(1 + M.np);
    std::vector<std::vector<double>> vv(1 + M.np);
    for (int m = 0; m <= M.np; ++m) {
      const Bcsr& A = *src[m];
      rp[m].resize(nv + 1);
      GMCP_CUDA(cudaMemcpyAsync(rp[m].data(), A.rowptr, (nv + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, S.stream));
      S.sync();
      const int64_t nb = rp[m][nv];
      cl[m].resize(nb);
      std::vector<double> raw(9 * (size_t)nb);
      if (nb) {
        GMCP_CUDA(cudaMemcpyAsync(cl[m].data(), A.cols, nb * sizeof(int32_t), cudaMemcpyDeviceToHost, S.stream));
        GMCP_CUDA(cudaMemcpyAsync(raw.data(), A.vals, 9 * nb * sizeof(double), cudaMemcpyDeviceToHost, S.stream));
      }
      S.sync();
      vv[m].resize(9 * (size_t)nb);
      for (int64_t k = 0; k < nb; ++k)
        for (int q = 0; q < 9; ++q) vv[m][9 * k + q] = raw[k * A.bs + q * A.cs];
    }
    S.cap_rowptr.assign(nv + 1, 0);
    S.cap_cols.clear();
    S.cap_vals.clear();
    for (int v = 0; v < nv; ++v) {
      std::map<int32_t, std::array<double, 9>> row;
      for (int m = 0; m <= M.np; ++m)
        for (int32_t k = rp[m][v]; k < rp[m][v + 1]; ++k) {
          auto& b = row[cl[m][k]];
          for (int q = 0; q < 9; ++q) b[q] += vv[m][9 * (size_t)k + q];
        }
      for (auto& [c, b] : row) {
        S.cap_cols.push_back(c);
        S.cap_vals.insert(S.cap_vals.end(), b.begin(), b.end());
      }
      S.cap_rowptr[v + 1] = (int32_t)S.cap_cols.size();
    }
    S.cap_mask = S.mask_d.to_host(S.stream);
    S.cap_grad = S.grad.to_host(S.stream);
    S.cap_dx = S.dx.to_host(S.stream);
  }
}

// Block-Jacobi PCG on the masked system (chunks of iterations replayed as one
// CUDA graph) for rhs = -mask .* gsrc. Returns iterations; solution in S.dx.


int pcg_core(SystemImpl& S, double tol, int maxit, double* rel_out, double shift, const double* gsrc) {
  const int nv = S.nv();
  MatSet M = mats(S);
  M.shift = shift;
  // a refinement pass (pcg(): rhs = the true residual) solves with the operator
  // and shift of the solve it refines, right after it
  const bool refine_pass = gsrc != S.grad.p && S.last_solve_shift == shift && S.last_solve_ops == S.u_gen;
  S.last_solve_shift = shift;
  S.last_solve_ops = S.u_gen;
  const bool pairs = S.has_pairs && S.pair_d.n == nv;
  const bool coarse = S.cs.enabled && M.np == 0;
  CoarseSpace& C = S.cs;
  if (coarse) {
    const int64_t gen = S.u_valid ? S.u_gen : -1;
    // reuse only once Newton is steady: the last two solves ran on fresh
    // inverses with iteration counts within 15% (the contact Hessian settled)
    const bool steady = C.prev_fresh_iters > 0 && C.ref_iters > 0 &&
                        std::abs(C.ref_iters - C.prev_fresh_iters) <= 0.15 * C.prev_fresh_iters;
    const bool same_context = C.have_inv && C.inv_step == S.load_step && C.inv_gen == gen && C.inv_shift == M.shift;
    // a refinement pass (rhs = the true residual) solves with the operator of
    // the solve it refines: that solve's coarse inverse is current
    const bool refining = gsrc != S.grad.p && same_context;
    const bool stale = !refining && (!same_context || S.coarse_refresh_always || !steady ||
                                     (C.ref_iters > 0 && C.last_iters > kCoarseStale * C.ref_iters));
    if (stale) C.prev_fresh_iters = same_context ? C.ref_iters : -1;
    if (stale) {
      coarse_setup(S, M);
      C.have_inv = true;
      C.inv_step = S.load_step;
      C.inv_gen = gen;
      C.inv_shift = M.shift;
      C.ref_iters = -1;  // set by this solve
    }
  }
  // two-level init: z += P Ac^+ P^T r, completing r.z (beta = 0)
  auto coarse_init = [&]() {
    k_restrict<<<C.n_agg, 256, 0, S.stream>>>(C.n_agg, C.agg_off.p, C.agg_verts.p, C.dvec.p, S.mask_d.p, S.r.p,
                                            C.scale.p, C.s.p);
    k_coarse_prolong<true><<<C.n_agg, kAggThreads, 0, S.stream>>>(C.n_pad, C.inv, C.scale.p, C.s.p, C.agg_off.p,
                                                               C.agg_verts.p, C.dvec.p, S.mask_d.p, S.z.p, S.scal.p,
                                                               S.slot(6));
    S.launches += 2;
  };
  if (pairs) {
    S.minv2.resize(18 * (int64_t)nv);
    S.r2.resize(3 * (int64_t)nv);
    if (!refine_pass)  // a refinement pass keeps the operator, so the smoother too
      k_pair_jacobi<<<grid_for(nv, 128), 128, 0, S.stream>>>(nv, M, S.mask_d.p, S.pair_d.p, S.minv2.p);
    if (coarse)
      k_pcg_init_pair<true><<<kBlocks, kThreads, 0, S.stream>>>(nv, gsrc, S.mask_d.p, S.minv2.p, S.pair_d.p, S.dx.p,
                                                                S.r.p, S.z.p, S.p.p, S.scal.p, S.slot(0));
    else
    k_pcg_init_pair<false><<<kBlocks, kThreads, 0, S.stream>>>(nv, gsrc, S.mask_d.p, S.minv2.p, S.pair_d.p, S.dx.p,
                                                        S.r.p, S.z.p, S.p.p, S.scal.p, S.slot(0));
  } else {
    if (!refine_pass)
      k_block_jacobi<<<grid_for(nv, 256), 256, 0, S.stream>>>(nv, M, S.mask_d.p, S.minv.p);
    if (coarse)
      k_pcg_init<true><<<kBlocks, kThreads, 0, S.stream>>>(nv, gsrc, S.mask_d.p, S.minv.p, S.dx.p, S.r.p, S.z.p,
                                                           S.p.p, S.scal.p, S.slot(0));
    else
    k_pcg_init<false><<<kBlocks, kThreads, 0, S.stream>>>(nv, gsrc, S.mask_d.p, S.minv.p, S.dx.p, S.r.p, S.z.p, S.p.p,
                                                   S.scal.p, S.slot(0));
  }
  S.launches += 2;
  if (coarse) coarse_init();
  double h[9];
  GMCP_CUDA(cudaMemcpyAsync(h, S.scal.p, sizeof h, cudaMemcpyDeviceToHost, S.stream));
  S.sync();
  const double bb = h[5];
  if (bb == 0) {
    *rel_out = 0;
    S.last_true_rel2 = S.last_true_relinf = 0;
    return 0;
  }
  const double target = tol * tol * bb;
  // small two-level systems: the whole iteration loop in one cooperative launch
  static const bool coop_on = !std::getenv("GMCP_PCG_COOP") || std::atoi(std::getenv("GMCP_PCG_COOP")) != 0;
  if (coop_on && coarse && pairs && nv <= kCoopMaxRows && C.n_agg > 0) {
    int sms = 0, occ = 0;
    GMCP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, S.device));
    GMCP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pcg_coop, kCoopThreads, 0));
    const int G = std::min({C.n_agg, kCoopMaxCtas, std::max(1, occ) * sms});
    S.coop_part.resize(4 * kCoopMaxCtas);
    S.r2.resize(3 * (int64_t)nv);
    CoopArgs ca{M, nv, S.mask_d.p, gsrc, S.minv2.p, S.pair_d.p, C.agg_off.p, C.agg_verts.p, C.dvec.p, C.scale.p,
                C.inv, C.n_agg, C.n_pad, S.dx.p, S.r.p, S.r2.p, S.z.p, S.p.p, S.w.p, S.q.p, C.s.p, S.coop_part.p,
                S.scal.p, tol * tol, maxit, gsrc == S.grad.p ? 1 : 0, kDriftFail * tol};
    void* args[] = {&ca};
    if (!S.ev0) {
      GMCP_CUDA(cudaEventCreate(&S.ev0));
      GMCP_CUDA(cudaEventCreate(&S.ev1));
    }
    GMCP_CUDA(cudaEventRecord(S.ev0, S.stream));
    const cudaError_t le = cudaLaunchCooperativeKernel((const void*)k_pcg_coop, G, kCoopThreads, args, 0, S.stream);
    if (le == cudaSuccess) {
      GMCP_CUDA(cudaEventRecord(S.ev1, S.stream));
      ++S.launches;
      double hc[11];
      GMCP_CUDA(cudaMemcpyAsync(hc, S.scal.p, sizeof hc, cudaMemcpyDeviceToHost, S.stream));
      S.sync();
      float ems = 0;
      GMCP_CUDA(cudaEventElapsedTime(&ems, S.ev0, S.ev1));
      const int it = (int)hc[10];
      S.pcg_ev_ms += ems;
      S.pcg_ev_iters += it;
      const int status = (int)hc[9];
      if (status == 2) ++S.drift_fails;
      *rel_out = status != 0 ? INFINITY : std::sqrt(hc[4] / bb);
      GMCP_CUDA(cudaGetLastError());
      return it;
    }
    (void)cudaGetLastError();  // not co-resident (shared SMs): the chunked path below
  }
  const int chunk = 16;
  const int lanes = nv < kSmallRows ? 8 : 4;
  const int gsp = std::min(grid_for((int64_t)nv * lanes, kThreads), kBlocks);
  const int gup = std::min(grid_for((int64_t)nv, kThreads), kBlocks);  // one vertex per thread
  // one chunk of iterations as a CUDA graph; the instantiated graph is kept
  // while its launch parameters (operand, vectors, shift, grids) are unchanged,
  // i.e. across the Newton iterations between rebuilds
  SystemImpl::PcgKey key;
  std::memset(&key, 0, sizeof key);
  key.M = M;
  key.nv = nv;
  key.lanes = lanes;
  key.gsp = gsp;
  key.gup = gup;
  const void* ptrs[14] = {S.mask_d.p, S.z.p, S.p.p, S.w.p, S.q.p, S.dx.p, S.r.p,
                          pairs ? (const void*)S.minv2.p : (const void*)S.minv.p, S.scal.p,
                          pairs ? (const void*)S.r2.p : (const void*)S.parts.p, S.counter.p,
                          coarse ? (const void*)C.inv : nullptr, coarse ? (const void*)C.s.p : nullptr,
                          coarse ? (const void*)C.agg.p : nullptr};
  static_assert(sizeof ptrs == sizeof key.ptrs, "PcgKey pointer list");
  std::memcpy(key.ptrs, ptrs, sizeof ptrs);
  auto same_bcsr = [](const Bcsr& a, const Bcsr& b) {
    return a.rowptr == b.rowptr && a.cols == b.cols && a.vals == b.vals && a.bs == b.bs && a.cs == b.cs;
  };
  auto same_key = [&](const SystemImpl::PcgKey& a, const SystemImpl::PcgKey& b) {
    if (!same_bcsr(a.M.el, b.M.el) || a.M.np != b.M.np || a.M.shift != b.M.shift || a.M.hix != b.M.hix ||
        a.M.hv != b.M.hv || a.M.hn != b.M.hn)
      return false;
    for (int k = 0; k < a.M.np; ++k)
      if (!same_bcsr(a.M.c[k], b.M.c[k])) return false;
    return a.nv == b.nv && a.lanes == b.lanes && a.gsp == b.gsp && a.gup == b.gup &&
           std::memcmp(a.ptrs, b.ptrs, sizeof a.ptrs) == 0;
  };
  if (!S.pcg_exec || !same_key(key, S.pcg_key)) {
    if (S.pcg_exec) cudaGraphExecDestroy(S.pcg_exec);
    S.pcg_exec = nullptr;
    cudaGraph_t graph;
    GMCP_CUDA(cudaStreamBeginCapture(S.stream, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < chunk; ++k) {  // p ping-pongs between S.p and S.w (chunk is even)
      double* p_old = (k & 1) ? S.w.p : S.p.p;
      double* p_new = (k & 1) ? S.p.p : S.w.p;
      const bool half = M.hv != nullptr && M.np == 0;
      const bool pre = pupdate_on();
      // large systems: p_new streamed by its own kernel, the SpMV gathers one vector
      // (C3 PCG iteration 47.1 -> 45.3 us); small ones keep the fused form (the
      // extra launch costs more than it saves: Hertz 5.4 -> 5.9 ms per Newton step)
      if (half && pre && lanes == 4) {
        k_pupdate<<<std::min(grid_for(3 * (int64_t)nv, kThreads), kBlocks), kThreads, 0, S.stream>>>(
            3 * (int64_t)nv, S.z.p, p_old, p_new, S.scal.p);
        k_spmv_cg<4, true, true><<<gsp, kThreads, 0, S.stream>>>(nv, M, S.mask_d.p, S.z.p, p_old, p_new, S.q.p,
                                                                  S.scal.p, S.slot(1));
      } else if (lanes == 8 && half)
        k_spmv_cg<8, true><<<gsp, kThreads, 0, S.stream>>>(nv, M, S.mask_d.p, S.z.p, p_old, p_new, S.q.p, S.scal.p,
                                                            S.slot(1));
      else if (lanes == 8)
        k_spmv_cg<8><<<gsp, kThreads, 0, S.stream>>>(nv, M, S.mask_d.p, S.z.p, p_old, p_new, S.q.p, S.scal.p,
                                                      S.slot(1));
      else if (half)
        k_spmv_cg<4, true><<<gsp, kThreads, 0, S.stream>>>(nv, M, S.mask_d.p, S.z.p, p_old, p_new, S.q.p, S.scal.p,
                                                            S.slot(1));
      else
        k_spmv_cg<4><<<gsp, kThreads, 0, S.stream>>>(nv, M, S.mask_d.p, S.z.p, p_old, p_new, S.q.p, S.scal.p,
                                                      S.slot(1));
      if (coarse) {  // update + restriction, then coarse solve + prolongation (per aggregate)
        const double* rin = pairs ? ((k & 1) ? S.r2.p : S.r.p) : S.r.p;
        double* rout = pairs ? ((k & 1) ? S.r.p : S.r2.p) : S.r.p;
        if (pairs)
          k_update_agg<true><<<C.n_agg, kAggThreads, 0, S.stream>>>(
              C.agg_off.p, C.agg_verts.p, C.dvec.p, S.mask_d.p, C.scale.p, p_new, S.q.p, S.dx.p, rin, rout, S.z.p,
              S.minv2.p, S.pair_d.p, C.s.p, S.scal.p, S.slot(2));
        else
          k_update_agg<false><<<C.n_agg, kAggThreads, 0, S.stream>>>(
              C.agg_off.p, C.agg_verts.p, C.dvec.p, S.mask_d.p, C.scale.p, p_new, S.q.p, S.dx.p, rin, rout, S.z.p,
              S.minv.p, nullptr, C.s.p, S.scal.p, S.slot(2));
        k_coarse_prolong<false><<<C.n_agg, kAggThreads, 0, S.stream>>>(C.n_pad, C.inv, C.scale.p, C.s.p,
                                                                    C.agg_off.p, C.agg_verts.p, C.dvec.p,
                                                                    S.mask_d.p, S.z.p, S.scal.p, S.slot(6));
      } else if (pairs) {  // r ping-pongs with p (chunk is even: r ends in S.r)
        k_update_cg_pair<false><<<gup, kThreads, 0, S.stream>>>(nv, p_new, S.q.p, S.dx.p, (k & 1) ? S.r2.p : S.r.p,
                                                                (k & 1) ? S.r.p : S.r2.p, S.z.p, S.minv2.p,
                                                                S.pair_d.p, S.scal.p, S.slot(2));
      } else {
        k_update_cg<false><<<gup, kThreads, 0, S.stream>>>(nv, p_new, S.q.p, S.dx.p, S.r.p, S.z.p, S.minv.p,
                                                           S.scal.p, S.slot(2));
      }
    }
    GMCP_CUDA(cudaStreamEndCapture(S.stream, &graph));
    GMCP_CUDA(cudaGraphInstantiate(&S.pcg_exec, graph, 0));
    cudaGraphDestroy(graph);
    S.pcg_key = key;
  }
  cudaGraphExec_t exec = S.pcg_exec;
  int it = 0;
  // with the coarse space a converging solve gains orders of magnitude per
  // 256 iterations, so a singular one is recognised four times sooner
  const int stag = coarse ? kStagWindowCoarse : kStagWindow;
  bool failed = false;
  double win_min = INFINITY, prev_min = INFINITY;  // stagnation windows
  if (!S.ev0) {
    GMCP_CUDA(cudaEventCreate(&S.ev0));
    GMCP_CUDA(cudaEventCreate(&S.ev1));
  }
  while (it < maxit) {
    GMCP_CUDA(cudaEventRecord(S.ev0, S.stream));
    GMCP_CUDA(cudaGraphLaunch(exec, S.stream));
    GMCP_CUDA(cudaEventRecord(S.ev1, S.stream));
    S.launches += ((coarse ? 3 : 2) + (M.hv && M.np == 0 && lanes == 4 && pupdate_on() ? 1 : 0)) * chunk;
    it += chunk;
    GMCP_CUDA(cudaMemcpyAsync(h, S.scal.p, sizeof h, cudaMemcpyDeviceToHost, S.stream));
    S.sync();
    float ems = 0;
    GMCP_CUDA(cudaEventElapsedTime(&ems, S.ev0, S.ev1));
    S.pcg_ev_ms += ems;
    S.pcg_ev_iters += chunk;
    if (!(h[4] > target)) break;  // rr <= tol^2 bb
    // a non-finite residual or r.z <= 0 (the preconditioner lost positivity):
    // the solve failed -> the caller retries regularized, as after a failed LDL^T
    if (!std::isfinite(h[4]) || !(h[0] > 0)) {
      failed = true;
      break;
    }
    // a singular system with an inconsistent rhs (a rigid mode before contact
    // engages) keeps shrinking its recursive residual while the true one
    // stalls: every kDriftWindow iterations the true residual is recomputed, and a
    // gap between the two that no refinement can close fails the solve now
    // (the regularized retry follows) instead of after thousands of iterations
    if (gsrc == S.grad.p && it % kDriftWindow == 0) {
      const bool cap = S.capture;
      S.capture = false;
      true_residual(S, M);
      S.capture = cap;
      if (S.last_true_rel2 - std::sqrt(h[4] / bb) > kDriftFail * tol ||
          (coarse && shift == 0 && S.last_true_rel2 > kDivergeRel)) {
        failed = true;
        ++S.drift_fails;
        break;
      }
    }
    win_min = std::min(win_min, h[4]);
    if (it % stag == 0) {
      if (it >= 2 * stag && !(win_min < 0.5 * prev_min) && h[4] > 1e-8 * bb) break;  // stagnated
      prev_min = std::min(prev_min, win_min);
      win_min = INFINITY;
    }
  }
  *rel_out = failed ? INFINITY : std::sqrt(h[4] / bb);
  GMCP_CUDA(cudaGetLastError());
  return it;
}

// PCG + residual replacement. CG stops on its recursive residual, which on
// stiff contact systems (condition ~1e9-1e10) drifts from the true one. The
// true residual r1 = H dx - b is recomputed; while it is above tol ||b||, the
// correction H d = -r1 is solved (to the relative accuracy that brings the
// sum to tol) and added: dx <- dx + d, until the residual stops halving
// (the rounding floor of evaluating H dx - b, ~eps ||H|| ||dx||; a dense
// LAPACK solve of the same system sits at the same floor,
// tests/test_gpu_linear_solve.py). Returns the total PCG iterations.
constexpr int kMaxRefine = 3;
constexpr double kRefineMaxDrift = 1e4;  // true / tolerance ratio beyond which the solve counts as failed
int pcg(SystemImpl& S, double tol, int maxit, double* rel_out, double shift = 0.0) {
  const NvtxRange nvtx_("gmcp:K9 PCG");
  int it = pcg_core(S, tol, maxit, rel_out, shift, S.grad.p);
  if (S.cs.enabled) {  // coarse refresh policy bookkeeping
    S.cs.last_iters = it;
    if (S.cs.ref_iters < 0) S.cs.ref_iters = it;
  }
  MatSet M = mats(S);
  M.shift = shift;
  if (*rel_out == 0) {  // zero rhs: dx = 0 exactly
    S.last_true_rel2 = S.last_true_relinf = 0;
    return it;
  }
  true_residual(S, M);
  static const bool trace = std::getenv("GMCP_TRACE") != nullptr;
  if (trace)
  {
    double npc = 0;
    GMCP_CUDA(cudaMemcpyAsync(&npc, S.scal.p + 8, sizeof npc, cudaMemcpyDeviceToHost, S.stream));
    S.sync();
    std::fprintf(stderr, "[gmcp] pcg shift %.3e: %d iterations, recursive %.3e, true %.3e (inf %.3e), p.Hp<=0 %g, drift fails %lld\n",
                 shift, it, *rel_out, S.last_true_rel2, S.last_true_relinf, npc, (long long)S.drift_fails);
  }
  const int n = (int)S.n_dof;
  // refine a drifted residual only; a true residual orders of magnitude above the
  // recursive one means a failed (e.g. singular) solve -> regularized retry
  // (a regularized solve is nonsingular: its drift is refined from further away)
  const double max_drift = shift > 0 ? std::max(kRefineMaxDrift * tol, 1e-2) : kRefineMaxDrift * tol;
  for (int k = 0; k < kMaxRefine && *rel_out <= tol && S.last_true_rel2 > tol && S.last_true_rel2 < max_drift &&
                  it < maxit;
       ++k) {
    GMCP_CUDA(cudaMemcpyAsync(S.xacc.p, S.dx.p, n * sizeof(double), cudaMemcpyDeviceToDevice, S.stream));
    double rel_c;
    const double tc = std::min(0.5, 0.5 * tol / S.last_true_rel2);
    it += pcg_core(S, tc, maxit - it, &rel_c, shift, S.rt.p);  // rhs = -mask .* r1 = -r1
    k_add_into<<<grid_for(n, 256), 256, 0, S.stream>>>(n, S.xacc.p, S.dx.p);
    ++S.launches;
    S.refinements += 1;
    const double before = S.last_true_rel2;
    true_residual(S, M);
    if (!(S.last_true_rel2 < 0.5 * before)) break;  // at the FP64 floor of evaluating H dx - b
  }
  return it;
}

// A solve the Newton loop accepted: its true residual enters the statistics.
void record_accepted_solve(SystemImpl& S) {
  S.true_rel2_max = std::max(S.true_rel2_max, S.last_true_rel2);
  S.true_relinf_max = std::max(S.true_relinf_max, S.last_true_relinf);
  S.n_linear_solves += 1;
}

}  // namespace

// ---------------------------------------------------------------------------
// solve loop (solver.hpp:125-228)

// Shared solve set-up: elastic BCSR, Dirichlet targets, device vectors, the
// fixed-dof mask, run-start anchor positions, pair contexts bound to S.x/S.dx.
void setup_solve(SystemImpl& S, int64_t& n_free, DBuf<double>& eps_ref) {
  n_free = 0;
  for (uint8_t f : S.fixed) n_free += f == 0;
  if (n_free == 0) throw StatusError(GMCP_ERR_CONFIG, "solve: no free degrees of freedom");
  static const bool trace = std::getenv("GMCP_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    S.sync();
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gmcp setup] %s %.1f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  if (!S.el_built) build_elastic(S);
  lap("elastic operator + pairing");
  // fixed dofs at their targets (solver.hpp:139-140)
  for (int64_t d = 0; d < S.n_dof; ++d)
    if (S.fixed[d]) S.x_host[d] = S.dirichlet[d];
  const int64_t n = S.n_dof;
  for (auto* b : {&S.x, &S.dx, &S.xtry, &S.grad, &S.gel, &S.r, &S.z, &S.p, &S.q, &S.w, &S.rt, &S.xacc}) b->resize(n);
  S.minv.resize(3 * n);
  S.scal.resize(16);
  S.eel.resize(4);
  S.lsco.resize(4);
  S.parts.resize(kBlocks * 4);
  S.counter.resize(16);
  S.counter.zero(S.stream);
  S.redu.resize(8);
  S.x.upload(S.x_host, S.stream);
  S.dx.zero(S.stream);
  S.rest_d.upload(S.rest, S.stream);
  S.fext_d.upload(S.f_ext, S.stream);
  std::vector<double> mask(n);
  for (int64_t d = 0; d < n; ++d) mask[d] = S.fixed[d] ? 0.0 : 1.0;
  S.mask_d.upload(mask, S.stream);
  if (S.pcg_exec) {  // the coarse space (and its launch shapes) is rebuilt below
    cudaGraphExecDestroy(S.pcg_exec);
    S.pcg_exec = nullptr;
  }
  lap("vectors + mask");
  build_coarse(S, mask);
  lap("coarse space");
  eps_ref.resize(n);
  GMCP_CUDA(cudaMemcpyAsync(eps_ref.p, S.x.p, n * sizeof(double), cudaMemcpyDeviceToDevice, S.stream));
  for (auto& pr : S.pairs) {
    pr->c->x_ext = S.x.p;
    pr->c->dx_ext = S.dx.p;
    pr->c->n_dof = n;
    pr->c->stream = S.stream;
  }
}

// ---------------------------------------------------------------------------
// Batched independent scenes: one System holds S scenes in
// contiguous vertex ranges; every reduction that steers the Newton loop is
// segmented by scene (residual, step filter + cap, line-search energies and
// coefficients), each scene converges and backtracks on its own, and the
// linear solve is one PCG over the active scenes (the Hessian is block
// diagonal per scene; converged scenes are masked like fixed dofs).
namespace {

constexpr int kSceneBlk = 256;

// per scene: out[5 s + 0..4] = g_el.dx, dx.K dx, f.dx, 0.5 gel.u, f.u  (u = x - rest)
__global__ void __launch_bounds__(kSceneBlk) k_sys_scene_el(const int64_t* __restrict__ voff, Bcsr K,
                                                           const double* __restrict__ dx,
                                                           const double* __restrict__ gel,
                                                           const double* __restrict__ fext,
                                                           const double* __restrict__ x,
                                                           const double* __restrict__ rest, double* __restrict__ out) {
  __shared__ double sh[5][kSceneBlk / 32];
  const int sc = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double d[5] = {0, 0, 0, 0, 0};
  for (int64_t v = voff[sc] + wid; v < voff[sc + 1]; v += kSceneBlk / 32) {
    d3 acc = row_mv(K, (int)v, dx, lane);
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    acc.z = warp_sum(acc.z);
    if (lane == 0) {
      const d3 dv = ld3(dx, (int)v), u = ld3(x, (int)v) - ld3(rest, (int)v);
      d[0] += dot(ld3(gel, (int)v), dv);
      d[1] += dot(dv, acc);
      d[2] += dot(ld3(fext, (int)v), dv);
      d[3] += dot(ld3(gel, (int)v), u);
      d[4] += dot(ld3(fext, (int)v), u);
    }
  }
  if (lane == 0)
    for (int q = 0; q < 5; ++q) sh[q][wid] = d[q];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < 5; ++q) {
      double t = 0;
      for (int i = 0; i < kSceneBlk / 32; ++i) t += sh[q][i];
      out[5 * sc + q] = q == 3 ? 0.5 * t : t;
    }
}

// per scene: ord_bits(max |grad_d|) over free dofs
__global__ void __launch_bounds__(kSceneBlk) k_sys_scene_resid(const int64_t* __restrict__ voff,
                                                              const double* __restrict__ grad,
                                                              const double* __restrict__ mask,
                                                              unsigned long long* __restrict__ out) {
  __shared__ unsigned long long sh[kSceneBlk / 32];
  const int sc = blockIdx.x;
  unsigned long long best = 0;
  for (int64_t d = 3 * voff[sc] + threadIdx.x; d < 3 * voff[sc + 1]; d += kSceneBlk)
    if (mask[d] != 0) {
      const unsigned long long b = ord_bits(fabs(grad[d]));
      best = b > best ? b : best;
    }
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long r = 0;
    for (int i = 0; i < kSceneBlk / 32; ++i) r = max(r, sh[i]);
    out[sc] = r;
  }
}

// xtry = x + alpha_s dx per scene; x = xtry where taken_s
__global__ void k_sys_scene_axpy(int64_t n, const int32_t* __restrict__ vscene, const double* __restrict__ alpha,
                                 const double* __restrict__ x, const double* __restrict__ dx, double* __restrict__ xt) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n; d += (int64_t)gridDim.x * blockDim.x)
    xt[d] = x[d] + alpha[vscene[d / 3]] * dx[d];
}
__global__ void k_sys_scene_take(int64_t n, const int32_t* __restrict__ vscene, const int32_t* __restrict__ take,
                                 const double* __restrict__ xt, double* __restrict__ x) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n; d += (int64_t)gridDim.x * blockDim.x)
    if (take[vscene[d / 3]]) x[d] = xt[d];
}

// per-scene max |x_v - ref_v| over a pair's vertices (pair_motion per scene)
__global__ void k_sys_scene_motion(int64_t m, const int32_t* __restrict__ verts, const int32_t* __restrict__ vscene,
                                   const double* __restrict__ x, const double* __restrict__ ref,
                                   unsigned long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int v = verts[i];
    atomicMax(&out[vscene[v]], ord_bits(norm(ld3(x, v) - ld3(ref, v))));  // order-free max
  }
}
// ref = x on the vertices of the re-sampled scenes
__global__ void k_sys_scene_refpos(int64_t n, const int32_t* __restrict__ vscene, const uint8_t* __restrict__ take,
                                   const double* __restrict__ x, double* __restrict__ ref) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n; d += (int64_t)gridDim.x * blockDim.x)
    if (take[vscene[d / 3]]) ref[d] = x[d];
}

}  // namespace

// ---------------------------------------------------------------------------
// Scene-segmented PCG (batched scenes): the same arithmetic as K9 per scene --
// every dot product, alpha, beta and the convergence test are per scene
// (contiguous vertex ranges, block-per-scene fixed-order sums), so each scene
// iterates exactly as its own PCG would, and stops on its own tolerance.
namespace {

// SpMV: p_new = z + beta_s p_old, q = mask .* ((H + shift_s I) p_new); dv[v] = p_new.q
template <int kRowLanes>
__global__ void __launch_bounds__(kThreads) k_spmv_seg(int nv, MatSet M, const double* __restrict__ mask,
                                                       const int32_t* __restrict__ vscene,
                                                       const int32_t* __restrict__ act,
                                                       const double* __restrict__ st,
                                                       const double* __restrict__ shift_s,
                                                       const double* __restrict__ z, const double* __restrict__ p_old,
                                                       double* __restrict__ p_new, double* __restrict__ q,
                                                       double* __restrict__ dv) {
  const int lane = threadIdx.x & 31, sub = lane & (kRowLanes - 1);
  const int rows_per_block = kThreads / kRowLanes;
  for (int v0 = blockIdx.x * rows_per_block + (threadIdx.x >> 5) * (32 / kRowLanes); v0 < nv;
       v0 += gridDim.x * rows_per_block) {
    const int v = v0 + (lane / kRowLanes);
    // neighbours share the row's scene (the matrix is block diagonal per scene);
    // scenes that stopped are skipped (their x, r stay as they converged)
    const bool live = v < nv && act[vscene[v]];
    const double beta = live ? st[8 * vscene[v] + 3] : 0.0;
    d3 acc = mk3(0, 0, 0);
    if (live) {
      acc = row_mv8<kRowLanes>(M.el, v, z, p_old, beta, sub);
      for (int k = 0; k < M.np; ++k) acc = acc + row_mv8<kRowLanes>(M.c[k], v, z, p_old, beta, sub);
    }
#pragma unroll
    for (int o = kRowLanes / 2; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    }
    if (sub == 0 && v < nv && !live) dv[v] = 0;
    if (sub == 0 && live) {
      const d3 m = ld3(mask, v);
      const d3 pv = ld3(z, v) + beta * ld3(p_old, v);
      const double sh = shift_s[vscene[v]];
      if (sh != 0) acc = acc + sh * pv;
      const d3 y = mk3(m.x * acc.x, m.y * acc.y, m.z * acc.z);
      q[3 * v] = y.x;
      q[3 * v + 1] = y.y;
      q[3 * v + 2] = y.z;
      p_new[3 * v] = pv.x;
      p_new[3 * v + 1] = pv.y;
      p_new[3 * v + 2] = pv.z;
      dv[v] = dot(pv, y);
    }
  }
}

// per scene: sum of dv over its vertices (fixed order). mode 0: pq -> alpha;
// mode 1: (rz_new, rr) -> beta, rz, rr, active flag; mode 2: init (rz, rr, bb)
template <int Mode>
__global__ void __launch_bounds__(kSceneBlk) k_seg_sums(const int64_t* __restrict__ voff,
                                                        const double* __restrict__ dv, int nv, double tol2,
                                                        double* __restrict__ st, int32_t* __restrict__ act) {
  // st[8 s + 0] rz, [1] pq, [2] alpha, [3] beta, [4] rr, [5] bb
  __shared__ double sh[2][kSceneBlk / 32];
  const int sc = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int W = Mode == 0 ? 1 : 2;
  double a[2] = {0, 0};
  for (int64_t v = voff[sc] + threadIdx.x; v < voff[sc + 1]; v += kSceneBlk)
    for (int q = 0; q < W; ++q) a[q] += dv[(int64_t)q * nv + v];
  for (int q = 0; q < W; ++q) {
    const double t = warp_sum(a[q]);
    if (lane == 0) sh[q][wid] = t;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double r[2] = {0, 0};
  for (int q = 0; q < W; ++q)
    for (int i = 0; i < kSceneBlk / 32; ++i) r[q] += sh[q][i];
  double* s = st + 8 * sc;
  if (Mode == 0) {
    s[1] = r[0];
    s[2] = act[sc] && r[0] != 0 ? s[0] / r[0] : 0.0;
  } else if (Mode == 1) {
    if (act[sc]) {
      s[3] = s[0] != 0 ? r[0] / s[0] : 0.0;
      s[0] = r[0];
      s[4] = r[1];
      act[sc] = r[1] > tol2 * s[5] ? 1 : 0;  // converged (or non-finite) -> stop
    }
  } else {
    s[0] = r[0];
    s[3] = 0.0;
    s[4] = r[1];
    s[5] = r[1];
    act[sc] = act[sc] && r[1] > 0 ? 1 : 0;
  }
}

// x += alpha_s p, r -= alpha_s q, z = Minv r; dv = (r.z, r.r) per vertex
__global__ void __launch_bounds__(kThreads) k_update_seg(int nv, const int32_t* __restrict__ vscene,
                                                         const int32_t* __restrict__ act,
                                                         const double* __restrict__ st, const double* __restrict__ p,
                                                         const double* __restrict__ q, double* __restrict__ x,
                                                         double* __restrict__ r, double* __restrict__ z,
                                                         const double* __restrict__ minv, double* __restrict__ dv) {
  for (int v = blockIdx.x * kThreads + threadIdx.x; v < nv; v += gridDim.x * kThreads) {
    if (!act[vscene[v]]) {
      dv[v] = 0;
      dv[nv + v] = 0;
      continue;
    }
    const double a = st[8 * vscene[v] + 2];
    const d3 xv = ld3nc(x, v) + a * ld3nc(p, v);
    const d3 rv = ld3nc(r, v) - a * ld3nc(q, v);
    const d3 zv = bmv(minv + 9 * (int64_t)v, rv);
    const double xa[3] = {xv.x, xv.y, xv.z}, ra[3] = {rv.x, rv.y, rv.z}, za[3] = {zv.x, zv.y, zv.z};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      x[3 * v + c] = xa[c];
      r[3 * v + c] = ra[c];
      z[3 * v + c] = za[c];
    }
    dv[v] = dot(rv, zv);
    dv[nv + v] = dot(rv, rv);
  }
}

// init: x = p = 0, r = -mask .* grad, z = Minv r; dv = (r.z, r.r)
__global__ void k_init_seg(int nv, const int32_t* __restrict__ vscene, const int32_t* __restrict__ act,
                           const double* __restrict__ grad, const double* __restrict__ mask,
                           const double* __restrict__ minv, double* __restrict__ x, double* __restrict__ r,
                           double* __restrict__ z, double* __restrict__ p, double* __restrict__ dv) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    if (!act[vscene[v]]) {  // scenes not being solved keep their x (dx)
      dv[v] = 0;
      dv[nv + v] = 0;
      continue;
    }
    const d3 m = ld3(mask, v), g = ld3(grad, v);
    const d3 rv = mk3(-m.x * g.x, -m.y * g.y, -m.z * g.z);
    const d3 zv = bmv(minv + 9 * (int64_t)v, rv);
    const double ra[3] = {rv.x, rv.y, rv.z}, za[3] = {zv.x, zv.y, zv.z};
    for (int k = 0; k < 3; ++k) {
      x[3 * v + k] = 0;
      p[3 * v + k] = 0;
      r[3 * v + k] = ra[k];
      z[3 * v + k] = za[k];
    }
    dv[v] = dot(rv, zv);
    dv[nv + v] = dot(rv, rv);
  }
}

// block-Jacobi with a per-scene diagonal shift
__global__ void k_block_jacobi_seg(int nv, MatSet M, const double* __restrict__ mask,
                                   const int32_t* __restrict__ vscene, const double* __restrict__ shift_s,
                                   double* __restrict__ minv) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    double D[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    get_diag(M.el, v, D);
    const double sh = shift_s[vscene[v]];
    D[0] += sh;
    D[4] += sh;
    D[8] += sh;
    const double m[3] = {mask[3 * v], mask[3 * v + 1], mask[3 * v + 2]};
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        if (m[a] == 0 || m[b] == 0) D[3 * a + b] = (a == b) ? 1.0 : 0.0;
    const double c00 = D[4] * D[8] - D[5] * D[7], c01 = D[2] * D[7] - D[1] * D[8], c02 = D[1] * D[5] - D[2] * D[4];
    const double c10 = D[5] * D[6] - D[3] * D[8], c11 = D[0] * D[8] - D[2] * D[6], c12 = D[2] * D[3] - D[0] * D[5];
    const double c20 = D[3] * D[7] - D[4] * D[6], c21 = D[1] * D[6] - D[0] * D[7], c22 = D[0] * D[4] - D[1] * D[3];
    const double det = D[0] * c00 + D[1] * c10 + D[2] * c20;
    double* o = minv + 9 * (int64_t)v;
    if (det != 0 && isfinite(det)) {
      const double id = 1.0 / det;
      o[0] = c00 * id; o[1] = c01 * id; o[2] = c02 * id;
      o[3] = c10 * id; o[4] = c11 * id; o[5] = c12 * id;
      o[6] = c20 * id; o[7] = c21 * id; o[8] = c22 * id;
    } else {
      for (int q = 0; q < 9; ++q) o[q] = 0;
      for (int a = 0; a < 3; ++a) o[4 * a] = D[4 * a] != 0 ? 1.0 / D[4 * a] : 1.0;
    }
  }
}

// per scene: sum of the free diagonal entries of H (the regularization scale)
__global__ void __launch_bounds__(kSceneBlk) k_seg_diag(int nv, MatSet M, const double* __restrict__ mask,
                                                        const int64_t* __restrict__ voff, double* __restrict__ out) {
  __shared__ double sh[kSceneBlk / 32];
  const int sc = blockIdx.x;
  double acc = 0;
  for (int64_t v = voff[sc] + threadIdx.x; v < voff[sc + 1]; v += kSceneBlk) {
    double e[9];
    if (get_diag(M.el, (int)v, e))
      for (int a = 0; a < 3; ++a)
        if (mask[3 * v + a] != 0) acc += e[4 * a];
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int i = 0; i < kSceneBlk / 32; ++i) t += sh[i];
    out[sc] = t;
  }
}

}  // namespace

struct SegPcgTmp {
  DBuf<unsigned long long> tr;  // per-scene true-residual maxima (k_scene_true_resid)
  DBuf<double> dv, st, shift;
  DBuf<int32_t> act, vscene;
  DBuf<int64_t> voff;
};

// Batched scenes with up to kCtaSceneRows rows each: one CTA runs one scene's
// whole PCG in a single launch. Scene matrices are independent (block
// diagonal), so a CTA needs no grid-level synchronisation: per iteration the
// SpMV (8-lane row groups over the merged BCSR, as k_spmv_cg<8>), the fixed-
// order block reductions of p.q and (r.z, r.r) and the vector updates are
// separated by __syncthreads, and the CTA stops at its own convergence. This
// removes the four whole-batch launches per iteration of the segmented path
// and lets converged scenes leave the GPU to the others.
constexpr int kCtaSceneRows = 16384;
constexpr int kCtaThreads = 128;  // 8 CTAs per SM: all 1024 C5 scenes resident in one wave

template <int NT = kCtaThreads>
__device__ __forceinline__ void cta_sum2(double& a, double& b, double (*sh)[NT / 32]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();  // sh free (previous readers done)
  if (lane == 0) {
    sh[0][wid] = a;
    sh[1][wid] = b;
  }
  __syncthreads();
  double s0 = 0, s1 = 0;
  for (int i = 0; i < NT / 32; ++i) {  // every thread, same order: uniform result
    s0 += sh[0][i];
    s1 += sh[1][i];
  }
  a = s0;
  b = s1;
}

// Per-scene two-level correction inside the CTA PCG (coarse.cuh): the scene's
// own rigid-mode coarse space and dense pseudo-inverse.
struct SceneCoarse {
  const int32_t* agg;        // [nv] global aggregate id
  const double* dvec;        // [nv][3]
  const int32_t* agg_off;    // aggregate vertex lists (ascending ids)
  const int32_t* agg_verts;
  const int32_t* scene_agg;  // [NS+1] aggregate range of each scene
  const int64_t* scene_coff; // [NS+1] offset of each scene's inverse
  const double* inv;         // scaled pseudo-inverses
  const double* scale;       // [6 n_agg]
};

// z += P Ac^+ P^T r over the CTA's scene (r, z written earlier in this
// kernel: plain loads); returns s.y, identical in every thread. Restriction:
// warp w sums aggregates w, w + 4, ... (lanes over the vertex list, fixed
// butterfly); coarse rows: one warp per row; prolongation: the thread's own
// vertices (the update loop's assignment).
template <int NT = kCtaThreads>
__device__ double scene_coarse(int sc, int v0, int v1, const double* r, double* z, const double* __restrict__ mask,
                               const SceneCoarse& C, double* s_sm, double* y_sm, double (*sh)[NT / 32]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int a0 = C.scene_agg[sc], na = C.scene_agg[sc + 1] - a0, dim = 6 * na;
  const double* Ai = C.inv + C.scene_coff[sc];
  const double* scl = C.scale + 6 * (int64_t)a0;
  for (int la = wid; la < na; la += NT / 32) {
    const int a = a0 + la;
    double t[6] = {0, 0, 0, 0, 0, 0};
    for (int e = __ldg(C.agg_off + a) + lane; e < __ldg(C.agg_off + a + 1); e += 32) {
      const int v = __ldg(C.agg_verts + e);
      const d3 m = ld3(mask, v), rv = ld3nc(r, v);
      const d3 q = mk3(m.x * rv.x, m.y * rv.y, m.z * rv.z);
      const d3 w = cross(ld3(C.dvec, v), q);
      t[0] += q.x;
      t[1] += q.y;
      t[2] += q.z;
      t[3] += w.x;
      t[4] += w.y;
      t[5] += w.z;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) t[k] = warp_sum(t[k]);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < 6; ++k) s_sm[6 * la + k] = t[k] * __ldg(scl + 6 * la + k);
  }
  __syncthreads();
  double sy = 0;
  for (int i = wid; i < dim; i += NT / 32) {
    const double* row = Ai + (int64_t)i * dim;
    double acc = 0;
    for (int j = lane; j < dim; j += 32) acc += __ldg(row + j) * s_sm[j];
    acc = warp_sum(acc);
    if (lane == 0) {
      y_sm[i] = __ldg(scl + i) * acc;
      sy += s_sm[i] * acc;
    }
  }
  __syncthreads();
  for (int v = v0 + threadIdx.x; v < v1; v += NT) {
    const int la = __ldg(C.agg + v) - a0;
    const double* ya = y_sm + 6 * la;
    const d3 u = mk3(ya[0], ya[1], ya[2]) + cross(mk3(ya[3], ya[4], ya[5]), ld3(C.dvec, v));
    const d3 m = ld3(mask, v);
    z[3 * v] += m.x * u.x;
    z[3 * v + 1] += m.y * u.y;
    z[3 * v + 2] += m.z * u.z;
  }
  double unused = 0;
  cta_sum2<NT>(sy, unused, sh);  // lane-0 partials of each warp, summed in warp order
  return sy;
}

// st[8 s + 0] rz, [1] pq, [2] alpha, [3] beta, [4] rr, [5] bb, [6] iterations,
// [7] 1 indefinite / 2 drifted (two-level only; the caller retries regularized)
template <bool kCoarse>
__global__ void __launch_bounds__(kCtaThreads, 8) k_pcg_scene(MatSet M, const double* __restrict__ mask,
                                                          const int64_t* __restrict__ voff,
                                                          const int32_t* __restrict__ act,
                                                          const double* __restrict__ shift_s,
                                                          const double* __restrict__ minv,
                                                          const double* __restrict__ grad, double* __restrict__ x,
                                                          double* r, double* z, double* __restrict__ p,
                                                          double* __restrict__ q, double tol2, int maxit,
                                                          double* __restrict__ st, SceneCoarse CS,
                                                          const int32_t* __restrict__ pair,
                                                          const double* __restrict__ minv2) {
  __shared__ double sh[2][kCtaThreads / 32];
  __shared__ double s_sm[kCoarse ? kSceneCoarseMax : 1], y_sm[kCoarse ? kSceneCoarseMax : 1];
  const int sc = blockIdx.x;
  if (!act[sc]) return;  // scenes not being solved keep their x (dx)
  const int v0 = (int)voff[sc], v1 = (int)voff[sc + 1];
  const double shift = shift_s[sc];
  // init: x = 0, r = -mask .* grad, z = Minv r, p = z
  double rz = 0, rr = 0;
  // vertex-pair smoother (pair != null): z_v = Minv2_v [r_v; r_partner] needs
  // the partner's residual, so r is written in its own loop and published first
  if (pair) {
    for (int v = v0 + threadIdx.x; v < v1; v += kCtaThreads) {
      const d3 m = ld3(mask, v), g = ld3(grad, v);
      r[3 * v] = -m.x * g.x;
      r[3 * v + 1] = -m.y * g.y;
      r[3 * v + 2] = -m.z * g.z;
    }
    __syncthreads();
  }
  for (int v = v0 + threadIdx.x; v < v1; v += kCtaThreads) {
    const d3 m = ld3(mask, v), g = ld3(grad, v);
    const d3 rv = mk3(-m.x * g.x, -m.y * g.y, -m.z * g.z);
    d3 zv;
    if (pair) {
      const int pp = pair[v];
      zv = pair_apply(minv2, v, rv, pp < 0 ? mk3(0, 0, 0) : ld3nc(r, pp));
    } else {
      zv = bmv(minv + 9 * (int64_t)v, rv);
    }
    const double ra[3] = {rv.x, rv.y, rv.z}, za[3] = {zv.x, zv.y, zv.z};
    for (int k = 0; k < 3; ++k) {
      x[3 * v + k] = 0;
      r[3 * v + k] = ra[k];
      z[3 * v + k] = za[k];
      if (!kCoarse) p[3 * v + k] = za[k];
    }
    rz += dot(rv, zv);
    rr += dot(rv, rv);
  }
  cta_sum2(rz, rr, sh);
  bool indefinite = false;  // two-level M^-1 lost positivity (r.z <= 0 with r != 0)
  bool drifted = false;     // true residual stalled far above the recursive one
  if (kCoarse) {  // z += P Ac^+ P^T r, then p = z (own rows)
    rz += scene_coarse(sc, v0, v1, r, z, mask, CS, s_sm, y_sm, sh);
    indefinite = !(rz > 0) && rr > 0;
    for (int v = v0 + threadIdx.x; v < v1; v += kCtaThreads)
      for (int k = 0; k < 3; ++k) p[3 * v + k] = z[3 * v + k];
  }
  const double bb = rr;
  int it = 0;
  double pq = 0, alpha = 0, beta = 0;
  double win_min = INFINITY, prev_min = INFINITY;  // stagnation windows (kStagWindow)
  const int lane = threadIdx.x & 31, sub = lane & 7;
  while (rr > tol2 * bb && it < maxit && !indefinite) {
    __syncthreads();  // p complete
    // q = mask .* ((H + shift I) p); pq
    double pqa = 0, unused = 0;
    for (int vb = v0 + (threadIdx.x >> 3); vb - (lane >> 3) < v1; vb += kCtaThreads / 8) {
      const int v = vb;  // 8 lanes per row; a warp covers 4 rows
      d3 acc = mk3(0, 0, 0);
      if (v < v1) acc = row_mv8<8>(M.el, v, p, p, 0.0, sub);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
      }
      if (sub == 0 && v < v1) {
        const d3 m = ld3(mask, v), pv = ld3nc(p, v);
        if (shift != 0) acc = acc + shift * pv;
        const d3 y = mk3(m.x * acc.x, m.y * acc.y, m.z * acc.z);
        q[3 * v] = y.x;
        q[3 * v + 1] = y.y;
        q[3 * v + 2] = y.z;
        pqa += dot(pv, y);
      }
    }
    cta_sum2(pqa, unused, sh);  // includes the barrier that publishes q
    pq = pqa;
    alpha = pq != 0 ? rz / pq : 0.0;
    // x += alpha p, r -= alpha q, z = Minv r; (r.z, r.r)
    double rzn = 0, rrn = 0;
    if (pair) {  // r first (published), then z from the vertex and its partner
      for (int v = v0 + threadIdx.x; v < v1; v += kCtaThreads) {
        const d3 xv = ld3nc(x, v) + alpha * ld3nc(p, v);
        const d3 rv = ld3nc(r, v) - alpha * ld3nc(q, v);
        x[3 * v] = xv.x;
        x[3 * v + 1] = xv.y;
        x[3 * v + 2] = xv.z;
        r[3 * v] = rv.x;
        r[3 * v + 1] = rv.y;
        r[3 * v + 2] = rv.z;
      }
      __syncthreads();
      for (int v = v0 + threadIdx.x; v < v1; v += kCtaThreads) {
        const d3 rv = ld3nc(r, v);
        const int pp = pair[v];
        const d3 zv = pair_apply(minv2, v, rv, pp < 0 ? mk3(0, 0, 0) : ld3nc(r, pp));
        z[3 * v] = zv.x;
        z[3 * v + 1] = zv.y;
        z[3 * v + 2] = zv.z;
        rzn += dot(rv, zv);
        rrn += dot(rv, rv);
      }
    } else {
    for (int v = v0 + threadIdx.x; v < v1; v += kCtaThreads) {
      const d3 xv = ld3nc(x, v) + alpha * ld3nc(p, v);
      const d3 rv = ld3nc(r, v) - alpha * ld3nc(q, v);
      const d3 zv = bmv(minv + 9 * (int64_t)v, rv);
      const double xa[3] = {xv.x, xv.y, xv.z}, ra[3] = {rv.x, rv.y, rv.z}, za[3] = {zv.x, zv.y, zv.z};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        x[3 * v + c] = xa[c];
        r[3 * v + c] = ra[c];
        z[3 * v + c] = za[c];
      }
      rzn += dot(rv, zv);
      rrn += dot(rv, rv);
    }
    }
    cta_sum2(rzn, rrn, sh);
    if (kCoarse) {
      rzn += scene_coarse(sc, v0, v1, r, z, mask, CS, s_sm, y_sm, sh);
      if (!(rzn > 0) && rrn > 0) {
        indefinite = true;
        rr = rrn;
        break;
      }
    }
    beta = rz != 0 ? rzn / rz : 0.0;
    rz = rzn;
    rr = rrn;
    ++it;
    if (!isfinite(rr)) break;
    if (kCoarse && it % kDriftWindow == 0) {
      // true residual ||mask .* (grad + (H + shift) x)|| (x complete: the
      // update's reductions ended in barriers); a gap to the recursive one that
      // no refinement closes (a singular scene) fails the solve now -> retry
      double tr = 0, unused2 = 0;
      for (int vb = v0 + (threadIdx.x >> 3); vb - (lane >> 3) < v1; vb += kCtaThreads / 8) {
        const int v = vb;
        d3 acc = mk3(0, 0, 0);
        if (v < v1) acc = row_mv8<8>(M.el, v, x, x, 0.0, sub);
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
          acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
        }
        if (sub == 0 && v < v1) {
          const d3 m = ld3(mask, v), g = ld3(grad, v), xv = ld3nc(x, v);
          if (shift != 0) acc = acc + shift * xv;
          const d3 e = mk3(m.x * (acc.x + g.x), m.y * (acc.y + g.y), m.z * (acc.z + g.z));
          tr += dot(e, e);
        }
      }
      cta_sum2(tr, unused2, sh);
      if (sqrt(tr / bb) - sqrt(rr / bb) > kDriftFail * sqrt(tol2) || (shift == 0 && sqrt(tr / bb) > kDivergeRel)) {
        drifted = true;
        break;
      }
    }
    win_min = fmin(win_min, rr);
    constexpr int stag = kCoarse ? kStagWindowCoarse : kStagWindow;
    if (it % stag == 0) {
      if (it >= 2 * stag && !(win_min < 0.5 * prev_min) && rr > 1e-8 * bb) break;  // stagnated
      prev_min = fmin(prev_min, win_min);
      win_min = INFINITY;
    }
    // p = z + beta p (own rows; the barrier at the loop head publishes it)
    for (int v = v0 + threadIdx.x; v < v1; v += kCtaThreads) {
      const d3 pv = ld3nc(z, v) + beta * ld3nc(p, v);
      p[3 * v] = pv.x;
      p[3 * v + 1] = pv.y;
      p[3 * v + 2] = pv.z;
    }
  }
  if (threadIdx.x == 0) {
    double* o = st + 8 * sc;
    o[0] = rz;
    o[1] = pq;
    o[2] = alpha;
    o[3] = beta;
    o[4] = rr;
    o[5] = bb;
    o[6] = (double)it;
    o[7] = indefinite ? 1.0 : drifted ? 2.0 : 0.0;
  }
}

// The same per-scene PCG with the scene's p, r and z in shared memory: the
// SpMV gathers p from shared memory, the smoother reads its partners' r there,
// and the operand, the smoother rows, the coarse inverse, q and x stream from
// HBM. Used when every scene fits (kSmSceneBytes); same arithmetic as
// k_pcg_scene except for the summation layout of the dots.
// NT threads per scene CTA, MINB CTAs per SM; p always in shared memory, r
// and z when kRZ (else in the global buffers rg / zg), q in global memory.
// (p alone in shared memory with 128 threads x 6 CTAs per SM: 6,736 vs 8,014
// scene-Newton-steps/s for the global kernel -- the 1.15-wave tail; p, r, z
// with 512 x 2: 8,403; 1024 x 1: 7,910.)
constexpr int kSmThreads = 512;
constexpr size_t kSmSceneBytes = 110 * 1024;  // two CTAs per SM
template <bool kCoarse, int NT, int MINB, bool kRZ>
__global__ void __launch_bounds__(NT, MINB) k_pcg_scene_sm(MatSet M, const double* __restrict__ mask,
                                                               const int64_t* __restrict__ voff,
                                                               const int32_t* __restrict__ act,
                                                               const double* __restrict__ shift_s,
                                                               const double* __restrict__ minv,
                                                               const double* __restrict__ grad,
                                                               double* __restrict__ x, double* __restrict__ qg,
                                                               double* __restrict__ rg, double* __restrict__ zg,
                                                               double tol2, int maxit,
                                                               double* __restrict__ st, SceneCoarse CS,
                                                               const int32_t* __restrict__ pair,
                                                               const double* __restrict__ minv2, int max_rows,
                                                               int coarse_dim) {
  extern __shared__ double dsm[];
  constexpr int kSmThreads = NT;
  __shared__ double sh[2][kSmThreads / 32];
  const int sc = blockIdx.x;
  if (!act[sc]) return;
  const int v0 = (int)voff[sc], v1 = (int)voff[sc + 1];
  // scene-local vectors, indexed by global vertex id through the shifted bases
  double* const ps = dsm;
  double* const rs = ps + 3 * (int64_t)max_rows;
  double* const zs = kRZ ? rs + 3 * (int64_t)max_rows : rs;
  double* const s_sm = kRZ ? zs + 3 * (int64_t)max_rows : rs;
  double* const y_sm = s_sm + coarse_dim;
  double* const p = ps - 3 * (int64_t)v0;
  double* const q = qg;  // q in global memory (written and read once per iteration)
  double* const r = kRZ ? rs - 3 * (int64_t)v0 : rg;
  double* const z = kRZ ? zs - 3 * (int64_t)v0 : zg;
  const double shift = shift_s[sc];
  double rz = 0, rr = 0;
  for (int v = v0 + threadIdx.x; v < v1; v += kSmThreads) {
    const d3 m = ld3(mask, v), g = ld3(grad, v);
    r[3 * v] = -m.x * g.x;
    r[3 * v + 1] = -m.y * g.y;
    r[3 * v + 2] = -m.z * g.z;
  }
  __syncthreads();
  for (int v = v0 + threadIdx.x; v < v1; v += kSmThreads) {
    const d3 rv = ld3nc(r, v);
    d3 zv;
    if (pair) {
      const int pp = pair[v];
      zv = pair_apply(minv2, v, rv, pp < 0 ? mk3(0, 0, 0) : ld3nc(r, pp));
    } else {
      zv = bmv(minv + 9 * (int64_t)v, rv);
    }
    x[3 * v] = x[3 * v + 1] = x[3 * v + 2] = 0;
    z[3 * v] = zv.x;
    z[3 * v + 1] = zv.y;
    z[3 * v + 2] = zv.z;
    if (!kCoarse) {
      p[3 * v] = zv.x;
      p[3 * v + 1] = zv.y;
      p[3 * v + 2] = zv.z;
    }
    rz += dot(rv, zv);
    rr += dot(rv, rv);
  }
  cta_sum2<kSmThreads>(rz, rr, sh);
  bool indefinite = false, drifted = false;
  if (kCoarse) {  // z += P Ac^+ P^T r, then p = z
    rz += scene_coarse<kSmThreads>(sc, v0, v1, r, z, mask, CS, s_sm, y_sm, sh);
    indefinite = !(rz > 0) && rr > 0;
    __syncthreads();
    for (int v = v0 + threadIdx.x; v < v1; v += kSmThreads)
      for (int k = 0; k < 3; ++k) p[3 * v + k] = z[3 * v + k];
  }
  const double bb = rr;
  int it = 0;
  double pq = 0, alpha = 0, beta = 0;
  double win_min = INFINITY, prev_min = INFINITY;
  const int lane = threadIdx.x & 31, sub = lane & 7;
  const Bcsr& A = M.el;
  while (rr > tol2 * bb && it < maxit && !indefinite) {
    __syncthreads();  // p complete
    double pqa = 0, unused = 0;
    for (int vb = v0 + (threadIdx.x >> 3); vb - (lane >> 3) < v1; vb += kSmThreads / 8) {
      const int v = vb;
      d3 acc0 = mk3(0, 0, 0), acc1 = mk3(0, 0, 0);
      if (v < v1) {
        const int a = __ldg(A.rowptr + v), b = __ldg(A.rowptr + v + 1);
        int k = a + sub;
        for (; k + 8 < b; k += 16) {
          const int j0 = __ldg(A.cols + k), j1 = __ldg(A.cols + k + 8);
          acc0 = acc0 + bmv_ro(A, k, ld3nc(p, j0));
          acc1 = acc1 + bmv_ro(A, k + 8, ld3nc(p, j1));
        }
        if (k < b) acc0 = acc0 + bmv_ro(A, k, ld3nc(p, __ldg(A.cols + k)));
      }
      d3 acc = acc0 + acc1;
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
      }
      if (sub == 0 && v < v1) {
        const d3 m = ld3(mask, v), pv = ld3nc(p, v);
        if (shift != 0) acc = acc + shift * pv;
        const d3 y = mk3(m.x * acc.x, m.y * acc.y, m.z * acc.z);
        q[3 * v] = y.x;
        q[3 * v + 1] = y.y;
        q[3 * v + 2] = y.z;
        pqa += dot(pv, y);
      }
    }
    cta_sum2<kSmThreads>(pqa, unused, sh);  // includes the barrier that publishes q
    pq = pqa;
    alpha = pq != 0 ? rz / pq : 0.0;
    double rzn = 0, rrn = 0;
    for (int v = v0 + threadIdx.x; v < v1; v += kSmThreads) {  // x += alpha p, r -= alpha q
      const d3 xv = ld3nc(x, v) + alpha * ld3nc(p, v);
      const d3 rv = ld3nc(r, v) - alpha * ld3nc(q, v);
      x[3 * v] = xv.x;
      x[3 * v + 1] = xv.y;
      x[3 * v + 2] = xv.z;
      r[3 * v] = rv.x;
      r[3 * v + 1] = rv.y;
      r[3 * v + 2] = rv.z;
    }
    __syncthreads();  // r published (pair partners)
    for (int v = v0 + threadIdx.x; v < v1; v += kSmThreads) {  // z = M1^-1 r
      const d3 rv = ld3nc(r, v);
      d3 zv;
      if (pair) {
        const int pp = pair[v];
        zv = pair_apply(minv2, v, rv, pp < 0 ? mk3(0, 0, 0) : ld3nc(r, pp));
      } else {
        zv = bmv(minv + 9 * (int64_t)v, rv);
      }
      z[3 * v] = zv.x;
      z[3 * v + 1] = zv.y;
      z[3 * v + 2] = zv.z;
      rzn += dot(rv, zv);
      rrn += dot(rv, rv);
    }
    cta_sum2<kSmThreads>(rzn, rrn, sh);
    if (kCoarse) {
      rzn += scene_coarse<kSmThreads>(sc, v0, v1, r, z, mask, CS, s_sm, y_sm, sh);
      if (!(rzn > 0) && rrn > 0) {
        indefinite = true;
        rr = rrn;
        break;
      }
    }
    beta = rz != 0 ? rzn / rz : 0.0;
    rz = rzn;
    rr = rrn;
    ++it;
    if (!isfinite(rr)) break;
    if (kCoarse && it % kDriftWindow == 0) {  // true residual from x (global, plain loads)
      __syncthreads();
      double tr = 0, unused2 = 0;
      for (int vb = v0 + (threadIdx.x >> 3); vb - (lane >> 3) < v1; vb += kSmThreads / 8) {
        const int v = vb;
        d3 acc = mk3(0, 0, 0);
        if (v < v1)
          for (int k = __ldg(A.rowptr + v) + sub; k < __ldg(A.rowptr + v + 1); k += 8)
            acc = acc + bmv_ro(A, k, ld3nc(x, __ldg(A.cols + k)));
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
          acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
        }
        if (sub == 0 && v < v1) {
          const d3 m = ld3(mask, v), g = ld3(grad, v), xv = ld3nc(x, v);
          if (shift != 0) acc = acc + shift * xv;
          const d3 e = mk3(m.x * (acc.x + g.x), m.y * (acc.y + g.y), m.z * (acc.z + g.z));
          tr += dot(e, e);
        }
      }
      cta_sum2<kSmThreads>(tr, unused2, sh);
      if (sqrt(tr / bb) - sqrt(rr / bb) > kDriftFail * sqrt(tol2) || (shift == 0 && sqrt(tr / bb) > kDivergeRel)) {
        drifted = true;
        break;
      }
    }
    win_min = fmin(win_min, rr);
    constexpr int stag = kCoarse ? kStagWindowCoarse : kStagWindow;
    if (it % stag == 0) {
      if (it >= 2 * stag && !(win_min < 0.5 * prev_min) && rr > 1e-8 * bb) break;  // stagnated
      prev_min = fmin(prev_min, win_min);
      win_min = INFINITY;
    }
    __syncthreads();  // z complete (coarse prolongation) before p = z + beta p
    for (int v = v0 + threadIdx.x; v < v1; v += kSmThreads) {
      const d3 pv = ld3nc(z, v) + beta * ld3nc(p, v);
      p[3 * v] = pv.x;
      p[3 * v + 1] = pv.y;
      p[3 * v + 2] = pv.z;
    }
  }
  if (threadIdx.x == 0) {
    double* o = st + 8 * sc;
    o[0] = rz;
    o[1] = pq;
    o[2] = alpha;
    o[3] = beta;
    o[4] = rr;
    o[5] = bb;
    o[6] = (double)it;
    o[7] = indefinite ? 1.0 : drifted ? 2.0 : 0.0;
  }
}

// Per scene (one CTA): max |mask .* ((H + shift I) dx) + mask .* grad| and
// max |mask .* grad| (the reference's inf-norm acceptance test,
// solver.hpp:349-356), as ordered bits (max is order-free).
__global__ void __launch_bounds__(kSceneBlk) k_scene_true_resid(MatSet M, const double* __restrict__ mask,
                                                                const int64_t* __restrict__ voff,
                                                                const int32_t* __restrict__ act,
                                                                const double* __restrict__ shift_s,
                                                                const double* __restrict__ dx,
                                                                const double* __restrict__ grad,
                                                                unsigned long long* __restrict__ out) {
  __shared__ unsigned long long sm[2][kSceneBlk / 32];
  const int sc = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long mr = 0, mb = 0;
  if (act[sc]) {
    for (int64_t v = voff[sc] + wid; v < voff[sc + 1]; v += kSceneBlk / 32) {
      d3 acc = mk3(0, 0, 0);
      for (int k = M.el.rowptr[v] + lane; k < M.el.rowptr[v + 1]; k += 32)
        acc = acc + bmv_ro(M.el, k, ld3(dx, M.el.cols[k]));
      acc.x = warp_sum(acc.x);
      acc.y = warp_sum(acc.y);
      acc.z = warp_sum(acc.z);
      if (lane == 0) {
        const d3 m = ld3(mask, (int)v), g = ld3(grad, (int)v), d = ld3(dx, (int)v);
        const double sh = shift_s[sc];
        const double y[3] = {acc.x + sh * d.x, acc.y + sh * d.y, acc.z + sh * d.z};
        const double ma[3] = {m.x, m.y, m.z}, ga[3] = {g.x, g.y, g.z};
        for (int a = 0; a < 3; ++a) {
          const unsigned long long br = ord_bits(fabs(ma[a] * y[a] + ma[a] * ga[a])), bb = ord_bits(fabs(ma[a] * ga[a]));
          mr = br > mr ? br : mr;
          mb = bb > mb ? bb : mb;
        }
      }
    }
  }
  if (lane == 0) {
    sm[0][wid] = mr;
    sm[1][wid] = mb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kSceneBlk / 32; ++w) {
      mr = max(mr, sm[0][w]);
      mb = max(mb, sm[1][w]);
    }
    out[2 * sc] = max(mr, sm[0][0]);
    out[2 * sc + 1] = max(mb, sm[1][0]);
  }
}

// Runs the segmented PCG for the scenes with active[s]; returns iterations of
// the slowest scene; rel[s] = sqrt(rr_s / bb_s) at exit (0 when bb_s = 0).
int pcg_batched(SystemImpl& S, SegPcgTmp& T, double tol, int maxit, const std::vector<int32_t>& active,
                const std::vector<double>& shift, std::vector<double>& rel, bool allow_coarse = false,
                std::vector<int32_t>* bad = nullptr) {
  const NvtxRange nvtx_("gmcp:K9 PCG (scenes)");
  const int nv = S.nv(), NS = S.n_scenes;
  cudaStream_t s = S.stream;
  MatSet M = mats(S);
  T.dv.resize(2 * (int64_t)nv);
  T.st.resize(8 * NS);
  T.st.zero(s);
  T.act.upload(active, s);
  T.shift.upload(shift, s);
  k_block_jacobi_seg<<<grid_for(nv, 256), 256, 0, s>>>(nv, M, S.mask_d.p, T.vscene.p, T.shift.p, S.minv.p);
  ++S.launches;
  // the per-scene CTA PCG smooths with the vertex-pair 6x6 block-Jacobi when
  // the system has a pairing (every pair lies in one body, so in one scene)
  const bool pair_smoother = S.has_pairs && S.pair_d.n == (size_t)nv;
  if (pair_smoother) {
    S.minv2.resize(18 * (int64_t)nv);
    k_pair_jacobi<<<grid_for(nv, 128), 128, 0, s>>>(nv, M, S.mask_d.p, S.pair_d.p, S.minv2.p, T.vscene.p, T.shift.p);
    ++S.launches;
  }
  int64_t max_rows = 0;
  for (int sc = 0; sc < NS; ++sc) max_rows = std::max(max_rows, S.scene_voff[sc + 1] - S.scene_voff[sc]);
  if (max_rows <= kCtaSceneRows && !std::getenv("GMCP_SEG_PCG")) {  // one CTA per scene
    CoarseSpace& C = S.cs;
    const bool coarse = allow_coarse && C.enabled && M.np == 0;
    SceneCoarse CS{};
    if (coarse) {
      coarse_setup_scenes(S, M, T.shift.p);
      CS = SceneCoarse{C.agg.p, C.dvec.p, C.agg_off.p, C.agg_verts.p, C.scene_agg.p, C.scene_coff.p, C.A.p,
                       C.scale.p};
    }
    // p, r and z of each scene in shared memory (512 threads, two scenes per SM)
    // when every scene fits; GMCP_SCENE_SMEM=0 selects the global-memory kernel
    static const bool smem_on = !std::getenv("GMCP_SCENE_SMEM") || std::atoi(std::getenv("GMCP_SCENE_SMEM")) != 0;
    const int cdim = coarse ? std::max(C.n_scene_c, 1) : 1;
    const size_t smem = (9 * (size_t)max_rows + 2 * cdim) * sizeof(double);
    auto launch = [&](auto kern) {
      GMCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<NS, kSmThreads, smem, s>>>(M, S.mask_d.p, T.voff.p, T.act.p, T.shift.p, S.minv.p, S.grad.p, S.dx.p,
                                        S.q.p, S.r.p, S.z.p, tol * tol, maxit, T.st.p, CS,
                                        pair_smoother ? S.pair_d.p : nullptr, S.minv2.p, (int)max_rows, cdim);
    };
    int n_act = 0;
    for (int32_t a : active) n_act += a != 0;
    // two scenes per SM: with nearly every scene of a large batch active the
    // global kernel's single wave (8 scenes per SM) wins, below it the shared one
    // (C5: 1024 active 123 vs 120 ms per pass; 871: 98 vs 110; 591: 70 vs 97)
    if (smem_on && smem <= kSmSceneBytes && n_act <= 960) {
      if (coarse) launch(k_pcg_scene_sm<true, kSmThreads, 2, true>);
      else launch(k_pcg_scene_sm<false, kSmThreads, 2, true>);
    } else if (coarse) {
      k_pcg_scene<true><<<NS, kCtaThreads, 0, s>>>(M, S.mask_d.p, T.voff.p, T.act.p, T.shift.p, S.minv.p, S.grad.p,
                                                   S.dx.p, S.r.p, S.z.p, S.p.p, S.q.p, tol * tol, maxit, T.st.p, CS,
                                                   pair_smoother ? S.pair_d.p : nullptr, S.minv2.p);
    } else {
      k_pcg_scene<false><<<NS, kCtaThreads, 0, s>>>(M, S.mask_d.p, T.voff.p, T.act.p, T.shift.p, S.minv.p,
                                                    S.grad.p, S.dx.p, S.r.p, S.z.p, S.p.p, S.q.p, tol * tol, maxit,
                                                    T.st.p, CS, pair_smoother ? S.pair_d.p : nullptr, S.minv2.p);
    }
    ++S.launches;
    std::vector<double> st = T.st.to_host(s);
    rel.resize(NS, 0.0);
    if (bad) bad->assign(NS, 0);
    if (coarse && bad) {  // two-level solves: reference acceptance on the recomputed residual
      T.tr.resize(2 * NS);
      k_scene_true_resid<<<NS, kSceneBlk, 0, s>>>(M, S.mask_d.p, T.voff.p, T.act.p, T.shift.p, S.dx.p, S.grad.p,
                                                   T.tr.p);
      ++S.launches;
      std::vector<unsigned long long> tr = T.tr.to_host(s);
      for (int sc = 0; sc < NS; ++sc) {
        if (!active[sc]) continue;
        const double rmax = from_ord_bits(tr[2 * sc]), bmax = from_ord_bits(tr[2 * sc + 1]);
        // indefinite, or converged on the recursive residual but not on the true one
        // (scenes that simply did not converge go to the regularized retry)
        const bool conv = st[8 * sc + 5] > 0 ? st[8 * sc + 4] <= tol * tol * st[8 * sc + 5] : true;
        (*bad)[sc] = st[8 * sc + 7] != 0 || (conv && !(rmax <= kAcceptRelInf * bmax)) ? 1 : 0;
      }
    }
    int it_max = 0;
    for (int sc = 0; sc < NS; ++sc) {
      if (!active[sc]) continue;
      if (!std::isfinite(st[8 * sc + 4])) throw StatusError(GMCP_ERR_SOLVER, "PCG diverged (non-finite residual)");
      rel[sc] = st[8 * sc + 5] > 0 ? std::sqrt(st[8 * sc + 4] / st[8 * sc + 5]) : 0.0;
      it_max = std::max(it_max, (int)st[8 * sc + 6]);
    }
    static const bool trace = std::getenv("GMCP_TRACE") != nullptr;
    if (trace) {
      std::vector<int> its;
      int failed = 0;
      for (int sc = 0; sc < NS; ++sc)
        if (active[sc]) {
          its.push_back((int)st[8 * sc + 6]);
          failed += !(rel[sc] <= tol);
        }
      std::sort(its.begin(), its.end());
      if (!its.empty())
        std::fprintf(stderr, "[gmcp pcg/cta] %zu scenes: iterations min %d median %d max %d, not converged %d\n",
                     its.size(), its.front(), its[its.size() / 2], its.back(), failed);
    }
    GMCP_CUDA(cudaGetLastError());
    return it_max;
  }
  k_init_seg<<<grid_for(nv, 256), 256, 0, s>>>(nv, T.vscene.p, T.act.p, S.grad.p, S.mask_d.p, S.minv.p, S.dx.p,
                                              S.r.p, S.z.p, S.p.p, T.dv.p);
  k_seg_sums<2><<<NS, kSceneBlk, 0, s>>>(T.voff.p, T.dv.p, nv, 0.0, T.st.p, T.act.p);
  S.launches += 2;
  const double tol2 = tol * tol;
  const int chunk = 16;
  const int lanes = nv / std::max(NS, 1) < kSmallRows ? 8 : 4;
  const int gsp = std::min(grid_for((int64_t)nv * lanes, kThreads), kBlocks);
  const int gup = std::min(grid_for((int64_t)nv, kThreads), kBlocks);
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  GMCP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < chunk; ++k) {
    double* p_old = (k & 1) ? S.w.p : S.p.p;
    double* p_new = (k & 1) ? S.p.p : S.w.p;
    if (lanes == 8)
      k_spmv_seg<8><<<gsp, kThreads, 0, s>>>(nv, M, S.mask_d.p, T.vscene.p, T.act.p, T.st.p, T.shift.p, S.z.p, p_old, p_new,
                                             S.q.p, T.dv.p);
    else
      k_spmv_seg<4><<<gsp, kThreads, 0, s>>>(nv, M, S.mask_d.p, T.vscene.p, T.act.p, T.st.p, T.shift.p, S.z.p, p_old, p_new,
                                             S.q.p, T.dv.p);
    k_seg_sums<0><<<NS, kSceneBlk, 0, s>>>(T.voff.p, T.dv.p, nv, tol2, T.st.p, T.act.p);
    k_update_seg<<<gup, kThreads, 0, s>>>(nv, T.vscene.p, T.act.p, T.st.p, p_new, S.q.p, S.dx.p, S.r.p, S.z.p,
                                          S.minv.p, T.dv.p);
    k_seg_sums<1><<<NS, kSceneBlk, 0, s>>>(T.voff.p, T.dv.p, nv, tol2, T.st.p, T.act.p);
  }
  GMCP_CUDA(cudaStreamEndCapture(s, &graph));
  GMCP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  int it = 0;
  std::vector<int32_t> act(NS);
  while (it < maxit) {
    GMCP_CUDA(cudaGraphLaunch(exec, s));
    S.launches += 4 * chunk;
    it += chunk;
    T.act.download(act.data(), NS, s);
    S.sync();
    bool any = false;
    for (int v : act) any |= v != 0;
    if (!any) break;
  }
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  std::vector<double> st = T.st.to_host(s);
  rel.resize(NS, 0.0);
  for (int sc = 0; sc < NS; ++sc) {
    if (!active[sc]) continue;  // not solved by this call
    if (!std::isfinite(st[8 * sc + 4])) throw StatusError(GMCP_ERR_SOLVER, "PCG diverged (non-finite residual)");
    rel[sc] = st[8 * sc + 5] > 0 ? std::sqrt(st[8 * sc + 4] / st[8 * sc + 5]) : 0.0;
  }
  GMCP_CUDA(cudaGetLastError());
  return it;
}

// solver.hpp:256-269 per scene (loads and bodies of that scene)
std::vector<double> derived_newton_tol_scenes(const SystemImpl& S) {
  const int NS = S.n_scenes;
  std::vector<double> scale(NS, 0.0), vol(NS, 0.0), emax(NS, 0.0);
  std::vector<long> nel(NS, 0);
  for (int64_t d = 0; d < S.n_dof; ++d) {
    const int sc = S.vscene[d / 3];
    scale[sc] = std::max(scale[sc], std::abs(S.f_ext[d]));
  }
  for (const Body& b : S.bodies) {
    const int sc = S.vscene[b.offset];
    for (double v : b.vol) vol[sc] += v;
    nel[sc] += (long)b.vol.size();
    emax[sc] = std::max(emax[sc], b.E);
  }
  std::vector<double> tol(NS);
  for (int sc = 0; sc < NS; ++sc) {
    const double h = std::cbrt(6.0 * vol[sc] / std::max<long>(nel[sc], 1));
    const double sv = std::max(scale[sc], 1e-6 * emax[sc] * h * h);
    tol[sc] = 1e-6 * std::max(sv, 1e-6);
  }
  return tol;
}

void system_solve_batched(SystemImpl& S, const gmcp_solver_settings& st, gmcp_step_callback cb, void* user,
                          gmcp_run_stats* out, std::chrono::steady_clock::time_point t_start) {
  const int NS = S.n_scenes;
  const std::vector<double> tol =
      st.newton_tol > 0 ? std::vector<double>(NS, st.newton_tol) : derived_newton_tol_scenes(S);
  int64_t n_free = 0;
  DBuf<double> eps_ref;
  setup_solve(S, n_free, eps_ref);
  const int64_t n = S.n_dof;
  cudaStream_t s = S.stream;
  DBuf<int32_t> vscene_d, active_d, take_d;
  DBuf<int64_t> voff_d;
  DBuf<double> alpha_d, el_d, mask_fixed;
  DBuf<unsigned long long> resid_d;
  vscene_d.upload(S.vscene, s);
  voff_d.upload(S.scene_voff, s);
  SegPcgTmp segT;
  segT.vscene.upload(S.vscene, s);
  segT.voff.upload(S.scene_voff, s);
  std::vector<int64_t> n_free_s(NS, 0);
  for (int64_t d = 0; d < n; ++d) n_free_s[S.vscene[d / 3]] += S.fixed[d] == 0;
  active_d.resize(NS);
  take_d.resize(NS);
  alpha_d.resize(NS);
  el_d.resize(5 * NS);
  resid_d.resize(NS);
  mask_fixed.resize(n);
  GMCP_CUDA(cudaMemcpyAsync(mask_fixed.p, S.mask_d.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  for (auto& pr : S.pairs) {  // the pairs' broadphase is scene-aware
    pr->c->vscene.upload(S.vscene, s);
    pr->c->n_scenes = NS;
  }
  const int np = (int)S.pairs.size();
  std::vector<std::vector<int64_t>> soff_h(np);
  std::vector<DBuf<int64_t>> soff_d(np);
  auto rebuild_all = [&]() {
    for (int p = 0; p < np; ++p) {
      rebuild_pair(S, *S.pairs[p], eps_ref.p);
      scene_sample_offsets(*S.pairs[p]->c, vscene_d.p, NS, soff_h[p], soff_d[p]);
    }
  };
  // re-sample only the flagged scenes of pair p (as separate Systems would):
  // sample everything, then keep the old per-scene segments elsewhere
  DBuf<uint8_t> flag_d;
  DBuf<unsigned long long> motion_d;
  std::vector<int64_t> soff_new;
  static const bool trace_rb = std::getenv("GMCP_TRACE") != nullptr;
  auto rebuild_scenes = [&](int p, const std::vector<uint8_t>& flag) {
    PairRt& pr = *S.pairs[p];
    Ctx& c = *pr.c;
    S.u_valid = false;
    double tms[6];
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](int k) {
      if (!trace_rb) return;
      S.sync();
      const auto t1 = std::chrono::steady_clock::now();
      tms[k] = std::chrono::duration<double, std::milli>(t1 - t0).count();
      t0 = t1;
    };
    snapshot_samples(c);
    lap(0);
    int64_t counts[3];
    // sample the flagged scenes only: the others keep their old segments
    c.scene_mask.upload(flag, s);
    c.use_scene_mask = true;
    try {
      run_broadphase(c, pr.params.detection_radius, counts);
      lap(1);
      run_sampler(c, eps_ref.p);
    } catch (...) {
      c.use_scene_mask = false;
      throw;
    }
    c.use_scene_mask = false;
    lap(2);
    DBuf<int64_t> tmp;
    scene_sample_offsets(c, vscene_d.p, NS, soff_new, tmp);
    std::vector<int64_t> merged;
    splice_samples(c, soff_h[p], soff_new, flag, merged);
    soff_h[p] = merged;
    soff_d[p].upload(merged, s);
    lap(3);
    c.plan.valid = false;
    build_assembly_plan(c);
    lap(4);
    if (trace_rb)
      std::fprintf(stderr, "[gmcp rebuild] snapshot %.1f broadphase %.1f sampler %.1f splice %.1f plan %.1f ms\n",
                   tms[0], tms[1], tms[2], tms[3], tms[4]);
    flag_d.upload(flag, s);
    k_sys_scene_refpos<<<grid_for(n, 256), 256, 0, s>>>(n, vscene_d.p, flag_d.p, S.x.p, pr.ref_pos.p);
    ++S.launches;
  };
  // contact energies per scene at xp (all pairs): feasible_s, energy_s, min gap
  std::vector<double> ce(NS), ce_try(NS), tmp_e(NS), tmp_mg(NS), mg(NS);
  std::vector<int64_t> tmp_bad(NS), tmp_deg(NS);
  std::vector<uint8_t> feas(NS);
  auto scene_contact = [&](double* xp, std::vector<double>& e) {
    std::fill(e.begin(), e.end(), 0.0);
    std::fill(feas.begin(), feas.end(), 1);
    std::fill(mg.begin(), mg.end(), 1.7976931348623157e308);
    for (int p = 0; p < np; ++p) {
      Ctx& c = *S.pairs[p]->c;
      double* saved = c.x_ext;
      c.x_ext = xp;
      run_scene_energy(c, xp, NS, soff_d[p].p, tmp_e.data(), tmp_bad.data(), tmp_deg.data(), tmp_mg.data());
      c.x_ext = saved;
      for (int sc = 0; sc < NS; ++sc) {
        if (tmp_deg[sc] >= 0 && (tmp_bad[sc] < 0 || tmp_deg[sc] < tmp_bad[sc]))
          throw StatusError(GMCP_ERR_DEGENERATE, "contact sample on a degenerate slave triangle");
        if (tmp_bad[sc] >= 0) feas[sc] = 0;
        e[sc] += tmp_e[sc];
        mg[sc] = std::min(mg[sc], tmp_mg[sc]);
      }
    }
  };
  std::vector<double> el(5 * NS);
  auto scene_el = [&]() {
    k_sys_scene_el<<<NS, kSceneBlk, 0, s>>>(voff_d.p, Bcsr{S.k_rowptr.p, S.k_cols.p, S.k_vals.p}, S.dx.p, S.gel.p,
                                            S.fext_d.p, S.x.p, S.rest_d.p, el_d.p);
    ++S.launches;
    el_d.download(el.data(), 5 * NS, s);
    S.sync();
  };
  std::vector<unsigned long long> resid_u(NS);
  std::vector<double> resid(NS);
  auto scene_resid = [&]() {
    k_sys_scene_resid<<<NS, kSceneBlk, 0, s>>>(voff_d.p, S.grad.p, mask_fixed.p, resid_d.p);
    ++S.launches;
    resid_d.download(resid_u.data(), NS, s);
    S.sync();
    for (int sc = 0; sc < NS; ++sc) resid[sc] = from_ord_bits(resid_u[sc]);
  };
  const int gn = grid_for(n, 256);
  S.scene_iters.assign(NS, 0);
  S.scene_stats.assign((size_t)st.load_steps * NS, gmcp_step_stats{});
  S.scene_stats_steps = 0;
  out->total_newton_iters = 0;
  out->total_rebuilds = 0;
  out->total_pcg_iters = 0;
  out->newton_tol_used = *std::min_element(tol.begin(), tol.end());
  std::vector<int32_t> active(NS), take(NS);
  std::vector<double> alpha(NS), a_pair(NS);
  std::vector<int64_t> deg(NS);
  std::vector<uint8_t> accepted(NS);
  std::vector<double> energy(NS);
  // GMCP_TRACE=1: per loop pass phase times (device-synchronized) on stderr
  static const bool trace = std::getenv("GMCP_TRACE") != nullptr;
  auto tnow = [&]() {
    if (trace) S.sync();
    return std::chrono::steady_clock::now();
  };
  auto ms_since = [](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  };
  for (int step = 1; step <= st.load_steps; ++step) {
    const double lambda = (double)step / st.load_steps;
    gmcp_step_stats ss{};
    ss.step = step;
    ss.min_gap = 1.7976931348623157e308;
    ss.energy_monotone = 1;
    const auto t_step = tnow();
    rebuild_all();
    const double ms_rb = ms_since(t_step);
    assemble(S, lambda);
    scene_el();
    scene_contact(S.x.p, ce);
    if (trace) std::fprintf(stderr, "[gmcp batched] step %d start: rebuild %.2f ms, assemble + energies %.2f ms\n", step,
                            ms_rb, ms_since(t_step) - ms_rb);
    gmcp_step_stats* sst = S.scene_stats.data() + (size_t)(step - 1) * NS;  // this step, per scene
    for (int sc = 0; sc < NS; ++sc) {
      if (!feas[sc]) throw StatusError(GMCP_ERR_SOLVER, "solve: configuration with penetrating contact sample");
      energy[sc] = el[5 * sc + 3] + ce[sc] - lambda * el[5 * sc + 4];
      ss.min_gap = std::min(ss.min_gap, mg[sc]);
      sst[sc].step = step;
      sst[sc].min_gap = mg[sc];
      sst[sc].energy_monotone = 1;
    }
    bool converged = false;
    for (int it = 0; it < st.max_newton_iters; ++it) {
      const auto t_it = std::chrono::steady_clock::now();
      const int64_t pcg_before = ss.pcg_iters;
      if (it > 0) assemble(S, lambda);
      scene_resid();
      int n_active = 0;
      for (int sc = 0; sc < NS; ++sc) {
        active[sc] = resid[sc] > tol[sc];
        n_active += active[sc];
      }
      if (n_active == 0) {
        converged = true;
        break;
      }
      // scene-segmented PCG over the active scenes; scenes that do not reach
      // the tolerance retry with their own diagonal shift (solver.hpp:352-361)
      const auto t_pcg = tnow();
      const double ms_asm = ms_since(t_it);
      S.dx.zero(s);
      std::vector<double> rel, shift(NS, 0.0);
      // two-level PCG first; a scene whose solve did not converge, lost
      // positivity, or fails the reference's acceptance test on the recomputed
      // residual (solver.hpp:349-356) retries regularized (solver.hpp:352-361):
      // two-level, then block-Jacobi alone
      std::vector<int32_t> bad;
      int pit = pcg_batched(S, segT, st.pcg_tol, st.pcg_max_iters, active, shift, rel, true, &bad);
      for (int sc = 0; sc < NS; ++sc)
        if (active[sc] && bad[sc]) rel[sc] = INFINITY;  // -> regularized retry
      std::vector<int32_t> retry(NS, 0);
      bool any_retry = false;
      for (int sc = 0; sc < NS; ++sc)
        if (active[sc] && !(rel[sc] <= st.pcg_tol)) {
          retry[sc] = 1;
          any_retry = true;
        }
      if (any_retry) {
        DBuf<double> dsum_d;
        dsum_d.resize(NS);
        k_seg_diag<<<NS, kSceneBlk, 0, s>>>(S.nv(), mats(S), S.mask_d.p, voff_d.p, dsum_d.p);
        ++S.launches;
        std::vector<double> dsum = dsum_d.to_host(s);
        for (int sc = 0; sc < NS; ++sc)
          if (retry[sc]) shift[sc] = kRegularization * dsum[sc] / (double)std::max<int64_t>(n_free_s[sc], 1);
        std::vector<int32_t> bad2;
        pit += pcg_batched(S, segT, st.pcg_tol, st.pcg_max_iters, retry, shift, rel, true, &bad2);
        std::vector<int32_t> retry2(NS, 0);
        bool any2 = false;
        for (int sc = 0; sc < NS; ++sc)
          if (retry[sc] && (bad2[sc] || !(rel[sc] <= st.pcg_tol))) {
            retry2[sc] = 1;
            any2 = true;
          }
        if (any2) {
          std::vector<double> rel3;
          pit += pcg_batched(S, segT, st.pcg_tol, st.pcg_max_iters, retry2, shift, rel3, false);
          for (int sc = 0; sc < NS; ++sc)
            if (retry2[sc]) rel[sc] = rel3[sc];
          S.coarse_fallbacks += std::count(retry2.begin(), retry2.end(), 1);
        }
        for (int sc = 0; sc < NS; ++sc)
          if (retry[sc] && !(rel[sc] <= st.pcg_tol))
            throw StatusError(GMCP_ERR_SOLVER, "scene " + std::to_string(sc) +
                                                   ": linear solve failed even with regularization; the system is "
                                                   "insufficiently constrained (unfixed rigid body modes?)");
      }
      ss.pcg_iters += pit;
      ss.newton_iters += 1;
      for (int sc = 0; sc < NS; ++sc) {
        S.scene_iters[sc] += active[sc];
        sst[sc].newton_iters += active[sc];
      }

      const double ms_pcg = ms_since(t_pcg);
      const auto t_ls = tnow();
      int n_trials = 0;
      // per-scene step size: min over pairs of min(1, filter, cap)
      for (int sc = 0; sc < NS; ++sc) alpha[sc] = active[sc] ? 1.0 : 0.0;
      for (int p = 0; p < np; ++p) {
        run_scene_alpha(*S.pairs[p]->c, NS, soff_d[p].p, voff_d.p, a_pair.data(), deg.data());
        for (int sc = 0; sc < NS; ++sc) {
          if (deg[sc] >= 0) throw StatusError(GMCP_ERR_DEGENERATE, "triangle_normal: degenerate triangle", deg[sc]);
          if (active[sc]) alpha[sc] = std::min(alpha[sc], a_pair[sc]);
        }
      }
      scene_el();  // g_el.dx, dx.K dx, f.dx per scene
      for (int sc = 0; sc < NS; ++sc) accepted[sc] = !active[sc];
      for (int ls = 0; ls < st.max_line_search; ++ls) {
        ++n_trials;
        alpha_d.upload(alpha, s);
        k_sys_scene_axpy<<<gn, 256, 0, s>>>(n, vscene_d.p, alpha_d.p, S.x.p, S.dx.p, S.xtry.p);
        ++S.launches;
        scene_contact(S.xtry.p, ce_try);
        bool all = true;
        for (int sc = 0; sc < NS; ++sc) {
          take[sc] = 0;
          if (accepted[sc]) continue;
          const double a = alpha[sc];
          const double dE =
              a * el[5 * sc] + 0.5 * a * a * el[5 * sc + 1] - lambda * a * el[5 * sc + 2] + (ce_try[sc] - ce[sc]);
          if (feas[sc] && dE < 0) {
            take[sc] = 1;
            accepted[sc] = 1;
            energy[sc] += dE;
            ce[sc] = ce_try[sc];
            ss.min_gap = std::min(ss.min_gap, mg[sc]);
            sst[sc].min_gap = std::min(sst[sc].min_gap, mg[sc]);
          } else {
            ss.backtracks += 1;
            sst[sc].backtracks += 1;
            alpha[sc] = 0.5 * a;
            all = false;
          }
        }
        take_d.upload(take, s);
        k_sys_scene_take<<<gn, 256, 0, s>>>(n, vscene_d.p, take_d.p, S.xtry.p, S.x.p);
        ++S.launches;
        if (all) break;
      }
      for (int sc = 0; sc < NS; ++sc)
        if (!accepted[sc])
          throw StatusError(GMCP_ERR_SOLVER, "load step " + std::to_string(step) + ", scene " + std::to_string(sc) +
                                                 ": line search failed to find a feasible decrease");
      const double ms_ls = ms_since(t_ls);
      const auto t_rb = tnow();
      int n_flag_total = 0;
      // re-sample the scenes whose vertices outran their frozen sampling
      // (solver.hpp:201-209, per scene)
      bool rebuild = false;
      for (int p = 0; p < np; ++p) {
        PairRt& pr = *S.pairs[p];
        const int64_t m = (int64_t)pr.motion_verts.n;
        motion_d.resize(NS);
        motion_d.zero(s);
        if (m) {
          k_sys_scene_motion<<<grid_for(m, 256), 256, 0, s>>>(m, pr.motion_verts.p, vscene_d.p, S.x.p, pr.ref_pos.p,
                                                              motion_d.p);
          ++S.launches;
        }
        std::vector<unsigned long long> mu = motion_d.to_host(s);
        std::vector<uint8_t> flag(NS, 0);
        int nflag = 0;
        for (int sc = 0; sc < NS; ++sc) {
          flag[sc] = from_ord_bits(mu[sc]) > 0.5 * pr.params.eps_max;
          nflag += flag[sc];
        }
        for (int sc = 0; sc < NS; ++sc) sst[sc].rebuilds += flag[sc];
        if (nflag) {
          rebuild_scenes(p, flag);
          rebuild = true;
        }
        n_flag_total += nflag;
      }
      if (rebuild) {
        ss.rebuilds += 1;
        assemble(S, lambda);
        scene_el();
        scene_contact(S.x.p, ce);
        for (int sc = 0; sc < NS; ++sc) {
          if (!feas[sc]) throw StatusError(GMCP_ERR_SOLVER, "solve: configuration with penetrating contact sample");
          energy[sc] = el[5 * sc + 3] + ce[sc] - lambda * el[5 * sc + 4];
        }
      }
      if (trace)
        std::fprintf(stderr,
                     "[gmcp batched] step %d it %d active %d: assemble+resid %.2f ms, pcg %.2f ms (%d it), "
                     "alpha+line search %.2f ms (%d trials), rebuild %.2f ms (%d scenes); pass %.2f ms\n",
                     step, it, n_active, ms_asm, ms_pcg, pit, ms_ls, n_trials, ms_since(t_rb), n_flag_total,
                     ms_since(t_it));
      if (S.iter_limit > 0) {  // timing mode (gmcp_system_time_newton): loop passes
        S.sync();
        S.iter_ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_it).count());
        S.iter_pcg.push_back(ss.pcg_iters - pcg_before);
        S.iter_active.push_back(n_active);
        if ((int64_t)S.iter_ms.size() >= S.iter_limit) {
          S.x.download(S.x_host.data(), n, s);
          S.sync();
          return;
        }
      }
    }
    if (!converged) {
      int worst = 0;
      for (int sc = 0; sc < NS; ++sc)
        if (resid[sc] / tol[sc] > resid[worst] / tol[worst]) worst = sc;
      out->residual = resid[worst];
      throw StatusError(GMCP_ERR_SOLVER, "load step " + std::to_string(step) + ", scene " + std::to_string(worst) +
                                             ": Newton exceeded " + std::to_string(st.max_newton_iters) +
                                             " iterations (residual " + std::to_string(resid[worst]) + ", tolerance " +
                                             std::to_string(tol[worst]) + ")");
    }
    scene_el();
    double e_tot = 0, r_max = 0;
    for (int sc = 0; sc < NS; ++sc) {
      e_tot += el[5 * sc + 3] + ce[sc] - lambda * el[5 * sc + 4];
      r_max = std::max(r_max, resid[sc]);
    }
    ss.residual = r_max;
    ss.energy = e_tot;
    for (int sc = 0; sc < NS; ++sc) {
      sst[sc].residual = resid[sc];
      sst[sc].energy = el[5 * sc + 3] + ce[sc] - lambda * el[5 * sc + 4];
    }
    S.scene_stats_steps = step;
    for (int p = 0; p < np; ++p) S.pairs[p]->scene_soff = soff_h[p];
    out->total_rebuilds += ss.rebuilds;
    out->total_pcg_iters += ss.pcg_iters;
    S.x.download(S.x_host.data(), n, s);
    S.sync();
    if (cb) cb(&ss, S.x_host.data(), n, user);
  }
  for (int64_t v : S.scene_iters) out->total_newton_iters += v;  // scene-Newton-iterations
  S.x.download(S.x_host.data(), n, s);
  S.sync();
  out->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

void system_solve(SystemImpl& S, const gmcp_solver_settings& st, gmcp_step_callback cb, void* user,
                  gmcp_run_stats* out) {
  if (S.bodies.empty()) throw StatusError(GMCP_ERR_CONFIG, "solve: no bodies");
  if (st.load_steps < 1) throw StatusError(GMCP_ERR_CONFIG, "solve: load_steps must be >= 1");
  if (st.max_newton_iters < 1) throw StatusError(GMCP_ERR_CONFIG, "solve: max_newton_iters must be >= 1");
  if (st.max_line_search < 1) throw StatusError(GMCP_ERR_CONFIG, "solve: max_line_search must be >= 1");
  const auto t_start = std::chrono::steady_clock::now();
  if (S.n_scenes > 1) {
    system_solve_batched(S, st, cb, user, out, t_start);
    return;
  }
  const double tol = st.newton_tol > 0 ? st.newton_tol : derived_newton_tol(S);
  int64_t n_free = 0;
  DBuf<double> eps_ref;  // run-start positions anchor every support radius (solver.hpp:146)
  setup_solve(S, n_free, eps_ref);
  const int64_t n = S.n_dof;
  out->total_newton_iters = 0;
  out->total_rebuilds = 0;
  out->total_pcg_iters = 0;
  out->newton_tol_used = tol;
  for (int step = 1; step <= st.load_steps; ++step) {
    const double lambda = (double)step / st.load_steps;
    S.load_step = step;
    gmcp_step_stats ss{};
    ss.step = step;
    ss.min_gap = 1.7976931348623157e308;
    ss.energy_monotone = 1;
    for (auto& pr : S.pairs) rebuild_pair(S, *pr, eps_ref.p);
    // total energy at x (solver.hpp:154): elastic via K u, contact, external work
    double resid = assemble(S, lambda);
    double e_el, work;
    elastic_terms(S, e_el, work);
    CE ce = contact_energy_at(S, S.x.p);
    if (!ce.feasible) throw StatusError(GMCP_ERR_SOLVER, "solve: configuration with penetrating contact sample");
    double energy = e_el + ce.energy - lambda * work;
    ss.min_gap = std::min(ss.min_gap, ce.min_gap);
    bool converged = false;
    static const bool trace = std::getenv("GMCP_TRACE") != nullptr;
    auto tp = [&]() {
      if (trace) S.sync();
      return std::chrono::steady_clock::now();
    };
    auto dms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    for (int it = 0; it < st.max_newton_iters; ++it) {
      const auto t_it = std::chrono::steady_clock::now();
      const int64_t pcg_before = ss.pcg_iters;
      if (it > 0) resid = assemble(S, lambda);
      const auto t_as = tp();
      if (resid <= tol) {
        converged = true;
        break;
      }
      double rel;
      int pit = pcg(S, st.pcg_tol, st.pcg_max_iters, &rel);
      // accepted as the reference accepts its LDL^T solve (solver.hpp:349-356):
      // converged, and the recomputed residual within 1e-6 of the rhs (inf-norm)
      if (!(rel <= st.pcg_tol) || !(S.last_true_relinf <= kAcceptRelInf)) {
        // solver.hpp:352-361: not solved (singular: an unconstrained rigid mode
        // before contact engages) -> retry with the diagonal shifted by
        // regularization (1e-8) x the mean free diagonal entry.
        k_diag_sum<<<kBlocks, kThreads, 0, S.stream>>>(S.nv(), mats(S), S.mask_d.p, S.scal.p + 10, S.slot(4));
        ++S.launches;
        double dsum;
        GMCP_CUDA(cudaMemcpyAsync(&dsum, S.scal.p + 10, sizeof dsum, cudaMemcpyDeviceToHost, S.stream));
        S.sync();
        const double shift = kRegularization * dsum / (double)n_free;
        pit += pcg(S, st.pcg_tol, st.pcg_max_iters, &rel, shift);
        if ((!(rel <= st.pcg_tol) || !(S.last_true_relinf <= kAcceptRelInf)) && S.cs.enabled) {
          // last resort: the regularized solve with the smoother alone
          S.cs.enabled = false;
          try {
            pit += pcg(S, st.pcg_tol, st.pcg_max_iters, &rel, shift);
          } catch (...) {
            S.cs.enabled = true;
            throw;
          }
          S.cs.enabled = true;
          ++S.coarse_fallbacks;
        }
        if (!(rel <= st.pcg_tol) || !(S.last_true_relinf <= kAcceptRelInf)) {
          out->residual = resid;
          throw StatusError(GMCP_ERR_SOLVER,
                            "linear solve failed even with regularization; the system is insufficiently "
                            "constrained (unfixed rigid body modes?)");
        }
      }
      record_accepted_solve(S);
      ss.pcg_iters += pit;
      ss.newton_iters += 1;
      const auto t_pcg = tp();
      double alpha = 1.0;
      for (auto& pr : S.pairs) {
        alpha = std::min(alpha, run_step_filter(*pr->c));
        alpha = std::min(alpha, run_displacement_cap(*pr->c));
      }
      // line search on the exact energy decrease:
      // dE(a) = a g_el.dx + a^2/2 dx.K dx - lambda a f.dx + Psi(x + a dx) - Psi(x)
      k_ls_coeffs<<<kBlocks, kThreads, 0, S.stream>>>(S.nv(), Bcsr{S.k_rowptr.p, S.k_cols.p, S.k_vals.p}, S.dx.p,
                                                      S.gel.p, S.fext_d.p, S.lsco.p, S.slot(3));
      ++S.launches;
      double co[3];
      GMCP_CUDA(cudaMemcpyAsync(co, S.lsco.p, sizeof co, cudaMemcpyDeviceToHost, S.stream));
      S.sync();
      bool accepted = false;
      for (int ls = 0; ls < st.max_line_search; ++ls) {
        k_axpy_to<<<grid_for(n, 256), 256, 0, S.stream>>>(n, S.x.p, alpha, S.dx.p, S.xtry.p);
        ++S.launches;
        const CE t = contact_energy_at(S, S.xtry.p);
        if (t.feasible) {
          const double dE = alpha * co[0] + 0.5 * alpha * alpha * co[1] - lambda * alpha * co[2] + (t.energy - ce.energy);
          if (dE < 0) {
            GMCP_CUDA(cudaMemcpyAsync(S.x.p, S.xtry.p, n * sizeof(double), cudaMemcpyDeviceToDevice, S.stream));
            energy += dE;
            ce = t;
            ss.min_gap = std::min(ss.min_gap, t.min_gap);
            accepted = true;
            break;
          }
        }
        ss.backtracks += 1;
        alpha *= 0.5;
      }
      if (!accepted) {
        out->residual = resid;
        throw StatusError(GMCP_ERR_SOLVER, "load step " + std::to_string(step) +
                                               ": line search failed to find a feasible decrease");
      }
      // re-sample pairs whose vertices outran the frozen sampling (solver.hpp:201-209)
      bool rebuilt = false;
      for (auto& pr : S.pairs) {
        const int64_t m = (int64_t)pr->motion_verts.n;
        GMCP_CUDA(cudaMemsetAsync(S.redu.p + 1, 0, sizeof(unsigned long long), S.stream));
        if (m) {
          k_motion<<<grid_for(m, 256), 256, 0, S.stream>>>(m, pr->motion_verts.p, S.x.p, pr->ref_pos.p, S.redu.p + 1);
          ++S.launches;
        }
        unsigned long long u;
        GMCP_CUDA(cudaMemcpyAsync(&u, S.redu.p + 1, sizeof u, cudaMemcpyDeviceToHost, S.stream));
        S.sync();
        if (from_ord_bits(u) > 0.5 * pr->params.eps_max) {
          rebuild_pair(S, *pr, eps_ref.p);
          rebuilt = true;
          ss.rebuilds += 1;
        }
      }
      if (rebuilt) {
        resid = assemble(S, lambda);
        elastic_terms(S, e_el, work);
        ce = contact_energy_at(S, S.x.p);
        if (!ce.feasible) throw StatusError(GMCP_ERR_SOLVER, "solve: configuration with penetrating contact sample");
        energy = e_el + ce.energy - lambda * work;
      }
      if (trace) {
        const auto t_end = tp();
        std::fprintf(stderr, "[gmcp] newton %d: assemble %.3f ms, linear solve %.3f ms (%d PCG), line search + "
                             "rebuild %.3f ms\n", it, dms(t_it, t_as), dms(t_as, t_pcg), pit, dms(t_pcg, t_end));
      }
      if (S.iter_limit > 0) {  // timing mode (gmcp_system_time_newton)
        S.sync();
        S.iter_ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_it).count());
        S.iter_pcg.push_back(ss.pcg_iters - pcg_before);
        if ((int64_t)S.iter_ms.size() >= S.iter_limit) {
          S.x.download(S.x_host.data(), n, S.stream);
          S.sync();
          return;
        }
      }
    }
    if (!converged) {
      out->residual = resid;
      throw StatusError(GMCP_ERR_SOLVER, "load step " + std::to_string(step) + ": Newton exceeded " +
                                             std::to_string(st.max_newton_iters) + " iterations");
    }
    // report the energy recomputed at the converged state
    elastic_terms(S, e_el, work);
    energy = e_el + ce.energy - lambda * work;
    ss.residual = resid;
    ss.energy = energy;
    out->total_newton_iters += ss.newton_iters;
    out->total_rebuilds += ss.rebuilds;
    out->total_pcg_iters += ss.pcg_iters;
    S.x.download(S.x_host.data(), n, S.stream);
    S.sync();
    if (cb) cb(&ss, S.x_host.data(), n, user);
  }
  S.x.download(S.x_host.data(), n, S.stream);
  S.sync();
  out->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

// Standalone linear solve (gmcp_system_linear_solve): the reference's
// solve_descent (solver.hpp:325-375) on a caller-given Newton matrix. The
// caller's AoS BCSR is the operand (Dirichlet dofs masked: P H P + I - P, rhs
// masked), the smoother pairs come from its values, and the two-level space
// from optional positions (one body). The ladder is the Newton loop's:
// PCG; if not accepted (converged and ||H dx - rhs||_inf <= 1e-6 ||rhs||_inf,
// solver.hpp:349-356), regularized by 1e-8 x the mean free diagonal entry
// (solver.hpp:352-361); last, regularized with the smoother alone.
struct LinearSolveOut {
  int32_t iterations = 0, regularized = 0;
  double relinf = 0;
};
LinearSolveOut linear_solve(SystemImpl& S, int64_t nv, const int32_t* rowptr, const int32_t* cols, const double* vals,
                            const uint8_t* fixed, const double* positions, const double* rhs, double tol, int maxit,
                            double* dx) {
  if (!S.bodies.empty() || !S.pairs.empty())
    throw StatusError(GMCP_ERR_CONFIG, "linear_solve: use a system handle without bodies or contact pairs");
  if (nv <= 0 || !rowptr || !cols || !vals || !rhs || !dx) throw StatusError(GMCP_ERR_ARG, "linear_solve: null input");
  if (!(tol > 0) || maxit < 1) throw StatusError(GMCP_ERR_ARG, "linear_solve: tol > 0 and max_iters >= 1");
  const int64_t n = 3 * nv, nnzb = rowptr[nv];
  if (rowptr[0] != 0 || nnzb < 0) throw StatusError(GMCP_ERR_ARG, "linear_solve: bad row pointers");
  for (int64_t v = 0; v < nv; ++v) {
    if (rowptr[v + 1] < rowptr[v]) throw StatusError(GMCP_ERR_ARG, "linear_solve: bad row pointers");
    for (int32_t k = rowptr[v]; k < rowptr[v + 1]; ++k)
      if (cols[k] < 0 || cols[k] >= nv || (k > rowptr[v] && cols[k] <= cols[k - 1]))
        throw StatusError(GMCP_ERR_ARG, "linear_solve: columns must be in range and ascending per row");
  }
  std::vector<int32_t> rp(rowptr, rowptr + nv + 1), cl(cols, cols + nnzb);
  std::vector<double> vl(vals, vals + 9 * nnzb);
  S.n_dof = n;
  S.k_rowptr.upload(rp, S.stream);
  S.k_cols.upload(cl, S.stream);
  S.k_vals.upload(vl, S.stream);
  S.el_nnzb = nnzb;
  S.el_built = true;
  build_pairing(S, (int)nv, rp.data(), cl.data(), vl.data());
  S.fixed.assign(n, 0);
  int64_t n_free = 0;
  std::vector<double> mask(n);
  for (int64_t d = 0; d < n; ++d) {
    S.fixed[d] = fixed ? (fixed[d] ? 1 : 0) : 0;
    mask[d] = S.fixed[d] ? 0.0 : 1.0;
    n_free += S.fixed[d] == 0;
  }
  if (n_free == 0) throw StatusError(GMCP_ERR_CONFIG, "linear_solve: no free degrees of freedom");
  for (auto* b : {&S.x, &S.dx, &S.grad, &S.r, &S.z, &S.p, &S.q, &S.w, &S.rt, &S.xacc}) b->resize(n);
  S.minv.resize(3 * n);
  S.scal.resize(16);
  S.parts.resize(kBlocks * 4);
  S.counter.resize(16);
  S.counter.zero(S.stream);
  S.redu.resize(8);
  S.mask_d.upload(mask, S.stream);
  std::vector<double> g(n);
  for (int64_t d = 0; d < n; ++d) g[d] = -rhs[d];  // PCG's rhs is -mask .* grad
  S.grad.upload(g, S.stream);
  if (S.pcg_exec) {
    cudaGraphExecDestroy(S.pcg_exec);
    S.pcg_exec = nullptr;
  }
  S.cs.enabled = false;
  if (positions) {  // the two-level space over one body spanning every vertex
    Body b;
    b.verts.assign(positions, positions + n);
    b.offset = 0;
    b.nv = (int32_t)nv;
    S.bodies.push_back(std::move(b));
    S.rest.assign(positions, positions + n);  // aggregate centroids and offsets
    try {
      build_coarse(S, mask);
    } catch (...) {
      S.bodies.clear();
      S.rest.clear();
      throw;
    }
    S.bodies.clear();
    S.rest.clear();
  }
  S.cs.have_inv = false;
  S.load_step += 1;  // a fresh coarse inverse for this operand
  LinearSolveOut out;
  double rel = 0;
  out.iterations = pcg(S, tol, maxit, &rel);
  if (!(rel <= tol) || !(S.last_true_relinf <= kAcceptRelInf)) {
    k_diag_sum<<<kBlocks, kThreads, 0, S.stream>>>(S.nv(), mats(S), S.mask_d.p, S.scal.p + 10, S.slot(4));
    double dsum = 0;
    GMCP_CUDA(cudaMemcpyAsync(&dsum, S.scal.p + 10, sizeof dsum, cudaMemcpyDeviceToHost, S.stream));
    S.sync();
    const double shift = kRegularization * dsum / (double)n_free;
    out.regularized = 1;
    out.iterations += pcg(S, tol, maxit, &rel, shift);
    if ((!(rel <= tol) || !(S.last_true_relinf <= kAcceptRelInf)) && S.cs.enabled) {
      S.cs.enabled = false;
      out.iterations += pcg(S, tol, maxit, &rel, shift);
      S.cs.enabled = true;
    }
    if (!(rel <= tol) || !(S.last_true_relinf <= kAcceptRelInf))
      throw StatusError(GMCP_ERR_SOLVER, "linear solve failed even with regularization; the system is insufficiently "
                                         "constrained (unfixed rigid body modes?)");
  }
  record_accepted_solve(S);
  out.relinf = S.last_true_relinf;
  GMCP_CUDA(cudaMemcpyAsync(dx, S.dx.p, n * sizeof(double), cudaMemcpyDeviceToHost, S.stream));
  S.sync();
  return out;
}

}  // namespace gmcp_b200

// ===========================================================================
// C-ABI (include/gmcp_solver.h)

using namespace gmcp_b200;

struct gmcp_system {
  SystemImpl s;
};

namespace {
thread_local std::string g_serr;
// every system entry binds the system's device and CUB scratch to the thread
template <class F>
int sguard(gmcp_system* sys, F&& f) {
  try {
    if (!sys) throw StatusError(GMCP_ERR_ARG, "null gmcp_system");
    const DeviceBind bind_(sys->s.device, &sys->s.cub);
    return f();
  } catch (const StatusError& e) {
    g_serr = e.what();
    return e.code;
  } catch (const CudaError& e) {
    g_serr = e.what();
    return GMCP_ERR_CUDA;
  } catch (const std::exception& e) {
    g_serr = e.what();
    return GMCP_ERR_ARG;
  }
}
}  // namespace

extern "C" {

const char* gmcp_system_last_error(void) { return g_serr.c_str(); }

// Grows the per-dof host arrays to n_dof (new entries: positions at rest,
// no load, free); O(new dofs), so adding many bodies stays linear.
static void sized_host(SystemImpl& S) {
  const size_t n = (size_t)S.n_dof, o = S.x_host.size();
  if (o == n) return;
  S.x_host.resize(n);
  S.dirichlet.resize(n);
  for (size_t d = o; d < n; ++d) S.x_host[d] = S.dirichlet[d] = S.rest[d];
  S.f_ext.resize(n, 0.0);
  S.fixed.resize(n, 0);
}

int gmcp_system_create(int device, gmcp_system** out) {
  try {
    int nd = 0;
    GMCP_CUDA(cudaGetDeviceCount(&nd));
    if (device < 0 || device >= nd) throw StatusError(GMCP_ERR_CUDA, "no such CUDA device");
    auto* s = new gmcp_system;
    s->s.device = device;
    const DeviceBind bind_(device, &s->s.cub);
    GMCP_CUDA(cudaStreamCreateWithFlags(&s->s.stream, cudaStreamNonBlocking));
    if (const char* e = std::getenv("GMCP_PAIR_JACOBI")) s->s.use_pair = std::atoi(e) != 0;
    if (const char* e = std::getenv("GMCP_HALF_SPMV")) s->s.use_half = std::atoi(e) != 0;
    if (const char* e = std::getenv("GMCP_COARSE")) s->s.use_coarse = std::atoi(e) != 0;
    if (const char* e = std::getenv("GMCP_COARSE_AGGS")) s->s.coarse_aggs = std::min(512, std::max(1, std::atoi(e)));
    if (const char* e = std::getenv("GMCP_COARSE_REFRESH")) s->s.coarse_refresh_always = std::atoi(e) != 0;
    if (const char* e = std::getenv("GMCP_COARSE_DROP")) s->s.coarse_drop = std::atof(e);
    if (const char* e = std::getenv("GMCP_COARSE_SCENE_AGGS"))
      s->s.coarse_scene_aggs = std::min(64, std::max(1, std::atoi(e)));
    *out = s;
    return GMCP_OK;
  } catch (const StatusError& e) {
    g_serr = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_serr = e.what();
    return GMCP_ERR_CUDA;
  }
}

void gmcp_system_destroy(gmcp_system* s) {
  if (!s) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(s->s.device);
  cudaStreamSynchronize(s->s.stream);
  cudaStream_t st = s->s.stream;
  for (auto& pr : s->s.pairs) pr->c->stream = nullptr;
  if (s->s.pcg_exec) cudaGraphExecDestroy(s->s.pcg_exec);
  if (s->s.ev0) cudaEventDestroy(s->s.ev0);
  if (s->s.ev1) cudaEventDestroy(s->s.ev1);
  delete s;
  cudaStreamDestroy(st);
  cudaSetDevice(prev);
}

int gmcp_system_add_body(gmcp_system* sys, const double* verts, int64_t nv, const int32_t* tets, int64_t nt, double E,
                         double nu, int32_t* vertex_offset) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    SystemImpl& S = sys->s;
    Body b;
    make_material(E, nu, b.lambda, b.mu);
    b.E = E;
    b.nu = nu;
    b.verts.assign(verts, verts + 3 * nv);
    b.tets.assign(tets, tets + 4 * nt);
    for (int64_t i = 0; i < 4 * nt; ++i)
      if (b.tets[i] < 0 || b.tets[i] >= nv) throw StatusError(GMCP_ERR_ARG, "tet vertex id out of range");
    b.offset = (int32_t)(S.n_dof / 3);
    b.nv = (int32_t)nv;
    build_operators(b);
    S.rest.insert(S.rest.end(), verts, verts + 3 * nv);
    S.n_dof = (int64_t)S.rest.size();  // per-dof host arrays grow lazily (sized_host)
    if (vertex_offset) *vertex_offset = b.offset;
    S.bodies.push_back(std::move(b));
    S.el_built = false;
    return GMCP_OK;
  });
}

int gmcp_system_set_vertex_scenes(gmcp_system* sys, const int32_t* scene, int64_t n_vertices) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    if (!sys) throw StatusError(GMCP_ERR_ARG, "null system");
    SystemImpl& S = sys->s;
    S.el_built = false;  // the vertex pairing / coarse space depend on the scene layout
    if (!scene) {
      S.vscene.clear();
      S.scene_voff.clear();
      S.n_scenes = 1;
      return GMCP_OK;
    }
    if (n_vertices != S.n_dof / 3) throw StatusError(GMCP_ERR_ARG, "vertex scenes: one id per system vertex");
    std::vector<int64_t> voff{0};
    for (int64_t v = 0; v < n_vertices; ++v) {
      if (scene[v] < 0 || (v > 0 && scene[v] < scene[v - 1]) || (v == 0 && scene[0] != 0) ||
          (v > 0 && scene[v] > scene[v - 1] + 1))
        throw StatusError(GMCP_ERR_ARG, "vertex scenes: ids must be 0, 1, ... in contiguous vertex ranges");
      if (v > 0 && scene[v] != scene[v - 1]) voff.push_back(v);
    }
    voff.push_back(n_vertices);
    for (const Body& b : S.bodies)
      if (scene[b.offset] != scene[b.offset + b.nv - 1])
        throw StatusError(GMCP_ERR_ARG, "vertex scenes: a body spans two scenes");
    S.vscene.assign(scene, scene + n_vertices);
    S.scene_voff = voff;
    S.n_scenes = (int32_t)voff.size() - 1;
    return GMCP_OK;
  });
}

int gmcp_system_timed_active_scenes(const gmcp_system* sys, int64_t* out, int32_t n) {
  if (!sys || !out) return GMCP_ERR_ARG;
  for (int32_t k = 0; k < n && k < (int32_t)sys->s.iter_active.size(); ++k) out[k] = sys->s.iter_active[k];
  return GMCP_OK;
}

int gmcp_system_scene_newton_iters(const gmcp_system* sys, int64_t* out) {
  if (!sys || !out) return GMCP_ERR_ARG;
  for (size_t k = 0; k < sys->s.scene_iters.size(); ++k) out[k] = sys->s.scene_iters[k];
  return GMCP_OK;
}

int gmcp_system_fix_dofs(gmcp_system* sys, int64_t n, const int64_t* dofs, const double* targets) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    SystemImpl& S = sys->s;
    sized_host(S);
    for (int64_t i = 0; i < n; ++i) {
      if (dofs[i] < 0 || dofs[i] >= S.n_dof) throw StatusError(GMCP_ERR_ARG, "dof out of range");
      S.fixed[dofs[i]] = 1;
      S.dirichlet[dofs[i]] = targets[i];
    }
    return GMCP_OK;
  });
}

int gmcp_system_set_external_force(gmcp_system* sys, const double* f, int64_t n_dof) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    SystemImpl& S = sys->s;
    sized_host(S);
    if (n_dof != S.n_dof) throw StatusError(GMCP_ERR_ARG, "f_ext size mismatch");
    S.f_ext.assign(f, f + n_dof);
    return GMCP_OK;
  });
}

int gmcp_system_add_contact_pair(gmcp_system* sys, const gmcp_surface* slave, const gmcp_surface* master,
                                 const gmcp_barrier_params* resolved, int32_t* pair_id) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    SystemImpl& S = sys->s;
    if ((int)S.pairs.size() >= kMaxPairs) throw StatusError(GMCP_ERR_CONFIG, "too many contact pairs");
    auto pr = std::make_unique<PairRt>();
    pr->c = std::make_unique<Ctx>();
    Ctx& c = *pr->c;
    c.device = S.device;
    c.stream = S.stream;
    c.params = *resolved;
    c.have_params = true;
    pr->params = *resolved;
    auto up = [&](DevSurface& d, const gmcp_surface* s) {
      d.n_tris = s->n_tris;
      d.n_edges = s->n_edges;
      d.n_verts = s->n_verts;
      d.h_tris.assign(s->tris, s->tris + 3 * (size_t)s->n_tris);
      d.h_tri_edges.assign(s->tri_edges, s->tri_edges + 3 * (size_t)s->n_tris);
      d.h_edges.assign(s->edges, s->edges + 2 * (size_t)s->n_edges);
      d.h_verts.assign(s->verts, s->verts + s->n_verts);
      d.tris.upload(d.h_tris, S.stream);
      d.tri_edges.upload(d.h_tri_edges, S.stream);
      d.edges.upload(d.h_edges, S.stream);
      d.verts.upload(d.h_verts, S.stream);
    };
    up(c.slave, slave);
    up(c.master, master);
    std::vector<int32_t> mv(c.slave.h_verts);
    mv.insert(mv.end(), c.master.h_verts.begin(), c.master.h_verts.end());
    pr->motion_verts.upload(mv, S.stream);
    S.sync();
    if (pair_id) *pair_id = (int32_t)S.pairs.size();
    S.pairs.push_back(std::move(pr));
    return GMCP_OK;
  });
}

int gmcp_system_solve(gmcp_system* sys, const gmcp_solver_settings* st, gmcp_step_callback cb, void* user,
                      gmcp_run_stats* out) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    sized_host(sys->s);
    system_solve(sys->s, *st, cb, user, out);
    return GMCP_OK;
  });
}

int gmcp_system_time_newton(gmcp_system* sys, const gmcp_solver_settings* st, int32_t n_iters, double* ms_per_iter,
                            int64_t* pcg_per_iter, int32_t* n_done) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    SystemImpl& S = sys->s;
    sized_host(S);
    if (n_iters < 1) throw StatusError(GMCP_ERR_ARG, "n_iters must be positive");
    S.iter_limit = n_iters;
    S.pcg_ev_ms = 0;
    S.pcg_ev_iters = 0;
    S.iter_ms.clear();
    S.iter_pcg.clear();
    S.iter_active.clear();
    gmcp_run_stats out{};
    try {
      system_solve(S, *st, nullptr, nullptr, &out);
    } catch (...) {
      S.iter_limit = 0;
      throw;
    }
    S.iter_limit = 0;
    *n_done = (int32_t)S.iter_ms.size();
    for (size_t i = 0; i < S.iter_ms.size(); ++i) {
      ms_per_iter[i] = S.iter_ms[i];
      pcg_per_iter[i] = S.iter_pcg[i];
    }
    return GMCP_OK;
  });
}

int gmcp_system_pcg_stats(const gmcp_system* sys, double* ev_ms, int64_t* ev_iters, int64_t* n_rows,
                          int64_t* nnzb) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    const SystemImpl& S = sys->s;
    *ev_ms = S.pcg_ev_ms;
    *ev_iters = S.pcg_ev_iters;
    *n_rows = S.nv();
    *nnzb = S.u_valid ? S.u_nnzb : 0;
    return GMCP_OK;
  });
}

int gmcp_system_positions(gmcp_system* sys, double* x, int64_t n_dof) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    if (n_dof != sys->s.n_dof) throw StatusError(GMCP_ERR_ARG, "size mismatch");
    sized_host(sys->s);
    std::copy(sys->s.x_host.begin(), sys->s.x_host.end(), x);
    return GMCP_OK;
  });
}

int gmcp_system_set_positions(gmcp_system* sys, const double* x, int64_t n_dof) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    if (n_dof != sys->s.n_dof) throw StatusError(GMCP_ERR_ARG, "size mismatch");
    sized_host(sys->s);
    sys->s.x_host.assign(x, x + n_dof);
    return GMCP_OK;
  });
}

int64_t gmcp_system_num_samples(gmcp_system* sys, int32_t pair) {
  if (!sys || pair < 0 || pair >= (int)sys->s.pairs.size()) return -1;
  return sys->s.pairs[pair]->c->ns;
}

int gmcp_system_pair_force_summary(gmcp_system* sys, int32_t pair, double* out12) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    SystemImpl& S = sys->s;
    if (pair < 0 || pair >= (int)S.pairs.size()) throw StatusError(GMCP_ERR_ARG, "no such pair");
    Ctx& c = *S.pairs[pair]->c;
    run_force_summary(c, out12);
    return GMCP_OK;
  });
}

int gmcp_system_pair_pressure(gmcp_system* sys, int32_t pair, int64_t* n, gmcp_pressure_record* out) {
  return sguard(const_cast<gmcp_system*>(sys), [&] {
    SystemImpl& S = sys->s;
    if (pair < 0 || pair >= (int)S.pairs.size()) throw StatusError(GMCP_ERR_ARG, "no such pair");
    Ctx& c = *S.pairs[pair]->c;
    *n = (int64_t)c.face_idx.n;
    if (out) run_pressure(c, out);
    return GMCP_OK;
  });
}

int gmcp_system_linear_stats(gmcp_system* sys, int32_t reset, double* max_rel2, double* max_relinf,
                             int64_t* n_solves) {
  return sguard(sys, [&] {
    SystemImpl& S = sys->s;
    if (max_rel2) *max_rel2 = S.true_rel2_max;
    if (max_relinf) *max_relinf = S.true_relinf_max;
    if (n_solves) *n_solves = S.n_linear_solves;
    if (reset) {
      S.true_rel2_max = S.true_relinf_max = 0;
      S.n_linear_solves = 0;
    }
    return GMCP_OK;
  });
}

int gmcp_system_capture_linear_system(gmcp_system* sys, int32_t on) {
  return sguard(sys, [&] {
    sys->s.capture = on != 0;
    return GMCP_OK;
  });
}

int gmcp_system_captured_linear_system(gmcp_system* sys, int64_t* nnzb, int32_t* rowptr, int32_t* cols, double* vals,
                                       double* mask, double* grad, double* dx, double* shift) {
  return sguard(sys, [&] {
    const SystemImpl& S = sys->s;
    if (S.cap_rowptr.empty()) throw StatusError(GMCP_ERR_ARG, "no captured linear system");
    *nnzb = (int64_t)S.cap_cols.size();
    if (rowptr) std::copy(S.cap_rowptr.begin(), S.cap_rowptr.end(), rowptr);
    if (cols) std::copy(S.cap_cols.begin(), S.cap_cols.end(), cols);
    if (vals) std::copy(S.cap_vals.begin(), S.cap_vals.end(), vals);
    if (mask) std::copy(S.cap_mask.begin(), S.cap_mask.end(), mask);
    if (grad) std::copy(S.cap_grad.begin(), S.cap_grad.end(), grad);
    if (dx) std::copy(S.cap_dx.begin(), S.cap_dx.end(), dx);
    if (shift) *shift = S.cap_shift;
    return GMCP_OK;
  });
}

int gmcp_system_precond_info(gmcp_system* sys, int32_t* pair_jacobi, int32_t* coarse, int32_t* n_aggregates,
                             int32_t* n_coarse_padded) {
  return sguard(sys, [&] {
    const SystemImpl& S = sys->s;
    *pair_jacobi = S.has_pairs ? 1 : 0;
    *coarse = S.cs.enabled ? 1 : 0;
    *n_aggregates = S.cs.enabled ? S.cs.n_agg : 0;
    *n_coarse_padded = S.cs.enabled ? S.cs.n_pad : 0;
    return GMCP_OK;
  });
}

int gmcp_system_linear_solve(gmcp_system* sys, int64_t n_vertices, const int32_t* rowptr, const int32_t* cols,
                             const double* vals, const uint8_t* fixed, const double* positions, const double* rhs,
                             double pcg_tol, int32_t max_iters, double* dx, int32_t* iterations,
                             double* residual_inf_rel, int32_t* regularized) {
  return sguard(sys, [&] {
    if (!sys) throw StatusError(GMCP_ERR_ARG, "null system");
    const LinearSolveOut o = linear_solve(sys->s, n_vertices, rowptr, cols, vals, fixed, positions, rhs, pcg_tol,
                                          max_iters, dx);
    if (iterations) *iterations = o.iterations;
    if (residual_inf_rel) *residual_inf_rel = o.relinf;
    if (regularized) *regularized = o.regularized;
    return GMCP_OK;
  });
}

int gmcp_system_operand_info(gmcp_system* sys, int64_t* stored_blocks) {
  return sguard(sys, [&] {
    const SystemImpl& S = sys->s;
    *stored_blocks = S.u_half_ok ? S.u_hn : 0;
    return GMCP_OK;
  });
}

int gmcp_system_scene_step_stats(gmcp_system* sys, int32_t* n_steps, gmcp_step_stats* out) {
  return sguard(sys, [&] {
    const SystemImpl& S = sys->s;
    *n_steps = S.scene_stats_steps;
    if (out)
      std::copy(S.scene_stats.begin(), S.scene_stats.begin() + (size_t)S.scene_stats_steps * S.n_scenes, out);
    return GMCP_OK;
  });
}

int gmcp_system_pair_scene_offsets(gmcp_system* sys, int32_t pair, int64_t* soff) {
  return sguard(sys, [&] {
    const SystemImpl& S = sys->s;
    if (pair < 0 || pair >= (int)S.pairs.size()) throw StatusError(GMCP_ERR_ARG, "no such pair");
    const auto& v = S.pairs[pair]->scene_soff;
    if (v.size() != (size_t)S.n_scenes + 1) throw StatusError(GMCP_ERR_ARG, "no batched solve has completed");
    std::copy(v.begin(), v.end(), soff);
    return GMCP_OK;
  });
}

int64_t gmcp_system_launch_count(const gmcp_system* sys) {
  if (!sys) return 0;
  int64_t n = sys->s.launches;
  for (auto& pr : sys->s.pairs) n += pr->c->launches;
  return n;
}

}  // extern "C"
