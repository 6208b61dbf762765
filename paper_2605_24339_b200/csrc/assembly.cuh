// Contact assembly kernels (included once, by contact_eval.cu).
//
//  K7 k_run_partials  one warp per slave run (consecutive samples sharing a
//                      slave triangle), no block-level synchronisation. Lanes
//                      own samples: gap, barrier and the in-plane vector r go
//                      into a per-warp staging tile, the run's moments are one
//                      Gram product on the FP64 tensor cores, and the warp
//                      finalizes the run's blocks into its partial.
//  K8 k_gather         one thread per BCSR block: sums the block's
//                      contributions from the run partials in ascending run
//                      order (listed by the plan); one thread per vertex row
//                      does the same for the gradient.
//
// Moment form. Within a run (one slave triangle) n, e1, e2 are shared and the
// slave gap gradients are dg_i = -b_i n + T_i(r) with T_0(v) = v x (e2-e1),
// T_1(v) = e2 x v, T_2(v) = v x e1 (contact_energy.hpp:67-70), linear in the
// per-sample r = (d - g n)/|c|. Hence the reference's per-sample Gauss-Newton
// entries h (dg_v[a] dg_w[c]) (contact_energy.hpp:161-176) sum over a run to
//   SS(i,j) = Mbb_ij n n^T - n T_j(Mbr_i)^T - T_i(Mbr_j) n^T + T_i Mrr T_j^T
//   SM(i,m) = a_{m,i} n^T,  a_{m,i} = -Hwb_{m,i} n + T_i(Hwr_m)
//   MM(m,l) = c_{ml} (n n^T)
// with moments Mbb = sum h b b^T, Mbr = sum h b r^T, Mrr = sum h r r^T,
// Hwb_m = sum h w_m b, Hwr_m = sum h w_m r, c_ml = sum h w_m w_l, and the
// gradient g_i = -Fb_i n + T_i(Fr), g_m = s_m n (Fb = sum f b, Fr = sum f r,
// s_m = sum f w_m). Upper SS blocks are stored once and mirrored, and every
// mirror entry is the same product in the same order, so the assembled
// matrix is exactly symmetric (test_contact.cpp:125).
#pragma once

#include "ctx.hpp"
#include "kin.cuh"
#include "reduce.cuh"
#include "partial_layout.cuh"

namespace gmcp_b200 {
namespace {

// ---------------------------------------------------------------------------
// K0: derived per-sample fields

__global__ void k_derive(int64_t n, const int8_t* __restrict__ type, const double* __restrict__ beta_m,
                         const double* __restrict__ eta, const double* __restrict__ weight,
                         const double* __restrict__ gamma, double kf, double ke, double kp,
                         double* __restrict__ wm, double* __restrict__ coef) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int8_t t = type[i];
    const double kappa = t == GMCP_FACE ? kf : (t == GMCP_EDGE ? ke : kp);  // contact_energy.hpp:75-84
    coef[i] = kappa * weight[i] * gamma[i];
    if (t == GMCP_FACE) {
      wm[3 * i] = beta_m[3 * i];
      wm[3 * i + 1] = beta_m[3 * i + 1];
      wm[3 * i + 2] = beta_m[3 * i + 2];
    } else if (t == GMCP_EDGE) {  // contact_energy.hpp:47-49
      wm[3 * i] = 1.0 - eta[i];
      wm[3 * i + 1] = eta[i];
      wm[3 * i + 2] = 0;
    } else {
      wm[3 * i] = 1;
      wm[3 * i + 1] = 0;
      wm[3 * i + 2] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// K7
//
// All per-run sums are entries of one small Gram product computed on the FP64
// tensor cores (mma.sync m8n8k4 f64 -> DMMA):
//   C = U'^T V   over the run's samples k (rows padded to a multiple of 4),
//   U'[k] = [b0 b1 b2 | r0 r1 r2 | W_0 .. W_{M-1} | 1]              (7 + M <= 16)
//   V[k]  = [h b0 h b1 h b2 | h r0 h r1 h r2 | h W_0 .. h W_{M-1} | f | eb]
// where W_m is the master weight of local master vertex m in sample k. So
//   Mbb = C[b][b], Mbr = C[b][r], Mrr = C[r][r], Fb = C[b][f], Fr = C[r][f],
//   E = C[1][eb], Fw_m = C[W_m][f], Hwb_m = C[W_m][b], Hwr_m = C[W_m][r],
//   c_ml = C[W_m][W_l].
// The accumulation order inside DMMA is fixed by the hardware, so results are
// bitwise reproducible.

constexpr int kUC = 16;               // U' / V columns

constexpr int kRunWarps = 4;          // warps (= runs in flight) per K7 block
#ifndef K7_MINB
#define K7_MINB 5  // 96 registers, no spills: 20 warps/SM (4: 128 registers, 16 warps/SM, K7 +4%)
#endif
#ifndef K7_PREFETCH
#define K7_PREFETCH 0  // next-run metadata prefetch: costs the registers of minB 5 (1: spills)
#endif
#ifndef K7_STAGE
#define K7_STAGE 16
#endif
constexpr int kStage = K7_STAGE;      // sample rows staged per tensor-core pass
constexpr int kLDS = kStage + 4;      // column stride (doubles): conflict-free fragment loads

// Per-warp shared memory: staged U' / V rows (column-major); after the last
// pass the same space holds C.
constexpr int kLDT = 9;               // T tile row stride (doubles)
constexpr int kPst = 2 * kUC * kLDS - kUC * (kUC + 1) - 16 * kLDT;  // what the staging tile leaves
static_assert(kPst >= partial_size(kRunMasters), "run partial staging does not fit");
struct alignas(16) RunSmem {
  union {
    struct {
      double u[kUC][kLDS];
      double v[kUC][kLDS];
    };
    struct {
      double C[kUC][kUC + 1];
      double T[16][kLDT];  // finalize: F C[0:8][0:8] rows, staged as DMMA A fragments
      double Pst[kPst];    // finalize: the run partial, stored out coalesced
    };
  };
  double A[27];   // A_i with T_i(v) = A_i v: [i][row][col]
  double geo[19];  // a0 a1 a2 | e1 e2 | n | 1/|c|
};


// row a of the matrix A_i with T_i(v) = A_i v
__device__ __forceinline__ d3 Trow(int i, int a, d3 e1, d3 e2) {
  d3 u;
  double s;
  if (i == 0) { u = e2 - e1; s = -1.0; }  // v x u = -[u]_x v
  else if (i == 1) { u = e2; s = 1.0; }   // u x v = [u]_x v
  else { u = e1; s = -1.0; }
  if (a == 0) return mk3(0, -s * u.z, s * u.y);
  if (a == 1) return mk3(s * u.z, 0, -s * u.x);
  return mk3(-s * u.y, s * u.x, 0);
}
__device__ __forceinline__ double comp(d3 v, int a) { return a == 0 ? v.x : (a == 1 ? v.y : v.z); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// K7: one warp per run, no block-level synchronisation. Lanes own samples
// (32 per chunk); each chunk is staged 16 rows at a time and multiplied into
// the warp's C = U'^T V accumulators on the tensor cores (rows in ascending
// sample order, padded with zero rows to a multiple of 4). The run's blocks
// are then finalized from C and written as its self-describing partial.
template <bool Hess>
__global__ void __launch_bounds__(32 * kRunWarps, K7_MINB) k_run_partials(
    DevSamples S, const double* __restrict__ x, int64_t n_runs, const int64_t* __restrict__ run_off,
    const int32_t* __restrict__ run_slave, const int32_t* __restrict__ lm_off,
    const uint32_t* __restrict__ li4, const int64_t* __restrict__ pbase, double* __restrict__ partial,
    unsigned long long* __restrict__ red, double* __restrict__ warp_energy) {
  __shared__ RunSmem wsm[kRunWarps];
  __shared__ unsigned char pair_tab[kRunMasters + 1][kRunMasters * (kRunMasters + 1) / 2];  // t -> m | l << 4
  __shared__ uint64_t ss_tab[2][32];  // per lane: SS slot offsets / mirror offsets (kept out of registers)
  pdl_trigger();  // K8 may take SM slots as K7's persistent blocks retire (it waits for K7's results)
  for (int q = threadIdx.x; q < (kRunMasters + 1) * kRunMasters; q += blockDim.x) {
    const int Mq = q / kRunMasters, m = q % kRunMasters;
    if (m < Mq)
      for (int l = m; l < Mq; ++l) pair_tab[Mq][tri_index(m, l, Mq)] = (unsigned char)(m | (l << 4));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  RunSmem& W = wsm[threadIdx.x >> 5];
  const int g = lane >> 2, t4 = lane & 3;
  // Tensor-core finalize, lane-constant parts. F (9 x 6, padded 16 x 8) maps
  // the moment vector [b0 b1 b2 | r] to the slave gap gradients,
  // dg_i = F_i [b; r] with F_i = [-n e_i^T | A_i]; this lane holds the DMMA
  // fragments F[8 mt + g][4 ks + t4]. SS output slot (mt, nt, e) is
  // SS[8 mt + g][8 nt + 2 t4 + e]: its partial offset (upper entries of the
  // six stored blocks, 0xff = not stored) and mirror offset (diagonal blocks).
  {
  uint64_t ss_off = ~0ull, ss_mir = ~0ull;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int ia = 8 * mt + g, jc = 8 * nt + 2 * t4 + e, slot = 4 * mt + 2 * nt + e;
        if (ia < 9 && jc < 9) {
          const int i = ia / 3, a = ia % 3, j = jc / 3, c = jc % 3;
          if (i < j || (i == j && a <= c)) {
            const int bid = i == 0 ? j : (i == 1 ? 2 + j : 5);
            const uint64_t clr = ~(0xffull << (8 * slot));
            ss_off = (ss_off & clr) | ((uint64_t)(kSSBase + 12 * bid + 3 * a + c) << (8 * slot));
            if (i == j && a != c) ss_mir = (ss_mir & clr) | ((uint64_t)(kSSBase + 12 * bid + 3 * c + a) << (8 * slot));
          }
        }
      }
  if (threadIdx.x < 32) {
    ss_tab[0][lane] = ss_off;
    ss_tab[1][lane] = ss_mir;
  }
  }
  __syncthreads();

  double e_warp = 0;  // this warp's run energies, summed in its run order
  // persistent warps; the next run's metadata loads during this run
  struct Meta {
    int64_t s0, s1, pb;
    int M, sid0, sid1, sid2;
  };
  auto load_meta = [&](int64_t r, Meta& m) {
    m.s0 = run_off[r];
    m.s1 = run_off[r + 1];
    const int L0 = lm_off[r];
    m.M = lm_off[r + 1] - L0;
    m.sid0 = run_slave[3 * r];
    m.sid1 = run_slave[3 * r + 1];
    m.sid2 = run_slave[3 * r + 2];
    m.pb = pbase[r];
  };
  const int64_t stride = (int64_t)gridDim.x * kRunWarps;
  int64_t r = blockIdx.x * (int64_t)kRunWarps + (threadIdx.x >> 5);
#if K7_PREFETCH
  Meta nxt;
  if (r < n_runs) load_meta(r, nxt);
#endif
  for (; r < n_runs; r += stride) {
#if K7_PREFETCH
    const Meta cur = nxt;
    if (r + stride < n_runs) load_meta(r + stride, nxt);
#else
    Meta cur;
    load_meta(r, cur);
#endif
    const int64_t s0 = cur.s0, s1 = cur.s1, pb = cur.pb;
    const int M = cur.M, sid0 = cur.sid0, sid1 = cur.sid1, sid2 = cur.sid2;
    {
      const d3 a0 = ld3(x, sid0), a1 = ld3(x, sid1), a2 = ld3(x, sid2);
      const d3 e1 = a1 - a0, e2 = a2 - a0;
      const d3 cr = cross(e1, e2);
      const double cn = norm(cr);
      const double icn = cn > 0 ? 1.0 / cn : 0.0;
      const d3 n = icn * cr;
      if (lane == 0) {
        const double gv[19] = {a0.x, a0.y, a0.z, a1.x, a1.y, a1.z, a2.x, a2.y, a2.z, e1.x,
                               e1.y, e1.z, e2.x, e2.y, e2.z, n.x,  n.y,  n.z,  icn};
#pragma unroll
        for (int q = 0; q < 19; ++q) W.geo[q] = gv[q];
        if (!(cn > 0)) atomicMin(&red[1], (unsigned long long)s0);
      }
      if (lane < 27) {  // A_i = s_i [u_i]_x: T_0(v) = v x (e2-e1), T_1(v) = e2 x v, T_2(v) = v x e1
        const int ti = lane / 9, ta = (lane / 3) % 3, tc = lane % 3;
        const d3 tr = Trow(ti, ta, e1, e2);
        W.A[lane] = comp(tr, tc);
      }
    }
    __syncwarp();
    // C quadrants [rows 0-7 | 8-15] x [cols 0-7 | 8-15]; the lower-left one
    // (W_m>=2 / ones rows x b, r, W_0, W_1 columns) is never read -- its entries
    // are read from the transposed upper-right quadrant -- so 3 DMMAs per step.
    double d00 = 0, d01 = 0, d10 = 0, d11 = 0, d30 = 0, d31 = 0;

    for (int64_t base = s0; base < s1; base += 32) {
      const int64_t i = base + lane;
      const int rows = s1 - base < 32 ? (int)(s1 - base) : 32;
      double ub[3] = {0, 0, 0}, rr[3] = {0, 0, 0}, w[3] = {0, 0, 0};
      double h = 0, f = 0, eb = 0;
      uint32_t li = 0xffffffffu;
      int nm = 0;
      if (lane < rows) {
        const double icn = W.geo[18];
        int mid[3];
        load_master(S, i, nm, w, mid);
        ub[0] = S.beta_s[3 * i];
        ub[1] = S.beta_s[3 * i + 1];
        ub[2] = S.beta_s[3 * i + 2];
        li = li4[i];
        const double eps = S.eps[i], cf = S.coef[i];
        if (icn > 0) {
          const d3 a0 = mk3(W.geo[0], W.geo[1], W.geo[2]), a1 = mk3(W.geo[3], W.geo[4], W.geo[5]);
          const d3 a2 = mk3(W.geo[6], W.geo[7], W.geo[8]), n = mk3(W.geo[15], W.geo[16], W.geo[17]);
          const d3 xs = (ub[0] * a0 + ub[1] * a1) + ub[2] * a2;
          d3 xm = mk3(0, 0, 0);
#pragma unroll
          for (int j = 0; j < 3; ++j) {  // branch-free: absent masters have w = 0 (index clamped)
            const int mj = j < nm ? mid[j] : mid[0];
            xm = xm + (j < nm ? w[j] : 0.0) * ld3(x, mj);
          }
          const d3 d = xm - xs;
          const double gap = dot(n, d);
          if (!(gap > 0)) {
            atomicMin(&red[0], (unsigned long long)i);
          } else {
            const d3 rv = icn * (d - gap * n);
            rr[0] = rv.x;
            rr[1] = rv.y;
            rr[2] = rv.z;
            if (gap < eps) {  // barrier.hpp:55-66 with one reciprocal
              const double dd = gap - eps, ig = 1.0 / gap;
              const double ln = log(gap / eps);
              const double q2 = dd * ig;
              eb = cf * (-dd * dd * ln);
              f = cf * (-2.0 * dd * ln - dd * q2);
              h = cf * dmax(-2.0 * ln - 4.0 * q2 + q2 * q2, 0.0);
            }
          }
        }
      }
      const int prow = (rows + 3) & ~3;  // rows incl. zero padding
      for (int half = 0; half * kStage < prow; ++half) {
        const int row = lane - half * kStage;
        __syncwarp();
        if (row >= 0 && row < kStage) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            W.u[c][row] = ub[c];
            W.v[c][row] = h * ub[c];
            W.u[3 + c][row] = rr[c];
            W.v[3 + c][row] = h * rr[c];
          }
#pragma unroll
          for (int c = 6; c < kUC; ++c) W.u[c][row] = W.v[c][row] = 0.0;
          if (lane < rows) W.u[6 + M][row] = 1.0;
          W.v[6 + M][row] = f;
          W.v[7 + M][row] = eb;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            if (j < nm) {
              const int m = (li >> (8 * j)) & 0xff;
              W.u[6 + m][row] = w[j];
              W.v[6 + m][row] = h * w[j];
            }
          }
        }
        __syncwarp();
        const int kk = min(kStage, prow - half * kStage);
        for (int k = t4; k < kk; k += 4) {
          const double ua = W.u[g][k], ub8 = W.u[8 + g][k];
          const double va = W.v[g][k], vb = W.v[8 + g][k];
          dmma(d00, d01, ua, va);
          dmma(d10, d11, ua, vb);
          dmma(d30, d31, ub8, vb);
        }
      }
    }
    __syncwarp();
    double (*C)[kUC + 1] = W.C;
    C[g][2 * t4] = d00;
    C[g][2 * t4 + 1] = d01;
    C[g][8 + 2 * t4] = d10;
    C[g][9 + 2 * t4] = d11;
    C[8 + g][8 + 2 * t4] = d30;
    C[8 + g][9 + 2 * t4] = d31;
    __syncwarp();
    double* P = partial + pb;
    double* Q = Hess ? W.Pst : P;  // Hess: the partial is staged, then stored coalesced
    const int colF = 6 + M, colE = 7 + M;
    const double* A = W.A;
    const double* nn = W.geo + 15;
    // T = F C[0:8][0:16] (8 DMMAs): column colF holds the slave gradients
    // g_i = -Fb_i n + T_i(Fr), columns 6 + m hold a_{m,i} = -Hwb_{m,i} n +
    // T_i(Hwr_m); then SS = T[:, 0:8] F^T (8 DMMAs) holds all nine slave
    // blocks F_i Z F_j^T of the moment matrix Z = C[0:6][0:6].
    double fa[2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int ia = 8 * mt + g, p = 4 * ks + t4;
        double v = 0.0;
        if (ia < 9 && p < 6) {
          const int i = ia / 3, a = ia % 3;
          v = p < 3 ? (p == i ? -nn[a] : 0.0) : A[9 * i + 3 * a + (p - 3)];
        }
        fa[mt][ks] = v;
      }
    double t[2][2][2] = {{{0, 0}, {0, 0}}, {{0, 0}, {0, 0}}};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const double b0 = C[4 * ks + t4][g], b1 = C[4 * ks + t4][8 + g];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        dmma(t[mt][0][0], t[mt][0][1], fa[mt][ks], b0);
        dmma(t[mt][1][0], t[mt][1][1], fa[mt][ks], b1);
      }
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int ia = 8 * mt + g, q = 8 * nt + 2 * t4 + e;
          if (ia < 9) {
            if (q == colF) Q[4 + ia + ia / 3] = t[mt][nt][e];  // [4 + 4 i + a]
            else if (Hess && q >= 6 && q < colF) Q[m_base(q - 6) + ia + ia / 3] = t[mt][nt][e];
          }
        }
    if (Hess) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        W.T[8 * mt + g][2 * t4] = t[mt][0][0];
        W.T[8 * mt + g][2 * t4 + 1] = t[mt][0][1];
      }
      __syncwarp();
      double sv[2][2][2] = {{{0, 0}, {0, 0}}, {{0, 0}, {0, 0}}};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const double ta0 = W.T[g][4 * ks + t4], ta1 = W.T[8 + g][4 * ks + t4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          dmma(sv[0][nt][0], sv[0][nt][1], ta0, fa[nt][ks]);
          dmma(sv[1][nt][0], sv[1][nt][1], ta1, fa[nt][ks]);
        }
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int slot = 4 * mt + 2 * nt + e;
            const int o = (int)((ss_tab[0][lane] >> (8 * slot)) & 0xff), om = (int)((ss_tab[1][lane] >> (8 * slot)) & 0xff);
            if (o != 0xff) Q[o] = sv[mt][nt][e];
            if (om != 0xff) Q[om] = sv[mt][nt][e];
          }
      for (int tq = lane; tq < M * (M + 1) / 2; tq += 32) {  // master pairs, dense upper triangle
        const int pr = pair_tab[M][tq];
        Q[pair_base(M) + tq] = C[6 + (pr & 15)][6 + (pr >> 4)];
      }
    }
    const double Erun = C[6 + M][colE];
    if (lane < 4) Q[lane] = lane == 3 ? Erun : nn[lane];
    if (lane < M) Q[m_base(lane) + 3] = C[6 + lane][colF];  // s_m
    if (Hess) {  // 16-byte chunks, consecutive lanes on consecutive chunks
      __syncwarp();
      const int nch = partial_size(M) / 2;
      for (int q = lane; q < nch; q += 32)
        reinterpret_cast<double2*>(P)[q] = reinterpret_cast<const double2*>(W.Pst)[q];
    }
    e_warp += Erun;
    __syncwarp();
  }
  if (lane == 0) warp_energy[blockIdx.x * kRunWarps + (threadIdx.x >> 5)] = e_warp;
}

// ---------------------------------------------------------------------------
// K8: gather. The plan lists, for every BCSR block, its contributions
// (run partial, row role, block index) in ascending run order; one thread per
// block sums them in that order (bitwise deterministic, no atomics), and one
// thread per vertex row sums its gradient the same way.
//   contribution code = (pbase << 12) | (M << 8) | (role << 4) | b
//   row entry code    = (pbase << 12) | (M << 8) | role
// role < 3: slave vertex i of the run, else local master role - 3; b indexes
// the run's columns the same way.

// Block (role, b) of a run partial P; every group read is one 256-bit load.
__device__ __forceinline__ void contrib_block(int role, int b, const double* __restrict__ P, int M, double* blk) {
  if (role < 3 && b < 3) {  // SS: upper blocks stored, lower = transpose
    const int lo = min(role, b), hi = max(role, b);
    const int bid = lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
    const double* Sb = P + kSSBase + 12 * bid;
    double sb[9];
    ldg4(Sb, sb[0], sb[1], sb[2], sb[3]);
    ldg4(Sb + 4, sb[4], sb[5], sb[6], sb[7]);
    sb[8] = __ldg(Sb + 8);
    if (role <= b) {
#pragma unroll
      for (int q = 0; q < 9; ++q) blk[q] = sb[q];
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) blk[3 * a + c] = sb[3 * c + a];
    }
    return;
  }
  double nn[3], e_;
  ldg4(P, nn[0], nn[1], nn[2], e_);
  if (role < 3 || b < 3) {  // SM(i, m) = a_{m,i} n^T, MS(m, i) = n a_{m,i}^T
    const bool sm = role < 3;
    double A[3], w_;
    ldg4(P + m_base(sm ? b - 3 : role - 3) + 4 * (sm ? role : b), A[0], A[1], A[2], w_);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) blk[3 * a + c] = sm ? A[a] * nn[c] : nn[a] * A[c];
    return;
  }
  const int m = role - 3, l = b - 3;  // MM(m, l) = c_ml n n^T
  const double cv = P[pair_base(M) + (m <= l ? tri_index(m, l, M) : tri_index(l, m, M))];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) blk[3 * a + c] = cv * (nn[a] * nn[c]);
}

constexpr int kGatherThreads = 256;

// Items [0, nnzb) are BCSR blocks (Hess only), then one item per vertex row
// (Rows). The next contribution code is loaded while the current one is summed.
#ifndef K8_MINB
#define K8_MINB 5  // 48 registers, 40 warps/SM: more loads in flight (pass -3%; 6 and 8 spill)
#endif
#ifndef K8_BLOCKS_MINB
#define K8_BLOCKS_MINB 5  // blocks-only gather (host-buffer path): 48 registers + 24 B of spills; 4 (62, no spills) is 2% slower end to end
#endif
template <bool Hess, bool Rows = true>
__global__ void __launch_bounds__(kGatherThreads, Rows ? K8_MINB : K8_BLOCKS_MINB) k_gather(int64_t nnzb, int32_t n_rows,
                                                           const int32_t* __restrict__ blk_off,
                                                           const int64_t* __restrict__ contrib,
                                                           double* __restrict__ vals,
                                                           const int32_t* __restrict__ ent_off,
                                                           const int64_t* __restrict__ ent,
                                                           const double* __restrict__ partial,
                                                           double* __restrict__ grad) {
  const int64_t nb = Hess ? nnzb : 0;
  const int64_t items = nb + (Rows ? n_rows : 0);
  __shared__ double stage[kGatherThreads / 32][9 * 32];  // per-warp block-value transpose
  pdl_trigger();
  pdl_wait();  // K7's partials
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < items; k += (int64_t)gridDim.x * blockDim.x) {
    if (k < nb) {
      const int64_t bk = k;  // natural order: neighbouring blocks share run partials in L1
      double acc[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) acc[q] = 0.0;
      const int c0 = blk_off[bk], c1 = blk_off[bk + 1];
      int64_t code = contrib[c0];
      for (int c = c0; c < c1; ++c) {
        const int64_t nxt = c + 1 < c1 ? contrib[c + 1] : 0;
        double blk[9];
        contrib_block((int)((code >> 4) & 0xf), (int)(code & 0xf), partial + (code >> 12), (int)((code >> 8) & 0xf),
                      blk);
#pragma unroll
        for (int q = 0; q < 9; ++q) acc[q] += blk[q];
        code = nxt;
      }
      const int64_t k0 = k - (threadIdx.x & 31);  // the warp's first item (warp-uniform)
      if (k0 + 31 < nb) {  // whole warp on blocks: transpose through shared memory, coalesced stores
        double* st = stage[threadIdx.x >> 5];
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int q = 0; q < 9; ++q) st[9 * lane + q] = acc[q];
        __syncwarp();
        double* out = vals + 9 * k0;
#pragma unroll
        for (int j = 0; j < 9; ++j) out[32 * j + lane] = st[32 * j + lane];
        __syncwarp();
      } else {
        double* out = vals + 9 * bk;
#pragma unroll
        for (int q = 0; q < 9; ++q) out[q] = acc[q];
      }
    } else {
      const int64_t v = k - nb;
      d3 g = mk3(0, 0, 0);
      const int e1 = ent_off[v + 1];
      for (int e = ent_off[v]; e < e1; ++e) {
        const int64_t en = ent[e];
        const double* P = partial + (en >> 12);
        const int role = (int)(en & 0xff);
        double v0, v1, v2, v3;
        if (role < 3) {
          ldg4(P + 4 + 4 * role, v0, v1, v2, v3);
          g = g + mk3(v0, v1, v2);
        } else {
          double n0, n1, n2, e_;
          ldg4(P, n0, n1, n2, e_);
          ldg4(P + m_base(role - 3), v0, v1, v2, v3);
          g = g + v3 * mk3(n0, n1, n2);
        }
      }
      grad[3 * v] = g.x;
      grad[3 * v + 1] = g.y;
      grad[3 * v + 2] = g.z;
    }
  }
}

__global__ void k_flush(double* buf, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = buf[i] * 0.5 + 1.0;
}

}  // namespace
}  // namespace gmcp_b200
