// Per-iteration contact kernels: energy (K6), two-level deterministic
// gradient + Gauss-Newton Hessian assembly (K7 run partials, K8 row gather),
// pressure field (K12), force summary and kinematics download.
//
// Reference: proj/include/gmcp/contact_energy.hpp:95-179, 225-276.
#include <algorithm>
#include <map>
#include <numeric>

#include "ctx.hpp"
#include "kin.cuh"
#include "reduce.cuh"

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
// K7: one warp per slave run -> compact partial.
// Partial layout (doubles) at pbase[r]:
//   [0] energy  [1..3] n  [4..12] slave gradients (i*3+k)
//   [13..66] SS blocks (0,0),(0,1),(0,2),(1,1),(1,2),(2,2), 9 each, row-major
//   [67 + 10m] s_m, [68 + 10m + 3i + k] a_{m,i}[k]   (m < M local master verts)
//   [67 + 10M + p] c_p                                 (p < P local master pairs)

constexpr int kRunWarps = 4;  // warps per block in K7
constexpr int kSSBase = 13;
constexpr int kMBase = 67;

struct ChunkSmem {
  double h[32];
  double f[32];
  double dgs[32][9];
  double w[32][3];
  int mid[32][3];
};

__constant__ unsigned char c_ss_entry[45][3];  // (block, a, c) of the 45 unique SS entries
__constant__ unsigned char c_ss_blk[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};

template <bool Hess>
__global__ void __launch_bounds__(32 * kRunWarps) k_run_partials(
    DevSamples S, const double* __restrict__ x, int64_t n_runs, const int64_t* __restrict__ run_off,
    const int32_t* __restrict__ run_slave, const int32_t* __restrict__ lm_off, const int32_t* __restrict__ lm_ids,
    const int32_t* __restrict__ lp_off, const int32_t* __restrict__ lp, const int64_t* __restrict__ pbase,
    double* __restrict__ partial, unsigned long long* __restrict__ red) {
  __shared__ ChunkSmem smem[kRunWarps];
  const int lane = threadIdx.x & 31;
  ChunkSmem& sm = smem[threadIdx.x >> 5];
  const int64_t nwarps = (int64_t)gridDim.x * kRunWarps;
  for (int64_t r = blockIdx.x * (int64_t)kRunWarps + (threadIdx.x >> 5); r < n_runs; r += nwarps) {
    const int64_t s0 = run_off[r], s1 = run_off[r + 1];
    const d3 a0 = ld3(x, run_slave[3 * r]), a1 = ld3(x, run_slave[3 * r + 1]), a2 = ld3(x, run_slave[3 * r + 2]);
    const d3 e1 = a1 - a0, e2 = a2 - a0;
    const d3 c = cross(e1, e2);
    const double cn = norm(c);
    const int64_t base = pbase[r];
    double* P = partial + base;
    if (!(cn > 0)) {
      if (lane == 0) atomicMin(&red[1], (unsigned long long)s0);
      continue;
    }
    const d3 n = c / cn;
    const int m0 = lm_off[r], M = lm_off[r + 1] - m0;
    const int p0 = lp_off[r], NP = lp_off[r + 1] - p0;
    const int nout = Hess ? (54 + 10 * M + NP) : (10 * M);
    for (int o = lane; o < nout; o += 32) {
      if (Hess) P[kSSBase + o] = 0;
      else P[kMBase + o] = 0;
    }
    double eacc = 0, gacc[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) gacc[q] = 0;

    for (int64_t cs = s0; cs < s1; cs += 32) {
      const int64_t i = cs + lane;
      double h = 0, f = 0;
      d3 dgs[3] = {mk3(0, 0, 0), mk3(0, 0, 0), mk3(0, 0, 0)};
      double w[3] = {0, 0, 0};
      int mid[3] = {-1, -1, -1};
      if (i < s1) {
        const double b0 = S.beta_s[3 * i], b1 = S.beta_s[3 * i + 1], b2 = S.beta_s[3 * i + 2];
        const d3 xs = (b0 * a0 + b1 * a1) + b2 * a2;
        int nm;
        load_master(S, i, nm, w, mid);
        d3 xm = mk3(0, 0, 0);
        for (int j = 0; j < nm; ++j) xm = xm + w[j] * ld3(x, mid[j]);
        for (int j = nm; j < 3; ++j) mid[j] = -1;
        const d3 d = xm - xs;
        const double g = dot(n, d);
        if (!(g > 0)) {
          atomicMin(&red[0], (unsigned long long)i);
        } else {
          const d3 rr = (d - g * n) / cn;
          dgs[0] = (-b0) * n + cross(rr, e2 - e1);
          dgs[1] = (-b1) * n + cross(e2, rr);
          dgs[2] = (-b2) * n + cross(rr, e1);
          double B, dB, ddB;
          barrier_eval(g, S.eps[i], B, dB, ddB);
          const double cf = S.coef[i];
          eacc += cf * B;
          f = cf * dB;
          h = cf * dmax(ddB, 0.0);
#pragma unroll
          for (int v = 0; v < 3; ++v) {
            gacc[3 * v] += f * dgs[v].x;
            gacc[3 * v + 1] += f * dgs[v].y;
            gacc[3 * v + 2] += f * dgs[v].z;
          }
        }
      }
      sm.h[lane] = h;
      sm.f[lane] = f;
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        sm.dgs[lane][3 * v] = dgs[v].x;
        sm.dgs[lane][3 * v + 1] = dgs[v].y;
        sm.dgs[lane][3 * v + 2] = dgs[v].z;
        sm.w[lane][v] = w[v];
        sm.mid[lane][v] = mid[v];
      }
      __syncwarp();
      const int nk = (int)(s1 - cs < 32 ? s1 - cs : 32);
      if (Hess) {
        for (int o = lane; o < 45; o += 32) {
          const int blk = c_ss_entry[o][0], a = c_ss_entry[o][1], cc = c_ss_entry[o][2];
          const int bi = c_ss_blk[blk][0], bj = c_ss_blk[blk][1];
          double s = 0;
          for (int k = 0; k < nk; ++k) s += sm.h[k] * (sm.dgs[k][3 * bi + a] * sm.dgs[k][3 * bj + cc]);
          P[kSSBase + 9 * blk + 3 * a + cc] += s;
          if (bi == bj && a != cc) P[kSSBase + 9 * blk + 3 * cc + a] += s;
        }
      }
      for (int m = lane; m < M; m += 32) {
        const int gm = lm_ids[m0 + m];
        double s = 0, av[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) av[q] = 0;
        for (int k = 0; k < nk; ++k) {
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            if (sm.mid[k][j] != gm) continue;
            const double wj = sm.w[k][j];
            s += sm.f[k] * wj;
            if (Hess) {
              const double hw = sm.h[k] * wj;
#pragma unroll
              for (int q = 0; q < 9; ++q) av[q] += hw * sm.dgs[k][q];
            }
          }
        }
        P[kMBase + 10 * m] += s;
        if (Hess)
#pragma unroll
          for (int q = 0; q < 9; ++q) P[kMBase + 10 * m + 1 + q] += av[q];
      }
      if (Hess) {
        for (int p = lane; p < NP; p += 32) {
          const int pk = lp[p0 + p];
          const int ga = lm_ids[m0 + (pk >> 16)], gb = lm_ids[m0 + (pk & 0xffff)];
          double s = 0;
          for (int k = 0; k < nk; ++k) {
            double wa = 0, wb = 0;
            bool ha = false, hb = false;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              if (sm.mid[k][j] == ga) { wa = sm.w[k][j]; ha = true; }
              if (sm.mid[k][j] == gb) { wb = sm.w[k][j]; hb = true; }
            }
            if (ha && hb) s += sm.h[k] * (wa * wb);
          }
          P[kMBase + 10 * M + p] += s;
        }
      }
      __syncwarp();
    }
    eacc = warp_sum(eacc);
#pragma unroll
    for (int q = 0; q < 9; ++q) gacc[q] = warp_sum(gacc[q]);
    if (lane == 0) {
      P[0] = eacc;
      P[1] = n.x;
      P[2] = n.y;
      P[3] = n.z;
#pragma unroll
      for (int q = 0; q < 9; ++q) P[4 + q] = gacc[q];
    }
  }
}

// Energy of the pass = sum of run energies in run order.
__global__ void __launch_bounds__(kRedThreads) k_run_energy(int64_t n_runs, const int64_t* __restrict__ pbase,
                                                             const double* __restrict__ partial,
                                                             double* __restrict__ parts) {
  __shared__ double sh[kRedThreads / 32];
  double e = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_runs; r += (int64_t)gridDim.x * blockDim.x)
    e += partial[pbase[r]];
  const double v = block_sum<kRedThreads>(e, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = v;
}

// ---------------------------------------------------------------------------
// K8: one warp per vertex row: gather run partials into the BCSR row + gradient.

__device__ __forceinline__ int find_col(const int32_t* __restrict__ cols, int lo, int hi, int col) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cols[mid] < col) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <bool Hess>
__global__ void __launch_bounds__(256) k_row_gather(
    int32_t n_rows, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols, double* __restrict__ vals,
    const int32_t* __restrict__ ent_off, const int64_t* __restrict__ ent, const int32_t* __restrict__ run_slave,
    const int32_t* __restrict__ lm_off, const int32_t* __restrict__ lm_ids, const int32_t* __restrict__ lp_off,
    const int32_t* __restrict__ lp, const int64_t* __restrict__ pbase, const double* __restrict__ partial,
    double* __restrict__ grad) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); v < n_rows; v += nwarps) {
    const int c0 = Hess ? rowptr[v] : 0, c1 = Hess ? rowptr[v + 1] : 0;
    if (Hess)
      for (int q = lane; q < 9 * (c1 - c0); q += 32) vals[9 * (int64_t)c0 + q] = 0;
    d3 g = mk3(0, 0, 0);
    __syncwarp();
    for (int e = ent_off[v]; e < ent_off[v + 1]; ++e) {
      const int64_t en = ent[e];
      const int64_t r = en >> 20;
      const int role = (int)(en & 0xfffff);
      const double* P = partial + pbase[r];
      const d3 n = mk3(P[1], P[2], P[3]);
      const int m0 = lm_off[r], M = lm_off[r + 1] - m0;
      if (role < 3) {
        const int i = role;
        g = g + mk3(P[4 + 3 * i], P[5 + 3 * i], P[6 + 3 * i]);
        if (Hess) {
          for (int b = lane; b < 3 + M; b += 32) {
            double blk[9];
            int col;
            if (b < 3) {
              const int j = b;
              col = run_slave[3 * r + j];
              const int lo = min(i, j), hi = max(i, j);
              const int bid = lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
              const double* S = P + kSSBase + 9 * bid;
              if (i <= j) {
#pragma unroll
                for (int q = 0; q < 9; ++q) blk[q] = S[q];
              } else {
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                  for (int cc = 0; cc < 3; ++cc) blk[3 * a + cc] = S[3 * cc + a];
              }
            } else {
              const int k = b - 3;
              col = lm_ids[m0 + k];
              const double* A = P + kMBase + 10 * k + 1 + 3 * i;
              const double nn[3] = {n.x, n.y, n.z};
#pragma unroll
              for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) blk[3 * a + cc] = A[a] * nn[cc];
            }
            const int slot = find_col(cols, c0, c1, col);
            double* out = vals + 9 * (int64_t)slot;
#pragma unroll
            for (int q = 0; q < 9; ++q) out[q] += blk[q];
          }
        }
      } else {
        const int m = role - 3;
        const double s = P[kMBase + 10 * m];
        g = g + s * n;
        if (Hess) {
          const int p0 = lp_off[r], NP = lp_off[r + 1] - p0;
          const double nn[3] = {n.x, n.y, n.z};
          for (int b = lane; b < 3 + NP; b += 32) {
            double blk[9];
            int col;
            if (b < 3) {
              const int j = b;
              col = run_slave[3 * r + j];
              const double* A = P + kMBase + 10 * m + 1 + 3 * j;
#pragma unroll
              for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) blk[3 * a + cc] = nn[a] * A[cc];
            } else {
              const int p = b - 3;
              const int pk = lp[p0 + p];
              const int la = pk >> 16, lb = pk & 0xffff;
              if (la != m && lb != m) continue;
              col = lm_ids[m0 + (la == m ? lb : la)];
              const double cv = P[kMBase + 10 * M + p];
#pragma unroll
              for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) blk[3 * a + cc] = cv * (nn[a] * nn[cc]);
            }
            const int slot = find_col(cols, c0, c1, col);
            double* out = vals + 9 * (int64_t)slot;
#pragma unroll
            for (int q = 0; q < 9; ++q) out[q] += blk[q];
          }
        }
      }
      __syncwarp();
    }
    if (lane == 0) {
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

int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

void init_ss_table() {
  static bool done = false;
  if (done) return;
  unsigned char tab[45][3];
  int k = 0;
  const int blks[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
  for (int b = 0; b < 6; ++b)
    for (int a = 0; a < 3; ++a)
      for (int cc = 0; cc < 3; ++cc) {
        if (blks[b][0] == blks[b][1] && cc < a) continue;
        tab[k][0] = (unsigned char)b;
        tab[k][1] = (unsigned char)a;
        tab[k][2] = (unsigned char)cc;
        ++k;
      }
  GMCP_CUDA(cudaMemcpyToSymbol(c_ss_entry, tab, sizeof tab));
  done = true;
}

}  // namespace

// ===========================================================================
// host entry points

void derive_sample_fields(Ctx& c) {
  const int64_t n = c.ns;
  c.s_wm.resize(3 * n);
  c.s_coef.resize(n);
  if (n) {
    k_derive<<<grid_for(n, 256), 256, 0, c.stream>>>(n, c.s_type.p, c.s_beta_m.p, c.s_eta.p, c.s_weight.p,
                                                     c.s_gamma.p, c.params.kappa_face, c.params.kappa_edge,
                                                     c.params.kappa_point, c.s_wm.p, c.s_coef.p);
    ++c.launches;
    GMCP_CUDA(cudaGetLastError());
  }
  // face sample index list (pressure-field order)
  std::vector<int8_t> t = c.s_type.to_host(c.stream);
  std::vector<int64_t> f;
  for (int64_t i = 0; i < n; ++i)
    if (t[i] == GMCP_FACE) f.push_back(i);
  c.face_idx.upload(f, c.stream);
  c.face_idx.n = f.size();
  c.plan.valid = false;
}

// Host-side assembly plan from the device sample set (per rebuild).
void build_assembly_plan(Ctx& c) {
  AssemblyPlan& P = c.plan;
  const int64_t n = c.ns;
  const std::vector<int32_t> sl = c.s_slave.to_host(c.stream);
  const std::vector<int32_t> ms = c.s_master.to_host(c.stream);
  std::vector<int64_t> run_off{0};
  std::vector<int32_t> run_slave;
  for (int64_t i = 0; i < n; ++i) {
    if (i == 0 || sl[3 * i] != sl[3 * i - 3] || sl[3 * i + 1] != sl[3 * i - 2] || sl[3 * i + 2] != sl[3 * i - 1]) {
      if (i > 0) run_off.push_back(i);
      run_slave.insert(run_slave.end(), {sl[3 * i], sl[3 * i + 1], sl[3 * i + 2]});
    }
  }
  if (n > 0) run_off.push_back(n);
  const int64_t R = (int64_t)run_slave.size() / 3;
  std::vector<int32_t> lm_off{0}, lm_ids, lp_off{0}, lp;
  std::vector<int64_t> pbase(R);
  int64_t plen = 0;
  std::vector<int32_t> loc;
  for (int64_t r = 0; r < R; ++r) {
    loc.clear();
    for (int64_t i = run_off[r]; i < run_off[r + 1]; ++i)
      for (int j = 0; j < 3; ++j)
        if (ms[3 * i + j] >= 0) loc.push_back(ms[3 * i + j]);
    std::sort(loc.begin(), loc.end());
    loc.erase(std::unique(loc.begin(), loc.end()), loc.end());
    if (loc.size() >= 65535) throw StatusError(GMCP_ERR_CONFIG, "slave triangle touches too many master vertices");
    lm_ids.insert(lm_ids.end(), loc.begin(), loc.end());
    lm_off.push_back((int32_t)lm_ids.size());
    std::vector<int32_t> pairs;
    for (int64_t i = run_off[r]; i < run_off[r + 1]; ++i) {
      int li[3], nm = 0;
      for (int j = 0; j < 3; ++j)
        if (ms[3 * i + j] >= 0)
          li[nm++] = (int)(std::lower_bound(loc.begin(), loc.end(), ms[3 * i + j]) - loc.begin());
      for (int a = 0; a < nm; ++a)
        for (int b = 0; b < nm; ++b)
          if (li[a] <= li[b]) pairs.push_back((li[a] << 16) | li[b]);
    }
    std::sort(pairs.begin(), pairs.end());
    pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
    lp.insert(lp.end(), pairs.begin(), pairs.end());
    lp_off.push_back((int32_t)lp.size());
    pbase[r] = plen;
    plen += kMBase + 10 * (int64_t)loc.size() + (int64_t)pairs.size();
  }
  // BCSR pattern + row entries over all N vertex rows
  const int64_t N = c.n_vertices();
  std::vector<std::vector<int32_t>> rc(N);
  std::vector<int32_t> ent_cnt(N + 1, 0);
  std::vector<std::vector<int64_t>> rent(N);
  for (int64_t r = 0; r < R; ++r) {
    const int32_t* s = &run_slave[3 * r];
    const int32_t* L = lm_ids.data() + lm_off[r];
    const int M = lm_off[r + 1] - lm_off[r];
    for (int i = 0; i < 3; ++i) {
      rent[s[i]].push_back((r << 20) | i);
      for (int j = 0; j < 3; ++j) rc[s[i]].push_back(s[j]);
      for (int k = 0; k < M; ++k) rc[s[i]].push_back(L[k]);
    }
    for (int k = 0; k < M; ++k) {
      rent[L[k]].push_back((r << 20) | (3 + k));
      for (int j = 0; j < 3; ++j) rc[L[k]].push_back(s[j]);
    }
    for (int p = lp_off[r]; p < lp_off[r + 1]; ++p) {
      const int a = lp[p] >> 16, b = lp[p] & 0xffff;
      rc[L[a]].push_back(L[b]);
      rc[L[b]].push_back(L[a]);
    }
  }
  std::vector<int32_t> rowptr(N + 1, 0), cols, eoff(N + 1, 0);
  std::vector<int64_t> ents;
  for (int64_t v = 0; v < N; ++v) {
    auto& cv = rc[v];
    std::sort(cv.begin(), cv.end());
    cv.erase(std::unique(cv.begin(), cv.end()), cv.end());
    cols.insert(cols.end(), cv.begin(), cv.end());
    rowptr[v + 1] = (int32_t)cols.size();
    ents.insert(ents.end(), rent[v].begin(), rent[v].end());
    eoff[v + 1] = (int32_t)ents.size();
  }
  cudaStream_t s = c.stream;
  P.n_runs = R;
  P.run_off.upload(run_off, s);
  P.run_slave.upload(run_slave, s);
  P.lm_off.upload(lm_off, s);
  P.lm_ids.upload(lm_ids, s);
  P.lp_off.upload(lp_off, s);
  P.lp.upload(lp, s);
  P.pbase.upload(pbase, s);
  P.partial_len = plen;
  P.partial.resize(std::max<int64_t>(plen, 1));
  P.n_rows = (int32_t)N;
  P.nnzb = (int64_t)cols.size();
  P.rowptr.upload(rowptr, s);
  P.cols.upload(cols, s);
  P.vals.resize(std::max<int64_t>(9 * P.nnzb, 1));
  P.row_ent_off.upload(eoff, s);
  P.row_ent.upload(ents, s);
  c.sync();
  P.valid = true;
}

namespace {
void launch_assembly(Ctx& c, int mode) {
  AssemblyPlan& P = c.plan;
  const DevSamples S = c.samples();
  const int rb = (int)std::max<int64_t>(1, std::min<int64_t>((P.n_runs + kRunWarps - 1) / kRunWarps, 148 * 16));
  if (mode == 1)
    k_run_partials<true><<<rb, 32 * kRunWarps, 0, c.stream>>>(S, c.X(), P.n_runs, P.run_off.p, P.run_slave.p,
                                                              P.lm_off.p, P.lm_ids.p, P.lp_off.p, P.lp.p,
                                                              P.pbase.p, P.partial.p, c.red_u.p);
  else
    k_run_partials<false><<<rb, 32 * kRunWarps, 0, c.stream>>>(S, c.X(), P.n_runs, P.run_off.p, P.run_slave.p,
                                                               P.lm_off.p, P.lm_ids.p, P.lp_off.p, P.lp.p,
                                                               P.pbase.p, P.partial.p, c.red_u.p);
  const int gb = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)P.n_rows + 7) / 8, 148 * 32));
  if (mode == 1)
    k_row_gather<true><<<gb, 256, 0, c.stream>>>(P.n_rows, P.rowptr.p, P.cols.p, P.vals.p, P.row_ent_off.p,
                                                 P.row_ent.p, P.run_slave.p, P.lm_off.p, P.lm_ids.p, P.lp_off.p,
                                                 P.lp.p, P.pbase.p, P.partial.p, c.grad.p);
  else
    k_row_gather<false><<<gb, 256, 0, c.stream>>>(P.n_rows, P.rowptr.p, P.cols.p, P.vals.p, P.row_ent_off.p,
                                                  P.row_ent.p, P.run_slave.p, P.lm_off.p, P.lm_ids.p, P.lp_off.p,
                                                  P.lp.p, P.pbase.p, P.partial.p, c.grad.p);
  k_run_energy<<<kRedBlocks, kRedThreads, 0, c.stream>>>(P.n_runs, P.pbase.p, P.partial.p, c.red_d.p);
  k_sum_parts<<<1, kRedThreads, 0, c.stream>>>(c.red_d.p, kRedBlocks, 1, c.red_d.p + kRedBlocks);
  c.launches += 4;
  GMCP_CUDA(cudaGetLastError());
}
}  // namespace

double run_assembly(Ctx& c, int mode, int64_t* bad) {
  init_ss_table();
  if (!c.plan.valid) build_assembly_plan(c);
  c.grad.resize(std::max<int64_t>(c.n_dof, 1));
  c.red_d.resize(kRedBlocks + 8);
  reset_red(c);
  *bad = -1;
  if (c.ns == 0) {
    c.grad.zero(c.stream);
    if (c.plan.nnzb) GMCP_CUDA(cudaMemsetAsync(c.plan.vals.p, 0, 9 * c.plan.nnzb * sizeof(double), c.stream));
    c.sync();
    return 0.0;
  }
  launch_assembly(c, mode);
  unsigned long long u[4];
  double e;
  GMCP_CUDA(cudaMemcpyAsync(u, c.red_u.p, sizeof u, cudaMemcpyDeviceToHost, c.stream));
  GMCP_CUDA(cudaMemcpyAsync(&e, c.red_d.p + kRedBlocks, sizeof e, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  const int64_t first_bad = u[0] == ~0ull ? -1 : (int64_t)u[0];
  const int64_t first_deg = u[1] == ~0ull ? -1 : (int64_t)u[1];
  if (first_deg >= 0 && (first_bad < 0 || first_deg < first_bad))
    throw StatusError(GMCP_ERR_DEGENERATE, "contact sample on a degenerate slave triangle", first_deg);
  if (first_bad >= 0) {
    *bad = first_bad;
    // report the offending gap like the reference message (contact_energy.hpp:132-135)
    Kin k;
    (void)k;
    throw StatusError(GMCP_ERR_INFEASIBLE, "contact sample " + std::to_string(first_bad) + " has non-positive gap",
                      first_bad);
  }
  return e;
}

void time_assembly(Ctx& c, int reps, int flush_l2, double* ms_pass, double* ms_kernel) {
  init_ss_table();
  if (!c.plan.valid) build_assembly_plan(c);
  c.grad.resize(std::max<int64_t>(c.n_dof, 1));
  c.red_d.resize(kRedBlocks + 8);
  reset_red(c);
  DBuf<double> flush;
  const int64_t nflush = flush_l2 ? (int64_t)(256ll << 20) / 8 : 0;  // 256 MB > 126 MB L2
  if (nflush) flush.resize(nflush);
  cudaEvent_t e0, e1, k0, k1;
  GMCP_CUDA(cudaEventCreate(&e0));
  GMCP_CUDA(cudaEventCreate(&e1));
  GMCP_CUDA(cudaEventCreate(&k0));
  GMCP_CUDA(cudaEventCreate(&k1));
  double tot = 0, totk = 0;
  for (int it = 0; it < reps; ++it) {
    if (nflush) {
      k_flush<<<148 * 8, 256, 0, c.stream>>>(flush.p, nflush);
      ++c.launches;
    }
    GMCP_CUDA(cudaEventRecord(e0, c.stream));
    launch_assembly(c, 1);
    GMCP_CUDA(cudaEventRecord(e1, c.stream));
    GMCP_CUDA(cudaEventSynchronize(e1));
    float ms;
    GMCP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    tot += ms;
  }
  // dominant kernel alone (K7 run partials), same conditions
  AssemblyPlan& P = c.plan;
  const DevSamples S = c.samples();
  const int rb = (int)std::max<int64_t>(1, std::min<int64_t>((P.n_runs + kRunWarps - 1) / kRunWarps, 148 * 16));
  for (int it = 0; it < reps; ++it) {
    if (nflush) {
      k_flush<<<148 * 8, 256, 0, c.stream>>>(flush.p, nflush);
      ++c.launches;
    }
    GMCP_CUDA(cudaEventRecord(k0, c.stream));
    k_run_partials<true><<<rb, 32 * kRunWarps, 0, c.stream>>>(S, c.X(), P.n_runs, P.run_off.p, P.run_slave.p,
                                                              P.lm_off.p, P.lm_ids.p, P.lp_off.p, P.lp.p,
                                                              P.pbase.p, P.partial.p, c.red_u.p);
    ++c.launches;
    GMCP_CUDA(cudaEventRecord(k1, c.stream));
    GMCP_CUDA(cudaEventSynchronize(k1));
    float ms;
    GMCP_CUDA(cudaEventElapsedTime(&ms, k0, k1));
    totk += ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(k0);
  cudaEventDestroy(k1);
  *ms_pass = tot / reps;
  *ms_kernel = totk / reps;
}

}  // namespace gmcp_b200
