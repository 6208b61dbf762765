// Bit-exact kernels (compiled with -fmad=false): energy / feasibility (K6),
// step-size filter (K10), displacement cap, pressure field (K12), force
// summary and kinematics. Min/max reductions are order-free, and every
// per-sample value follows the reference's IEEE operation order, so the
// returned alpha equals the reference's bitwise.
//
// Reference: proj/include/gmcp/contact_energy.hpp:184-213.
#include "ctx.hpp"
#include "kin.cuh"
#include "reduce.cuh"

namespace gmcp_b200 {

namespace {

// ---------------------------------------------------------------------------
// K6: energy / feasibility (try_contact_energy, contact_energy)
// red_u[0] = first non-positive gap index, red_u[1] = first degenerate index,
// red_u[2] = ord_bits(min gap). Samples i >= limit are skipped.

__global__ void __launch_bounds__(kRedThreads, 4) k_energy(DevSamples S, const double* __restrict__ x, int64_t limit,
                                                         double* __restrict__ parts, unsigned long long* red) {
  __shared__ double sh[kRedThreads / 32];
  double e = 0;
  double mg = 1.7976931348623157e308;
  unsigned long long bad = ~0ull, deg = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < limit; i += (int64_t)gridDim.x * blockDim.x) {
    double g;
    if (!sample_gap(S, i, x, g)) {
      deg = min(deg, (unsigned long long)i);
      continue;
    }
    mg = dmin(mg, g);
    if (!(g > 0)) {
      bad = min(bad, (unsigned long long)i);
      continue;
    }
    double B, dB, ddB;
    barrier_eval(g, S.eps[i], B, dB, ddB);
    e += S.coef[i] * B;
  }
  const double r = block_sum<kRedThreads>(e, sh);
  if (threadIdx.x == 0) parts[blockIdx.x] = r;
  if (bad != ~0ull) atomicMin(&red[0], bad);
  if (deg != ~0ull) atomicMin(&red[1], deg);
  atomicMin(&red[2], ord_bits(mg));
}

// ---------------------------------------------------------------------------
// pressure field, force summary, kinematics

__global__ void k_pressure(DevSamples S, const double* __restrict__ x, int64_t nf, const int64_t* __restrict__ fidx,
                           double kappa_face, gmcp_pressure_record* __restrict__ out, unsigned long long* red) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nf; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = fidx[j];
    Kin k;
    gmcp_pressure_record rec;
    rec.sample = i;
    if (!kinematics<false>(S, i, x, k)) {
      atomicMin(&red[1], (unsigned long long)i);
      continue;
    }
    if (!(k.g > 0)) {
      atomicMin(&red[0], (unsigned long long)i);
      continue;
    }
    double B, dB, ddB;
    barrier_eval(k.g, S.eps[i], B, dB, ddB);
    rec.position[0] = k.xs.x;
    rec.position[1] = k.xs.y;
    rec.position[2] = k.xs.z;
    rec.radius = hypot(k.xs.x, k.xs.y);
    rec.gap = k.g;
    rec.pressure = kappa_face * S.gamma[i] * (-dB);
    out[j] = rec;
  }
}

__global__ void __launch_bounds__(kRedThreads) k_force(DevSamples S, const double* __restrict__ x,
                                                        double* __restrict__ parts, unsigned long long* red) {
  __shared__ double sh[kRedThreads / 32];
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S.n; i += (int64_t)gridDim.x * blockDim.x) {
    Kin k;
    if (!kinematics<true>(S, i, x, k)) {
      atomicMin(&red[1], (unsigned long long)i);
      continue;
    }
    if (!(k.g > 0)) continue;
    double B, dB, ddB;
    barrier_eval(k.g, S.eps[i], B, dB, ddB);
    const double f = S.coef[i] * dB;
    d3 F = mk3(0, 0, 0);
    for (int v = 0; v < 3; ++v) F = F - f * k.dg[v];
    const int t = S.type[i] == GMCP_FACE ? 0 : (S.type[i] == GMCP_EDGE ? 1 : 2);
    acc[3 * t] += F.x;
    acc[3 * t + 1] += F.y;
    acc[3 * t + 2] += F.z;
  }
  for (int q = 0; q < 9; ++q) {
    const double v = block_sum<kRedThreads>(acc[q], sh);
    if (threadIdx.x == 0) parts[(int64_t)blockIdx.x * 9 + q] = v;
  }
}

__global__ void k_kinematics(DevSamples S, const double* __restrict__ x, double* g, int32_t* nv, int32_t* ids,
                             double* dg, unsigned long long* red) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S.n; i += (int64_t)gridDim.x * blockDim.x) {
    Kin k;
    if (!kinematics<true>(S, i, x, k)) {
      atomicMin(&red[1], (unsigned long long)i);
      continue;
    }
    g[i] = k.g;
    nv[i] = k.nv;
    for (int v = 0; v < 6; ++v) {
      int id = -1;
      if (v < 3) id = S.slave[3 * i + v];
      else if (v < k.nv) id = S.master[3 * i + v - 3];
      ids[6 * i + v] = id;
      dg[18 * i + 3 * v] = v < k.nv ? k.dg[v].x : 0.0;
      dg[18 * i + 3 * v + 1] = v < k.nv ? k.dg[v].y : 0.0;
      dg[18 * i + 3 * v + 2] = v < k.nv ? k.dg[v].z : 0.0;
    }
  }
}


// red[0] = ord_bits(alpha), red[1] = first degenerate index
__global__ void __launch_bounds__(256, 3) k_step_filter(DevSamples S, const double* __restrict__ x, const double* __restrict__ dx,
                              unsigned long long* red) {
  unsigned long long best = ord_bits(1.0), deg = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S.n; i += (int64_t)gridDim.x * blockDim.x) {
    Kin k;
    if (!kinematics<true>(S, i, x, k)) {
      deg = min(deg, (unsigned long long)i);
      continue;
    }
    double dgdx = 0;
    for (int v = 0; v < k.nv; ++v) {
      const int id = v < 3 ? S.slave[3 * i + v] : S.master[3 * i + v - 3];
      dgdx += dot(k.dg[v], ld3(dx, id));
    }
    if (dgdx < 0) {
      const unsigned long long b = ord_bits(0.9 * k.g / (-dgdx));
      best = b < best ? b : best;
    }
  }
  // warp-level pre-reduction keeps atomics at one per warp
  for (int o = 16; o > 0; o >>= 1) {
    best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    deg = min(deg, __shfl_xor_sync(0xffffffffu, deg, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&red[0], best);
    if (deg != ~0ull) atomicMin(&red[1], deg);
  }
}

// red[2] = first sample with g < eps, red[1] = first degenerate, red[3] = ord_bits(max |dx_v|)
__global__ void k_cap_active(DevSamples S, const double* __restrict__ x, unsigned long long* red) {
  unsigned long long act = ~0ull, deg = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S.n; i += (int64_t)gridDim.x * blockDim.x) {
    double g;
    if (!sample_gap(S, i, x, g)) {
      deg = min(deg, (unsigned long long)i);
      continue;
    }
    if (g < S.eps[i]) act = min(act, (unsigned long long)i);
  }
  for (int o = 16; o > 0; o >>= 1) {
    act = min(act, __shfl_xor_sync(0xffffffffu, act, o));
    deg = min(deg, __shfl_xor_sync(0xffffffffu, deg, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (act != ~0ull) atomicMin(&red[2], act);
    if (deg != ~0ull) atomicMin(&red[1], deg);
  }
}

__global__ void k_max_move(int64_t nv, const double* __restrict__ dx, unsigned long long* red) {
  unsigned long long best = ord_bits(0.0);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long b = ord_bits(norm(ld3(dx, (int)v)));
    best = b > best ? b : best;
  }
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&red[3], best);
}

// ---------------------------------------------------------------------------
// Scene-segmented variants (batched scenes): one block per scene
// over its contiguous sample range, per-sample arithmetic identical to K6 /
// K10 / the cap, block reductions in a fixed order (sums) or order-free
// (mins / maxes): deterministic.

constexpr int kSceneThreads = 256;

__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v, unsigned long long* sh) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long r = sh[0];
  for (int i = 1; i < kSceneThreads / 32; ++i) r = min(r, sh[i]);
  return r;
}
__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v, unsigned long long* sh) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long r = sh[0];
  for (int i = 1; i < kSceneThreads / 32; ++i) r = max(r, sh[i]);
  return r;
}

// u[4 s + 0] first non-positive gap, [1] first degenerate, [2] ord_bits(min gap)
__global__ void __launch_bounds__(kSceneThreads) k_scene_energy(DevSamples S, const double* __restrict__ x,
                                                                const int64_t* __restrict__ soff,
                                                                double* __restrict__ e, unsigned long long* u) {
  __shared__ double shd[kSceneThreads / 32];
  __shared__ unsigned long long shu[kSceneThreads / 32];
  const int sc = blockIdx.x;
  double acc = 0;
  double mg = 1.7976931348623157e308;
  unsigned long long bad = ~0ull, deg = ~0ull;
  for (int64_t i = soff[sc] + threadIdx.x; i < soff[sc + 1]; i += kSceneThreads) {
    double g;
    if (!sample_gap(S, i, x, g)) {
      deg = min(deg, (unsigned long long)i);
      continue;
    }
    mg = dmin(mg, g);
    if (!(g > 0)) {
      bad = min(bad, (unsigned long long)i);
      continue;
    }
    double B, dB, ddB;
    barrier_eval(g, S.eps[i], B, dB, ddB);
    acc += S.coef[i] * B;
  }
  const double r = block_sum<kSceneThreads>(acc, shd);
  const unsigned long long b = block_min_u64(bad, shu), d = block_min_u64(deg, shu), m = block_min_u64(ord_bits(mg), shu);
  if (threadIdx.x == 0) {
    e[sc] = r;
    u[4 * sc] = b;
    u[4 * sc + 1] = d;
    u[4 * sc + 2] = m;
  }
}

// per scene: u[4 s] ord_bits(filter alpha), [1] first degenerate, [2] first
// sample with g < eps (cap active), [3] ord_bits(max |dx_v| over the scene)
__global__ void __launch_bounds__(kSceneThreads) k_scene_alpha(DevSamples S, const double* __restrict__ x,
                                                               const double* __restrict__ dx,
                                                               const int64_t* __restrict__ soff,
                                                               const int64_t* __restrict__ voff,
                                                               unsigned long long* u) {
  __shared__ unsigned long long shu[kSceneThreads / 32];
  const int sc = blockIdx.x;
  unsigned long long best = ord_bits(1.0), deg = ~0ull, act = ~0ull, mv = ord_bits(0.0);
  for (int64_t i = soff[sc] + threadIdx.x; i < soff[sc + 1]; i += kSceneThreads) {
    Kin k;
    if (!kinematics<true>(S, i, x, k)) {
      deg = min(deg, (unsigned long long)i);
      continue;
    }
    if (k.g < S.eps[i]) act = min(act, (unsigned long long)i);
    double dgdx = 0;
    for (int v = 0; v < k.nv; ++v) {
      const int id = v < 3 ? S.slave[3 * i + v] : S.master[3 * i + v - 3];
      dgdx += dot(k.dg[v], ld3(dx, id));
    }
    if (dgdx < 0) {
      const unsigned long long b = ord_bits(0.9 * k.g / (-dgdx));
      best = b < best ? b : best;
    }
  }
  for (int64_t v = voff[sc] + threadIdx.x; v < voff[sc + 1]; v += kSceneThreads) {
    const unsigned long long b = ord_bits(norm(ld3(dx, (int)v)));
    mv = b > mv ? b : mv;
  }
  const unsigned long long a = block_min_u64(best, shu), d = block_min_u64(deg, shu), c = block_min_u64(act, shu),
                           m = block_max_u64(mv, shu);
  if (threadIdx.x == 0) {
    u[4 * sc] = a;
    u[4 * sc + 1] = d;
    u[4 * sc + 2] = c;
    u[4 * sc + 3] = m;
  }
}

// samples per scene (scene of a sample = scene of its first slave vertex)
__global__ void k_scene_count(DevSamples S, const int32_t* __restrict__ vscene, int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S.n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[vscene[S.slave[3 * i]]], 1);  // integer counts: order-free
}

int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

}  // namespace

EnergyOut run_energy(Ctx& c, bool need_prefix_min) {
  const NvtxRange nvtx_("gmcp:K6 energy");
  EnergyOut o{0, 1.7976931348623157e308, 1.7976931348623157e308, -1, -1};
  reset_red(c);
  c.red_d.resize(kRedBlocks + 8);
  const DevSamples S = c.samples();
  if (S.n == 0) return o;
  k_energy<<<kRedBlocks, kRedThreads, 0, c.stream>>>(S, c.X(), S.n, c.red_d.p, c.red_u.p);
  k_sum_parts<<<1, kRedThreads, 0, c.stream>>>(c.red_d.p, kRedBlocks, 1, c.red_d.p + kRedBlocks);
  c.launches += 2;
  GMCP_CUDA(cudaGetLastError());
  unsigned long long u[4];
  double e;
  GMCP_CUDA(cudaMemcpyAsync(u, c.red_u.p, sizeof u, cudaMemcpyDeviceToHost, c.stream));
  GMCP_CUDA(cudaMemcpyAsync(&e, c.red_d.p + kRedBlocks, sizeof e, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  o.energy = e;
  o.first_bad = u[0] == ~0ull ? -1 : (int64_t)u[0];
  o.first_degenerate = u[1] == ~0ull ? -1 : (int64_t)u[1];
  o.min_gap = from_ord_bits(u[2]);
  o.min_gap_prefix = o.min_gap;
  if (o.first_bad >= 0 && need_prefix_min) {
    // try_contact_energy stops at the first offending sample: its energy and
    // min gap cover samples [0, first_bad] only (contact_energy.hpp:98-104).
    reset_red(c);
    k_energy<<<kRedBlocks, kRedThreads, 0, c.stream>>>(S, c.X(), o.first_bad + 1, c.red_d.p, c.red_u.p);
    k_sum_parts<<<1, kRedThreads, 0, c.stream>>>(c.red_d.p, kRedBlocks, 1, c.red_d.p + kRedBlocks);
    c.launches += 2;
    GMCP_CUDA(cudaGetLastError());
    GMCP_CUDA(cudaMemcpyAsync(u, c.red_u.p, sizeof u, cudaMemcpyDeviceToHost, c.stream));
    GMCP_CUDA(cudaMemcpyAsync(&e, c.red_d.p + kRedBlocks, sizeof e, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    o.energy = e;
    o.min_gap_prefix = from_ord_bits(u[2]);
  }
  return o;
}

void run_pressure(Ctx& c, gmcp_pressure_record* out_host) {
  const NvtxRange nvtx_("gmcp:pressure field");
  const int64_t nf = (int64_t)c.face_idx.n;
  if (nf == 0) return;
  DBuf<gmcp_pressure_record> out;
  out.resize(nf);
  reset_red(c);
  k_pressure<<<grid_for(nf, 256), 256, 0, c.stream>>>(c.samples(), c.X(), nf, c.face_idx.p, c.params.kappa_face,
                                                      out.p, c.red_u.p);
  ++c.launches;
  GMCP_CUDA(cudaGetLastError());
  unsigned long long u[4];
  GMCP_CUDA(cudaMemcpyAsync(u, c.red_u.p, sizeof u, cudaMemcpyDeviceToHost, c.stream));
  out.download(out_host, nf, c.stream);
  c.sync();
  const int64_t bad = u[0] == ~0ull ? -1 : (int64_t)u[0], deg = u[1] == ~0ull ? -1 : (int64_t)u[1];
  if (deg >= 0 && (bad < 0 || deg < bad))
    throw StatusError(GMCP_ERR_DEGENERATE, "contact sample on a degenerate slave triangle", deg);
  if (bad >= 0) throw StatusError(GMCP_ERR_INFEASIBLE, "barrier: non-positive gap", bad);
}

void run_force_summary(Ctx& c, double* out12) {
  c.red_d.resize(9 * kRedBlocks + 16);
  reset_red(c);
  if (c.ns == 0) {
    for (int q = 0; q < 12; ++q) out12[q] = 0;
    return;
  }
  k_force<<<kRedBlocks, kRedThreads, 0, c.stream>>>(c.samples(), c.X(), c.red_d.p, c.red_u.p);
  k_sum_parts<<<1, kRedThreads, 0, c.stream>>>(c.red_d.p, kRedBlocks, 9, c.red_d.p + 9 * kRedBlocks);
  c.launches += 2;
  GMCP_CUDA(cudaGetLastError());
  double v[9];
  unsigned long long u[4];
  GMCP_CUDA(cudaMemcpyAsync(v, c.red_d.p + 9 * kRedBlocks, sizeof v, cudaMemcpyDeviceToHost, c.stream));
  GMCP_CUDA(cudaMemcpyAsync(u, c.red_u.p, sizeof u, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (u[1] != ~0ull) throw StatusError(GMCP_ERR_DEGENERATE, "contact sample on a degenerate slave triangle");
  for (int q = 0; q < 9; ++q) out12[q] = v[q];
  for (int k = 0; k < 3; ++k) out12[9 + k] = (v[k] + v[3 + k]) + v[6 + k];
}

void run_kinematics(Ctx& c, double* g, int32_t* nv, int32_t* ids, double* dg) {
  const int64_t n = c.ns;
  if (n == 0) return;
  DBuf<double> dgd, gd;
  DBuf<int32_t> nvd, idd;
  gd.resize(n);
  dgd.resize(18 * n);
  nvd.resize(n);
  idd.resize(6 * n);
  reset_red(c);
  k_kinematics<<<grid_for(n, 256), 256, 0, c.stream>>>(c.samples(), c.X(), gd.p, nvd.p, idd.p, dgd.p, c.red_u.p);
  ++c.launches;
  GMCP_CUDA(cudaGetLastError());
  unsigned long long u[4];
  GMCP_CUDA(cudaMemcpyAsync(u, c.red_u.p, sizeof u, cudaMemcpyDeviceToHost, c.stream));
  gd.download(g, n, c.stream);
  dgd.download(dg, 18 * n, c.stream);
  nvd.download(nv, n, c.stream);
  idd.download(ids, 6 * n, c.stream);
  c.sync();
  if (u[1] != ~0ull) throw StatusError(GMCP_ERR_DEGENERATE, "contact sample on a degenerate slave triangle");
}


double run_step_filter(Ctx& c) {
  const NvtxRange nvtx_("gmcp:K10 step filter");
  if (c.ns == 0) return 1.0;
  c.red_u.resize(4);
  const unsigned long long init[4] = {ord_bits_host(1.0), ~0ull, ~0ull, 0ull};
  GMCP_CUDA(cudaMemcpyAsync(c.red_u.p, init, sizeof init, cudaMemcpyHostToDevice, c.stream));
  k_step_filter<<<grid_for(c.ns, 256), 256, 0, c.stream>>>(c.samples(), c.X(), c.DX(), c.red_u.p);
  ++c.launches;
  GMCP_CUDA(cudaGetLastError());
  unsigned long long u[4];
  GMCP_CUDA(cudaMemcpyAsync(u, c.red_u.p, sizeof u, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (u[1] != ~0ull) throw StatusError(GMCP_ERR_DEGENERATE, "contact sample on a degenerate slave triangle", (int64_t)u[1]);
  return from_ord_bits(u[0]);
}

double run_displacement_cap(Ctx& c) {
  const NvtxRange nvtx_("gmcp:K10 displacement cap");
  c.red_u.resize(4);
  const unsigned long long init[4] = {0ull, ~0ull, ~0ull, ord_bits_host(0.0)};
  GMCP_CUDA(cudaMemcpyAsync(c.red_u.p, init, sizeof init, cudaMemcpyHostToDevice, c.stream));
  if (c.ns) {
    k_cap_active<<<grid_for(c.ns, 256), 256, 0, c.stream>>>(c.samples(), c.X(), c.red_u.p);
    ++c.launches;
  }
  const int64_t nv = c.n_vertices();
  if (nv) {
    k_max_move<<<grid_for(nv, 256), 256, 0, c.stream>>>(nv, c.DX(), c.red_u.p);
    ++c.launches;
  }
  GMCP_CUDA(cudaGetLastError());
  unsigned long long u[4];
  GMCP_CUDA(cudaMemcpyAsync(u, c.red_u.p, sizeof u, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  const int64_t act = u[2] == ~0ull ? -1 : (int64_t)u[2], deg = u[1] == ~0ull ? -1 : (int64_t)u[1];
  if (deg >= 0 && (act < 0 || deg < act))
    throw StatusError(GMCP_ERR_DEGENERATE, "triangle_normal: degenerate triangle (area below cutoff)", deg);
  if (act < 0) return 1.0;
  const double max_move = from_ord_bits(u[3]);
  if (max_move <= 0.5 * c.params.eps_max) return 1.0;
  return 0.5 * c.params.eps_max / max_move;
}

// ===========================================================================
// scene-segmented host entry points (batched System solve)

struct SceneTmp : TmpBase {
  DBuf<double> e;
  DBuf<unsigned long long> u;
  DBuf<int32_t> cnt;
};
static SceneTmp& scene_tmp(Ctx& c) {
  if (!c.scene_tmp) c.scene_tmp = std::make_unique<SceneTmp>();
  return *static_cast<SceneTmp*>(c.scene_tmp.get());
}

void scene_sample_offsets(Ctx& c, const int32_t* vscene_dev, int n_scenes, std::vector<int64_t>& soff_host,
                          DBuf<int64_t>& soff_dev) {
  SceneTmp& T = scene_tmp(c);
  T.cnt.resize(n_scenes);
  T.cnt.zero(c.stream);
  if (c.ns) {
    k_scene_count<<<grid_for(c.ns, 256), 256, 0, c.stream>>>(c.samples(), vscene_dev, T.cnt.p);
    ++c.launches;
  }
  std::vector<int32_t> cnt = T.cnt.to_host(c.stream);
  soff_host.assign(n_scenes + 1, 0);
  for (int s = 0; s < n_scenes; ++s) soff_host[s + 1] = soff_host[s] + cnt[s];
  soff_dev.upload(soff_host, c.stream);
}

void run_scene_energy(Ctx& c, const double* xp, int n_scenes, const int64_t* soff_dev, double* e,
                      int64_t* first_bad, int64_t* first_deg, double* min_gap) {
  SceneTmp& T = scene_tmp(c);
  T.e.resize(n_scenes);
  T.u.resize(4 * n_scenes);
  k_scene_energy<<<n_scenes, kSceneThreads, 0, c.stream>>>(c.samples(), xp, soff_dev, T.e.p, T.u.p);
  ++c.launches;
  GMCP_CUDA(cudaGetLastError());
  std::vector<unsigned long long> u(4 * n_scenes);
  T.e.download(e, n_scenes, c.stream);
  T.u.download(u.data(), 4 * n_scenes, c.stream);
  c.sync();
  for (int s = 0; s < n_scenes; ++s) {
    first_bad[s] = u[4 * s] == ~0ull ? -1 : (int64_t)u[4 * s];
    first_deg[s] = u[4 * s + 1] == ~0ull ? -1 : (int64_t)u[4 * s + 1];
    min_gap[s] = from_ord_bits(u[4 * s + 2]);
  }
}

// alpha_s = min(1, step_filter_s, displacement_cap_s) (contact_energy.hpp:184-213 per scene)
void run_scene_alpha(Ctx& c, int n_scenes, const int64_t* soff_dev, const int64_t* voff_dev, double* alpha,
                     int64_t* first_deg) {
  SceneTmp& T = scene_tmp(c);
  T.u.resize(4 * n_scenes);
  k_scene_alpha<<<n_scenes, kSceneThreads, 0, c.stream>>>(c.samples(), c.X(), c.DX(), soff_dev, voff_dev, T.u.p);
  ++c.launches;
  GMCP_CUDA(cudaGetLastError());
  std::vector<unsigned long long> u(4 * n_scenes);
  T.u.download(u.data(), 4 * n_scenes, c.stream);
  c.sync();
  for (int s = 0; s < n_scenes; ++s) {
    double a = from_ord_bits(u[4 * s]);
    first_deg[s] = u[4 * s + 1] == ~0ull ? -1 : (int64_t)u[4 * s + 1];
    if (u[4 * s + 2] != ~0ull) {  // cap active in this scene
      const double max_move = from_ord_bits(u[4 * s + 3]);
      if (max_move > 0.5 * c.params.eps_max) a = std::min(a, 0.5 * c.params.eps_max / max_move);
    }
    alpha[s] = std::min(1.0, a);
  }
}

}  // namespace gmcp_b200
