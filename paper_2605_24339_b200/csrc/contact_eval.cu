// Per-iteration contact assembly (host side): derived sample fields, the
// per-rebuild assembly plan, and launches of K7/K8 (assembly.cuh). Energy,
// gradient and Gauss-Newton Hessian blocks are assembled into BCSR with no
// floating-point atomics: results are bitwise reproducible run to run.
//
// Reference: proj/include/gmcp/contact_energy.hpp:126-179 (add_contact_gradient,
// add_contact_gradient_hessian) and solver.hpp:315-344 (assembly into the
// sparse Newton matrix).
#include <algorithm>
#include <numeric>

#include "assembly.cuh"
#include "cubutil.cuh"

namespace gmcp_b200 {

namespace {

int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}


// K7 warps write their run-energy sums at red_d[kWarpE + warp]
constexpr int kWarpE = kRedBlocks + 8;

int launch_k7(Ctx& c, int mode) {
  AssemblyPlan& P = c.plan;
  const DevSamples S = c.samples();
  int& resident = c.k7_resident;  // persistent grid: resident blocks on all SMs of c's device
  if (!resident) {
    int occ = 0, dev = 0, sms = 148;
    GMCP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_run_partials<true>, 32 * kRunWarps, 0));
    GMCP_CUDA(cudaGetDevice(&dev));
    GMCP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    resident = std::max(1, occ) * sms;
  }
  const int64_t blocks = (P.n_runs + kRunWarps - 1) / kRunWarps;
  const int gb = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, resident));
  c.red_d.resize(kWarpE + (int64_t)gb * kRunWarps);
  double* we = c.red_d.p + kWarpE;
  if (mode == 1)
    k_run_partials<true><<<gb, 32 * kRunWarps, 0, c.stream>>>(S, c.X(), P.n_runs, P.run_off.p, P.run_slave.p,
                                                              P.lm_off.p, P.li4.p, P.pbase.p,
                                                              P.partial.p, c.red_u.p, we);
  else
    k_run_partials<false><<<gb, 32 * kRunWarps, 0, c.stream>>>(S, c.X(), P.n_runs, P.run_off.p, P.run_slave.p,
                                                               P.lm_off.p, P.li4.p, P.pbase.p,
                                                               P.partial.p, c.red_u.p, we);
  ++c.launches;
  return gb * kRunWarps;
}

// energy of the pass -> red_d[kRedBlocks]: the K7 warps' sums in warp order
// (each warp summed its runs in its own, fixed, run order)
void launch_energy_sum(Ctx& c, int k7_warps) {
  launch_pdl(k_sum_parts, 1, kRedThreads, c.stream, (const double*)(c.red_d.p + kWarpE), k7_warps, 1,
             c.red_d.p + kRedBlocks);
  c.launches += 1;
}

void launch_k8(Ctx& c, int mode) {
  AssemblyPlan& P = c.plan;
  const int64_t items = (mode == 1 ? P.nnzb : 0) + P.n_rows;
  const int gb = grid_for(items, kGatherThreads);
  if (mode == 1)
    launch_pdl(k_gather<true>, gb, kGatherThreads, c.stream, P.nnzb, P.n_rows, P.blk_off.p, P.contrib.p,
               P.vals.p, P.row_ent_off.p, P.row_ent.p, P.partial.p, c.grad.p);
  else
    launch_pdl(k_gather<false>, gb, kGatherThreads, c.stream, P.nnzb, P.n_rows, P.blk_off.p, P.contrib.p,
               P.vals.p, P.row_ent_off.p, P.row_ent.p, P.partial.p, c.grad.p);
  ++c.launches;
}

void launch_assembly(Ctx& c, int mode) {
  const int w = launch_k7(c, mode);
  launch_k8(c, mode);
  launch_energy_sum(c, w);
  GMCP_CUDA(cudaGetLastError());
}

}  // namespace

// ===========================================================================
// host entry points

__global__ void k_face_flags(int64_t n, const int8_t* __restrict__ type, int64_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = type[i] == GMCP_FACE ? 1 : 0;
}
__global__ void k_face_scatter(int64_t n, const int64_t* __restrict__ flag, const int64_t* __restrict__ pos,
                               int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[pos[i]] = i;
}

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
  // face sample index list (pressure-field order): flags, scan, scatter
  c.face_flag.resize(n + 1);
  c.face_pos.resize(n + 1);
  int64_t nf = 0;
  if (n) {
    k_face_flags<<<grid_for(n, 256), 256, 0, c.stream>>>(n, c.s_type.p, c.face_flag.p);
    GMCP_CUDA(cudaMemsetAsync(c.face_flag.p + n, 0, sizeof(int64_t), c.stream));
    exclusive_scan(c.face_flag.p, c.face_pos.p, n + 1, c.stream);
    GMCP_CUDA(cudaMemcpyAsync(&nf, c.face_pos.p + n, sizeof nf, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
  }
  c.face_idx.resize(std::max<int64_t>(nf, 1));
  if (nf) {
    k_face_scatter<<<grid_for(n, 256), 256, 0, c.stream>>>(n, c.face_flag.p, c.face_pos.p, c.face_idx.p);
    c.launches += 2;
  }
  c.face_idx.n = nf;
  c.plan.valid = false;
}

struct SampleRefs {
  int8_t* type;
  int32_t *slave, *master;
  double *beta_s, *beta_m, *eta, *weight, *gamma, *eps, *gref;
};
__device__ __forceinline__ void copy_sample(const SampleRefs& a, int64_t i, const SampleRefs& b, int64_t j) {
  a.type[i] = b.type[j];
  for (int k = 0; k < 3; ++k) {
    a.slave[3 * i + k] = b.slave[3 * j + k];
    a.master[3 * i + k] = b.master[3 * j + k];
    a.beta_s[3 * i + k] = b.beta_s[3 * j + k];
    a.beta_m[3 * i + k] = b.beta_m[3 * j + k];
  }
  a.eta[i] = b.eta[j];
  a.weight[i] = b.weight[j];
  a.gamma[i] = b.gamma[j];
  a.eps[i] = b.eps[j];
  a.gref[i] = b.gref[j];
}
__global__ void k_snapshot(int64_t n, SampleRefs dst, SampleRefs src) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    copy_sample(dst, i, src, i);
}
// out sample i of scene s (merged offsets moff) comes from the new arrays at
// soff_new[s] + k or the snapshot at soff_old[s] + k
__global__ void k_splice(int64_t n, int ns, const int64_t* __restrict__ moff, const int64_t* __restrict__ soff_old,
                         const int64_t* __restrict__ soff_new, const uint8_t* __restrict__ take, SampleRefs out,
                         SampleRefs fresh, SampleRefs old) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = ns;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (moff[mid] <= i) lo = mid; else hi = mid;
    }
    const int64_t k = i - moff[lo];
    if (take[lo]) copy_sample(out, i, fresh, soff_new[lo] + k);
    else copy_sample(out, i, old, soff_old[lo] + k);
  }
}

__global__ void k_add_into(int64_t n, double* __restrict__ dst, const double* __restrict__ src) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = dst[i] + src[i];
}

void add_into(Ctx& c, double* dst, const double* src, int64_t n) {
  if (n <= 0) return;
  k_add_into<<<grid_for(n, 256), 256, 0, c.stream>>>(n, dst, src);
  ++c.launches;
}

static SampleRefs refs_of(Ctx& c) {
  return SampleRefs{c.s_type.p, c.s_slave.p, c.s_master.p, c.s_beta_s.p, c.s_beta_m.p, c.s_eta.p,
                    c.s_weight.p, c.s_gamma.p, c.s_eps.p, c.s_gref.p};
}
static SampleRefs refs_of(Ctx::Snapshot& a) {
  return SampleRefs{a.type.p, a.slave.p, a.master.p, a.beta_s.p, a.beta_m.p, a.eta.p,
                    a.weight.p, a.gamma.p, a.eps.p, a.gref.p};
}
static void size_snapshot(Ctx::Snapshot& a, int64_t n) {
  const int64_t m = std::max<int64_t>(n, 1);
  a.type.resize(m);
  a.slave.resize(3 * m);
  a.master.resize(3 * m);
  a.beta_s.resize(3 * m);
  a.beta_m.resize(3 * m);
  for (auto* b : {&a.eta, &a.weight, &a.gamma, &a.eps, &a.gref}) b->resize(m);
}

void snapshot_samples(Ctx& c) {
  size_snapshot(c.snap, c.ns);
  c.snap.ns = c.ns;
  if (c.ns) {
    k_snapshot<<<grid_for(c.ns, 256), 256, 0, c.stream>>>(c.ns, refs_of(c.snap), refs_of(c));
    ++c.launches;
  }
}

void splice_samples(Ctx& c, const std::vector<int64_t>& soff_old, const std::vector<int64_t>& soff_new,
                    const std::vector<uint8_t>& take_new, std::vector<int64_t>& soff_out) {
  const int ns = (int)take_new.size();
  soff_out.assign(ns + 1, 0);
  for (int s = 0; s < ns; ++s)
    soff_out[s + 1] = soff_out[s] + (take_new[s] ? soff_new[s + 1] - soff_new[s] : soff_old[s + 1] - soff_old[s]);
  const int64_t n = soff_out[ns];
  Ctx::Snapshot& merged = c.spliced;
  size_snapshot(merged, n);
  DBuf<int64_t> moff, so, sn;
  DBuf<uint8_t> take;
  moff.upload(soff_out, c.stream);
  so.upload(soff_old, c.stream);
  sn.upload(soff_new, c.stream);
  take.upload(take_new, c.stream);
  if (n) {
    k_splice<<<grid_for(n, 256), 256, 0, c.stream>>>(n, ns, moff.p, so.p, sn.p, take.p, refs_of(merged), refs_of(c),
                                                      refs_of(c.snap));
    ++c.launches;
  }
  // merged -> c's arrays
  c.s_type.swap(merged.type);
  c.s_slave.swap(merged.slave);
  c.s_master.swap(merged.master);
  c.s_beta_s.swap(merged.beta_s);
  c.s_beta_m.swap(merged.beta_m);
  c.s_eta.swap(merged.eta);
  c.s_weight.swap(merged.weight);
  c.s_gamma.swap(merged.gamma);
  c.s_eps.swap(merged.eps);
  c.s_gref.swap(merged.gref);
  c.ns = n;
  derive_sample_fields(c);  // c.spliced now holds the previous arrays (reused next time)
}

double run_assembly(Ctx& c, int mode, int64_t* bad) {
  const NvtxRange nvtx_("gmcp:K6-K8 assembly");
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
    *bad = first_bad;  // contact_energy.hpp:132-135
    throw StatusError(GMCP_ERR_INFEASIBLE, "contact sample " + std::to_string(first_bad) + " has non-positive gap",
                      first_bad);
  }
  return e;
}

__global__ void k_add3(int64_t n, double* __restrict__ dst, const double* __restrict__ a, const double* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = a[i] + b[i];
}

double run_assembly_host(Ctx& c, int mode, const double* x, double* grad, int64_t* bad) {
  const NvtxRange nvtx_("gmcp:K6-K8 assembly (host buffers)");
  *bad = -1;
  const int64_t n = c.n_dof;
  c.ensure_aux();
  c.x.upload(x, n, c.stream);
  if (!c.plan.valid) build_assembly_plan(c);
  c.grad.resize(std::max<int64_t>(n, 1));
  c.red_d.resize(kRedBlocks + 8);
  reset_red(c);
  if (grad) {  // behind x on the copy engine, overlapping K7
    c.grad_in.resize(std::max<int64_t>(n, 1));
    c.grad_sum.resize(std::max<int64_t>(n, 1));
    GMCP_CUDA(cudaEventRecord(c.x_ready, c.stream));
    GMCP_CUDA(cudaStreamWaitEvent(c.aux, c.x_ready, 0));
    GMCP_CUDA(cudaMemcpyAsync(c.grad_in.p, grad, n * sizeof(double), cudaMemcpyHostToDevice, c.aux));
  }
  unsigned long long u[4] = {~0ull, ~0ull, ~0ull, ~0ull};
  double e = 0.0;
  if (c.ns == 0) {
    c.grad.zero(c.stream);
    if (mode == 1 && c.plan.nnzb) GMCP_CUDA(cudaMemsetAsync(c.plan.vals.p, 0, 9 * c.plan.nnzb * sizeof(double), c.stream));
    GMCP_CUDA(cudaEventRecord(c.rows_done, c.stream));
  } else {
    AssemblyPlan& P = c.plan;
    const int w = launch_k7(c, mode);
    // gradient rows first: grad + g_c goes down while the blocks are gathered
    launch_pdl(k_gather<false>, grid_for(P.n_rows, kGatherThreads), kGatherThreads, c.stream, P.nnzb, P.n_rows,
               P.blk_off.p, P.contrib.p, P.vals.p, P.row_ent_off.p, P.row_ent.p, P.partial.p,
               c.grad.p);
    GMCP_CUDA(cudaEventRecord(c.rows_done, c.stream));
    if (mode == 1)
      k_gather<true, false><<<grid_for(P.nnzb, kGatherThreads), kGatherThreads, 0, c.stream>>>(
          P.nnzb, P.n_rows, P.blk_off.p, P.contrib.p, P.vals.p, P.row_ent_off.p, P.row_ent.p,
          P.partial.p, c.grad.p);
    launch_energy_sum(c, w);
    c.launches += 2 + (mode == 1);
  }
  if (grad) {
    GMCP_CUDA(cudaStreamWaitEvent(c.aux, c.rows_done, 0));
    k_add3<<<grid_for(n, 256), 256, 0, c.aux>>>(n, c.grad_sum.p, c.grad_in.p, c.grad.p);
    ++c.launches;
    GMCP_CUDA(cudaMemcpyAsync(grad, c.grad_sum.p, n * sizeof(double), cudaMemcpyDeviceToHost, c.aux));
  }
  unsigned long long* hu = static_cast<unsigned long long*>(c.host_scalars);  // pinned
  double* he = reinterpret_cast<double*>(hu + 4);
  if (c.ns) {
    GMCP_CUDA(cudaMemcpyAsync(hu, c.red_u.p, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream));
    GMCP_CUDA(cudaMemcpyAsync(he, c.red_d.p + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  }
  c.sync();
  if (grad) GMCP_CUDA(cudaStreamSynchronize(c.aux));
  if (c.ns) {
    for (int k = 0; k < 4; ++k) u[k] = hu[k];
    e = *he;
  }
  GMCP_CUDA(cudaGetLastError());
  const int64_t first_bad = u[0] == ~0ull ? -1 : (int64_t)u[0];
  const int64_t first_deg = u[1] == ~0ull ? -1 : (int64_t)u[1];
  const bool fail = first_bad >= 0 || first_deg >= 0;
  if (fail && grad) {  // the caller's gradient is left as it was
    GMCP_CUDA(cudaMemcpyAsync(grad, c.grad_in.p, n * sizeof(double), cudaMemcpyDeviceToHost, c.aux));
    GMCP_CUDA(cudaStreamSynchronize(c.aux));
  }
  if (first_deg >= 0 && (first_bad < 0 || first_deg < first_bad))
    throw StatusError(GMCP_ERR_DEGENERATE, "contact sample on a degenerate slave triangle", first_deg);
  if (first_bad >= 0) {
    *bad = first_bad;  // contact_energy.hpp:132-135
    throw StatusError(GMCP_ERR_INFEASIBLE, "contact sample " + std::to_string(first_bad) + " has non-positive gap",
                      first_bad);
  }
  return e;
}

void time_assembly(Ctx& c, int reps, int flush_l2, double* ms_pass, double* ms_kernel) {
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
  // dominant kernel alone (K7), same conditions
  for (int it = 0; it < reps; ++it) {
    if (nflush) {
      k_flush<<<148 * 8, 256, 0, c.stream>>>(flush.p, nflush);
      ++c.launches;
    }
    GMCP_CUDA(cudaEventRecord(k0, c.stream));
    launch_k7(c, 1);
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
