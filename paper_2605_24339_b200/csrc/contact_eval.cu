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

namespace gmcp_b200 {

namespace {

int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

void init_kernels() {
  static bool done = false;
  if (done) return;
  init_ss_table();
  done = true;
}

void launch_k7(Ctx& c, int mode) {
  AssemblyPlan& P = c.plan;
  const DevSamples S = c.samples();
  static int resident = 0;  // persistent grid: resident blocks on all SMs
  if (!resident) {
    int occ = 0, dev = 0, sms = 148;
    GMCP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_run_partials<true>, 32 * kRunWarps, 0));
    GMCP_CUDA(cudaGetDevice(&dev));
    GMCP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    resident = std::max(1, occ) * sms;
  }
  const int64_t blocks = (P.n_runs + kRunWarps - 1) / kRunWarps;
  const int gb = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, resident));
  if (mode == 1)
    k_run_partials<true><<<gb, 32 * kRunWarps, 0, c.stream>>>(S, c.X(), P.n_runs, P.run_off.p, P.run_slave.p,
                                                              P.lm_off.p, P.lm_ids.p, P.li4.p, P.pbase.p,
                                                              P.partial.p, c.red_u.p);
  else
    k_run_partials<false><<<gb, 32 * kRunWarps, 0, c.stream>>>(S, c.X(), P.n_runs, P.run_off.p, P.run_slave.p,
                                                               P.lm_off.p, P.lm_ids.p, P.li4.p, P.pbase.p,
                                                               P.partial.p, c.red_u.p);
  ++c.launches;
}

void launch_k8(Ctx& c, int mode) {
  AssemblyPlan& P = c.plan;
  const int64_t items = (mode == 1 ? P.nnzb : 0) + P.n_rows;
  const int gb = grid_for(items, kGatherThreads);
  if (mode == 1)
    k_gather<true><<<gb, kGatherThreads, 0, c.stream>>>(P.nnzb, P.n_rows, P.blk_off.p, P.contrib.p, P.vals.p,
                                                        P.row_ent_off.p, P.row_ent.p, P.partial.p, c.grad.p);
  else
    k_gather<false><<<gb, kGatherThreads, 0, c.stream>>>(P.nnzb, P.n_rows, P.blk_off.p, P.contrib.p, P.vals.p,
                                                         P.row_ent_off.p, P.row_ent.p, P.partial.p, c.grad.p);
  ++c.launches;
}

void launch_assembly(Ctx& c, int mode) {
  AssemblyPlan& P = c.plan;
  launch_k7(c, mode);
  launch_k8(c, mode);
  k_run_energy<<<kRedBlocks, kRedThreads, 0, c.stream>>>(P.n_runs, P.pbase.p, P.partial.p, c.red_d.p);
  k_sum_parts<<<1, kRedThreads, 0, c.stream>>>(c.red_d.p, kRedBlocks, 1, c.red_d.p + kRedBlocks);
  c.launches += 2;
  GMCP_CUDA(cudaGetLastError());
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

// Host-side assembly plan from the device sample set (per rebuild): runs
// (consecutive samples sharing a slave triangle, split at kRunSamples samples
// or kRunMasters local masters), local master tables, incidence lists, BCSR pattern, row entries.
void build_assembly_plan(Ctx& c) {
  AssemblyPlan& P = c.plan;
  const int64_t n = c.ns;
  const std::vector<int32_t> sl = c.s_slave.to_host(c.stream);
  const std::vector<int32_t> ms = c.s_master.to_host(c.stream);
  const std::vector<int8_t> ty = c.s_type.to_host(c.stream);
  std::vector<int64_t> run_off{0};
  std::vector<int32_t> run_slave;
  std::vector<int32_t> run_masters;  // distinct master ids of the open run
  for (int64_t i = 0; i < n; ++i) {
    const bool new_tri =
        i == 0 || sl[3 * i] != sl[3 * i - 3] || sl[3 * i + 1] != sl[3 * i - 2] || sl[3 * i + 2] != sl[3 * i - 1];
    int add = 0;  // new distinct masters this sample would bring
    for (int j = 0; j < 3; ++j) {
      const int32_t m = ms[3 * i + j];
      if (m >= 0 && std::find(run_masters.begin(), run_masters.end(), m) == run_masters.end()) ++add;
    }
    if (new_tri || i - run_off.back() >= kRunSamples || (int)run_masters.size() + add > kRunMasters) {
      if (i > 0) run_off.push_back(i);
      run_slave.insert(run_slave.end(), {sl[3 * i], sl[3 * i + 1], sl[3 * i + 2]});
      run_masters.clear();
    }
    for (int j = 0; j < 3; ++j) {
      const int32_t m = ms[3 * i + j];
      if (m >= 0 && std::find(run_masters.begin(), run_masters.end(), m) == run_masters.end())
        run_masters.push_back(m);
    }
  }
  if (n > 0) run_off.push_back(n);
  const int64_t R = (int64_t)run_slave.size() / 3;
  std::vector<int32_t> lm_off{0}, lm_ids, lp_off{0}, lp;
  std::vector<uint32_t> li4(n > 0 ? n : 1, 0xffffffffu);  // per sample local master indices (u8 x 3)
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
    std::vector<int32_t> pr;  // local master pairs (a << 16 | b), a <= b
    for (int64_t i = run_off[r]; i < run_off[r + 1]; ++i) {
      const int nm = ty[i] == GMCP_FACE ? 3 : (ty[i] == GMCP_EDGE ? 2 : 1);
      int li[3];
      uint32_t packed = 0xffffffffu;
      for (int j = 0; j < nm; ++j) {
        li[j] = (int)(std::lower_bound(loc.begin(), loc.end(), ms[3 * i + j]) - loc.begin());
        packed = (packed & ~(0xffu << (8 * j))) | ((uint32_t)li[j] << (8 * j));
      }
      li4[i] = packed;
      for (int a = 0; a < nm; ++a)
        for (int b = 0; b < nm; ++b)
          if (li[a] <= li[b]) pr.push_back((li[a] << 16) | li[b]);
    }
    std::sort(pr.begin(), pr.end());
    pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
    lp.insert(lp.end(), pr.begin(), pr.end());
    lp_off.push_back((int32_t)lp.size());
    pbase[r] = plen;
    plen += partial_size((int)loc.size());
  }
  // BCSR pattern, per-block contribution lists and row entries over all N
  // vertex rows. Runs are visited in ascending order and the per-row sort is
  // stable, so every block lists its contributions in ascending run order.
  const int64_t N = c.n_vertices();
  struct Contrib {
    int32_t col;
    int64_t code;
  };
  std::vector<std::vector<Contrib>> rc(N);
  std::vector<std::vector<int64_t>> rent(N);
  for (int64_t r = 0; r < R; ++r) {
    const int32_t* s = &run_slave[3 * r];
    const int32_t* L = lm_ids.data() + lm_off[r];
    const int M = lm_off[r + 1] - lm_off[r];
    const int64_t head = (pbase[r] << 12) | ((int64_t)M << 8);
    auto col_of = [&](int b) { return b < 3 ? s[b] : L[b - 3]; };
    for (int i = 0; i < 3; ++i) {
      rent[s[i]].push_back(head | i);
      for (int b = 0; b < 3 + M; ++b) rc[s[i]].push_back({col_of(b), head | (i << 4) | b});
    }
    for (int k = 0; k < M; ++k) {
      rent[L[k]].push_back(head | (3 + k));
      for (int b = 0; b < 3; ++b) rc[L[k]].push_back({s[b], head | ((3 + k) << 4) | b});
    }
    for (int p = lp_off[r]; p < lp_off[r + 1]; ++p) {  // listed master pairs only
      const int a = lp[p] >> 16, b = lp[p] & 0xffff;
      rc[L[a]].push_back({L[b], head | ((3 + a) << 4) | (3 + b)});
      if (a != b) rc[L[b]].push_back({L[a], head | ((3 + b) << 4) | (3 + a)});
    }
  }
  std::vector<int32_t> rowptr(N + 1, 0), cols, eoff(N + 1, 0), boff{0};
  std::vector<int64_t> ents, contrib;
  for (int64_t v = 0; v < N; ++v) {
    auto& cv = rc[v];
    std::stable_sort(cv.begin(), cv.end(), [](const Contrib& a, const Contrib& b) { return a.col < b.col; });
    for (size_t q = 0; q < cv.size(); ++q) {
      if (q == 0 || cv[q].col != cv[q - 1].col) {
        if (q > 0) boff.push_back((int32_t)contrib.size());
        cols.push_back(cv[q].col);
      }
      contrib.push_back(cv[q].code);
    }
    if (!cv.empty()) boff.push_back((int32_t)contrib.size());
    rowptr[v + 1] = (int32_t)cols.size();
    ents.insert(ents.end(), rent[v].begin(), rent[v].end());
    eoff[v + 1] = (int32_t)ents.size();
    std::vector<Contrib>().swap(cv);
  }
  if (contrib.size() >= (size_t)INT32_MAX) throw StatusError(GMCP_ERR_CONFIG, "contact Hessian too large");
  cudaStream_t s = c.stream;
  P.n_runs = R;
  P.run_off.upload(run_off, s);
  P.run_slave.upload(run_slave, s);
  P.lm_off.upload(lm_off, s);
  P.lm_ids.upload(lm_ids, s);
  P.lp_off.upload(lp_off, s);
  P.lp.upload(lp, s);
  P.li4.upload(li4, s);
  P.pbase.upload(pbase, s);
  P.partial_len = plen;
  P.partial.resize(std::max<int64_t>(plen, 1));
  P.n_rows = (int32_t)N;
  P.nnzb = (int64_t)cols.size();
  P.rowptr.upload(rowptr, s);
  P.cols.upload(cols, s);
  P.h_rowptr = rowptr;
  P.h_cols = cols;
  P.vals.resize(std::max<int64_t>(9 * P.nnzb, 1));
  P.row_ent_off.upload(eoff, s);
  P.row_ent.upload(ents, s);
  P.blk_off.upload(boff, s);
  P.contrib.upload(contrib, s);
  c.sync();
  P.valid = true;
}

double run_assembly(Ctx& c, int mode, int64_t* bad) {
  init_kernels();
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

void time_assembly(Ctx& c, int reps, int flush_l2, double* ms_pass, double* ms_kernel) {
  init_kernels();
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
