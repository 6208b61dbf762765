// Device context behind gmcp_ctx (include/gmcp_b200.h).
#pragma once

#include <memory>

#include "common.cuh"

namespace gmcp_b200 {

struct DevSurface {
  int32_t n_tris = 0, n_edges = 0, n_verts = 0;
  DBuf<int32_t> tris, edges, tri_edges, verts;
  std::vector<int32_t> h_tris, h_edges, h_tri_edges, h_verts;  // host mirror (setup only)
};

// Contact-Hessian assembly plan, rebuilt whenever the sample set changes.
// Level 1 (K7, one warp per slave run) reduces each run of samples sharing a
// slave triangle into a compact partial; level 2 (K8, one thread per BCSR
// block / vertex row) gathers the partials' contributions to that block or
// gradient row. Both levels sum in a fixed order: bitwise deterministic.
struct AssemblyPlan {
  int64_t n_runs = 0;
  DBuf<int64_t> run_off;     // [R+1] sample range of each run
  DBuf<int32_t> run_slave;   // [R][3]
  DBuf<int32_t> lm_off;      // [R+1] local master vertex table offsets
  DBuf<int32_t> lm_ids;      // global ids, ascending within a run
  DBuf<int64_t> pbase;       // [R] partial base offset (doubles)
  DBuf<uint32_t> li4;        // per sample: local master index of each slot (u8 x 3, 0xff = none)
  int64_t partial_len = 0;
  DBuf<double> partial;
  // BCSR pattern over all N vertex rows
  int32_t n_rows = 0;
  int64_t nnzb = 0;
  DBuf<int32_t> rowptr;      // [N+1]
  DBuf<int32_t> cols;        // [nnzb]
  // device planner scratch (plan.cu), reused across rebuilds
  struct Tmp {
    DBuf<int32_t> head, hscan, run_cnt, run_first, run_M, rowcnt, ucnt, nuniq;
    DBuf<int64_t> seg_start, psize, ccount, coff, ecount, eoff, cval, cval2, eval, eval2;
    DBuf<unsigned long long> pmask, ckey, ckey2, ekey, ekey2, ukey;
  } tmp;
  DBuf<double> vals;         // [nnzb][9]
  DBuf<int32_t> row_ent_off; // [N+1]
  DBuf<int32_t> blk_off;     // [nnzb+1] contribution list of each BCSR block
  DBuf<int64_t> contrib;     // (pbase << 12) | (M << 8) | (role << 4) | b, ascending run per block
  DBuf<int64_t> row_ent;     // (pbase << 12) | (M << 8) | role ; role < 3 slave i, else 3 + local master
  bool valid = false;
};

// Base of per-context scratch defined next to the code that uses it.
struct TmpBase {
  virtual ~TmpBase() = default;
};

struct Ctx {
  int device = 0;
  CubScratch cub;        // CUB temp storage (bound per C-ABI call)
  int k7_resident = 0;   // K7 persistent grid size on this context's device
  bool thread_query = std::getenv("GMCP_THREAD_QUERY") != nullptr;  // broadphase: per-thread traversal
  std::unique_ptr<TmpBase> rebuild_tmp;  // broadphase + sampler scratch (sampler.cu)
  std::unique_ptr<TmpBase> embed_tmp;    // dual-mesh embedding scratch (sampler.cu)
  std::unique_ptr<TmpBase> scene_tmp;    // scene-segmented reductions scratch (exact.cu)
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  int64_t n_dof = 0;
  gmcp_barrier_params params{};
  bool have_params = false;

  DevSurface slave, master;
  DBuf<double> x, dx, grad, eps_ref;
  // A System (solver.cu) points its contact pairs at its own x / dx buffers.
  double* x_ext = nullptr;
  double* dx_ext = nullptr;
  double* X() const { return x_ext ? x_ext : x.p; }
  double* DX() const { return dx_ext ? dx_ext : dx.p; }

  // batched scenes: scene id per vertex (empty = one scene)
  DBuf<int32_t> vscene;
  int32_t n_scenes = 1;
  // batched re-sampling: when set, the broadphase queries only slave
  // triangles of scenes with scene_mask[s] != 0 (the others get no samples)
  DBuf<uint8_t> scene_mask;
  bool use_scene_mask = false;

  // candidate pairs (CSR per slave tri)
  DBuf<int64_t> pair_off[3];
  DBuf<int32_t> pair_ids[3];
  bool have_pairs = false;

  // samples
  int64_t ns = 0;
  DBuf<int8_t> s_type;
  DBuf<int32_t> s_slave, s_master;
  DBuf<double> s_beta_s, s_beta_m, s_wm, s_eta, s_weight, s_gamma, s_eps, s_gref, s_coef;
  DBuf<int64_t> face_idx;  // indices of face samples (pressure field order)
  DBuf<int64_t> face_flag, face_pos;  // derive_sample_fields scratch

  AssemblyPlan plan;

  // snapshot of the raw sample fields (batched per-scene rebuilds splice old
  // and new per-scene segments)
  struct Snapshot {
    int64_t ns = 0;
    DBuf<int8_t> type;
    DBuf<int32_t> slave, master;
    DBuf<double> beta_s, beta_m, eta, weight, gamma, eps, gref;
  } snap, spliced;  // spliced: double buffer for the merged arrays (no per-rebuild allocation)

  // reduction scratch
  DBuf<double> red_d;
  DBuf<unsigned long long> red_u;

  // accumulate-into-caller gradients: the caller's buffer is uploaded on an
  // auxiliary stream while the assembly runs, summed on the device, downloaded once
  cudaStream_t aux = nullptr;
  cudaEvent_t aux_done = nullptr;
  DBuf<double> grad_in;
  // single-call host path (run_assembly_host): positions landed, contact
  // gradient rows ready, caller gradient + contact gradient
  cudaEvent_t x_ready = nullptr, rows_done = nullptr;
  DBuf<double> grad_sum;
  void* host_scalars = nullptr;  // pinned: status words + energy of the single-call path
  Ctx() = default;
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
  ~Ctx() {
    if (host_scalars) cudaFreeHost(host_scalars);
    if (aux_done) cudaEventDestroy(aux_done);
    if (x_ready) cudaEventDestroy(x_ready);
    if (rows_done) cudaEventDestroy(rows_done);
    if (aux) cudaStreamDestroy(aux);
  }
  void ensure_aux() {
    if (aux && x_ready) return;
    GMCP_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    GMCP_CUDA(cudaEventCreateWithFlags(&aux_done, cudaEventDisableTiming));
    GMCP_CUDA(cudaEventCreateWithFlags(&x_ready, cudaEventDisableTiming));
    GMCP_CUDA(cudaEventCreateWithFlags(&rows_done, cudaEventDisableTiming));
    GMCP_CUDA(cudaMallocHost(&host_scalars, 64));
  }

  DevSamples samples() const {
    DevSamples d;
    d.n = ns;
    d.type = s_type.p;
    d.slave = s_slave.p;
    d.master = s_master.p;
    d.beta_s = s_beta_s.p;
    d.wm = s_wm.p;
    d.coef = s_coef.p;
    d.eps = s_eps.p;
    d.gamma = s_gamma.p;
    return d;
  }
  int64_t n_vertices() const { return n_dof / 3; }
  void sync() { GMCP_CUDA(cudaStreamSynchronize(stream)); }
};

// --- entry points implemented in the .cu files (all enqueue on ctx.stream) ---
// contact_eval.cu
void derive_sample_fields(Ctx& c);  // coef, wm, face_idx from the raw fields
void snapshot_samples(Ctx& c);      // raw sample fields -> c.snap
// per scene s: keep the snapshot's segment [soff_old[s], soff_old[s+1]) or take
// the current (new) segment [soff_new[s], soff_new[s+1]); result in c's arrays
void splice_samples(Ctx& c, const std::vector<int64_t>& soff_old, const std::vector<int64_t>& soff_new,
                    const std::vector<uint8_t>& take_new, std::vector<int64_t>& soff_out);
struct EnergyOut {
  double energy, min_gap, min_gap_prefix;
  int64_t first_bad, first_degenerate;
};
EnergyOut run_energy(Ctx& c, bool need_prefix_min);
void add_into(Ctx& c, double* dst, const double* src, int64_t n);  // dst += src on c.stream
void build_assembly_plan(Ctx& c);  // host-side plan from the device samples
// mode 0: gradient only, 1: gradient + Hessian. Returns energy; throws on infeasible.
double run_assembly(Ctx& c, int mode, int64_t* bad);
// One host call of the reference's add_contact_gradient[_hessian](state,
// params, x, grad[, H]): x (host, 3N) goes up, the caller's grad (host, may be
// null) travels up behind it while K7 runs, the contact gradient rows are
// gathered first so grad + g_c comes down while the Hessian blocks are
// gathered; one synchronisation. On an infeasible / degenerate sample the
// caller's grad is left as it was and StatusError is thrown.
double run_assembly_host(Ctx& c, int mode, const double* x, double* grad, int64_t* bad);
void run_pressure(Ctx& c, gmcp_pressure_record* out_host);
void run_force_summary(Ctx& c, double* out12);
void run_kinematics(Ctx& c, double* g, int32_t* nv, int32_t* ids, double* dg);
void time_assembly(Ctx& c, int reps, int flush_l2, double* ms_pass, double* ms_kernel);
// exact.cu (-fmad=false)
double run_step_filter(Ctx& c);
double run_displacement_cap(Ctx& c);
// batched scenes (contiguous per scene): sample offsets per scene, per-scene
// energy / feasibility, per-scene step size min(1, filter, cap)
void scene_sample_offsets(Ctx& c, const int32_t* vscene_dev, int n_scenes, std::vector<int64_t>& soff_host,
                          DBuf<int64_t>& soff_dev);
void run_scene_energy(Ctx& c, const double* xp, int n_scenes, const int64_t* soff_dev, double* e,
                      int64_t* first_bad, int64_t* first_deg, double* min_gap);
void run_scene_alpha(Ctx& c, int n_scenes, const int64_t* soff_dev, const int64_t* voff_dev, double* alpha,
                     int64_t* first_deg);
void run_broadphase(Ctx& c, double r, int64_t* counts);
int64_t run_sampler(Ctx& c, const double* eps_ref_dev);
void run_embed(Ctx& c, const double* points, int64_t np, const double* host_v, int64_t nhv, const int32_t* host_t,
               int64_t nht, int32_t* tri, double* bary, double* offset, int64_t* bad);
void run_apply_embedding(Ctx& c, const int32_t* tri, const double* bary, const double* offset, int64_t n,
                         const int32_t* host_t, int64_t nht, const double* host_x, int64_t nhv, double* out,
                         int64_t* bad);

}  // namespace gmcp_b200
