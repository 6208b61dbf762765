// C-ABI entry points (include/gmcp_b200.h). Translates C++ exceptions into
// GMCP_* status codes and a thread-local message; never falls back to a CPU
// path.
#include <cstring>
#include <string>

#include "../../include/gmcp_b200.h"
#include "ctx.hpp"

using namespace gmcp_b200;

struct gmcp_ctx {
  Ctx c;
};

namespace gmcp_b200 {
CubScratch*& bound_scratch() {
  thread_local CubScratch* s = nullptr;
  return s;
}
}  // namespace gmcp_b200

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const StatusError& e) {
    return fail(e.code, e.what());
  } catch (const CudaError& e) {
    return fail(GMCP_ERR_CUDA, e.what());
  } catch (const std::bad_alloc& e) {
    return fail(GMCP_ERR_CUDA, std::string("allocation failed: ") + e.what());
  } catch (const std::exception& e) {
    return fail(GMCP_ERR_ARG, e.what());
  }
}

void need(bool ok, const char* what) {
  if (!ok) throw StatusError(GMCP_ERR_ARG, what);
}

void set_surface(Ctx& c, DevSurface& d, const gmcp_surface* s) {
  need(s != nullptr, "null surface");
  need(s->n_tris >= 0 && s->n_edges >= 0 && s->n_verts >= 0, "negative surface size");
  d.n_tris = s->n_tris;
  d.n_edges = s->n_edges;
  d.n_verts = s->n_verts;
  d.h_tris.assign(s->tris, s->tris + 3 * (size_t)s->n_tris);
  d.h_tri_edges.assign(s->tri_edges, s->tri_edges + 3 * (size_t)s->n_tris);
  d.h_edges.assign(s->edges, s->edges + 2 * (size_t)s->n_edges);
  d.h_verts.assign(s->verts, s->verts + (size_t)s->n_verts);
  d.tris.upload(d.h_tris, c.stream);
  d.tri_edges.upload(d.h_tri_edges, c.stream);
  d.edges.upload(d.h_edges, c.stream);
  d.verts.upload(d.h_verts, c.stream);
}

void check_ctx(gmcp_ctx* ctx) { need(ctx != nullptr, "null gmcp_ctx"); }

void throw_bad(int64_t bad) {
  throw StatusError(GMCP_ERR_INFEASIBLE, "contact sample " + std::to_string(bad) + " has non-positive gap", bad);
}
}  // namespace

extern "C" {

const char* gmcp_last_error(void) { return g_err.c_str(); }

int gmcp_device_count(int* n) {
  return guarded([&] {
    GMCP_CUDA(cudaGetDeviceCount(n));
    return GMCP_OK;
  });
}

int gmcp_ctx_create(int device, gmcp_ctx** out) {
  return guarded([&] {
    need(out != nullptr, "null out");
    int n = 0;
    GMCP_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw StatusError(GMCP_ERR_CUDA, "no such CUDA device");
    auto* ctx = new gmcp_ctx;
    ctx->c.device = device;
    const DeviceBind bind_(device, &ctx->c.cub);  // the caller's current device is restored
    GMCP_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
    *out = ctx;
    return GMCP_OK;
  });
}

void gmcp_ctx_destroy(gmcp_ctx* ctx) {
  if (!ctx) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  cudaStream_t s = ctx->c.stream;
  delete ctx;
  cudaStreamDestroy(s);
  cudaSetDevice(prev);
}

int64_t gmcp_launch_count(const gmcp_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int gmcp_resolve_barrier_params(gmcp_barrier_params* p, double m) {
  // barrier.hpp:25-46 (host arithmetic; identical expressions)
  if (!p) return fail(GMCP_ERR_ARG, "null params");
  if (!(m > 0)) return fail(GMCP_ERR_CONFIG, "barrier params: mean slave edge length must be positive");
  if (!(p->kappa_face > 0)) return fail(GMCP_ERR_CONFIG, "barrier params: kappa_face must be positive");
  if (p->kappa_edge < 0) p->kappa_edge = 1e-3 * p->kappa_face * m;
  if (p->kappa_point < 0) p->kappa_point = 1e-3 * p->kappa_face * m * m;
  if (!(p->kappa_edge > 0) || !(p->kappa_point > 0))
    return fail(GMCP_ERR_CONFIG, "barrier params: per-type stiffnesses must be positive");
  if (!(p->eps_max > 0)) return fail(GMCP_ERR_CONFIG, "barrier params: eps_max must be positive");
  if (!(p->delta_face > 0) || p->delta_face > 1.0 / 3.0)
    return fail(GMCP_ERR_CONFIG, "barrier params: delta_face must lie in (0, 1/3]");
  if (!(p->delta_edge > 0) || p->delta_edge > 0.5)
    return fail(GMCP_ERR_CONFIG, "barrier params: delta_edge must lie in (0, 1/2]");
  if (p->detection_radius < 0) p->detection_radius = 10.0 * p->eps_max;
  if (!(p->detection_radius > 0)) return fail(GMCP_ERR_CONFIG, "barrier params: detection_radius must be positive");
  if (p->quad_order_face < 1 || p->quad_order_face > 4)
    return fail(GMCP_ERR_CONFIG, "barrier params: quad_order_face must lie in 1..4");
  if (p->quad_order_edge < 1 || p->quad_order_edge > 5)
    return fail(GMCP_ERR_CONFIG, "barrier params: quad_order_edge must lie in 1..5");
  return GMCP_OK;
}

int gmcp_set_params(gmcp_ctx* ctx, const gmcp_barrier_params* p) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    need(p != nullptr, "null params");
    if (!(p->kappa_face > 0) || !(p->kappa_edge > 0) || !(p->kappa_point > 0) || !(p->eps_max > 0))
      throw StatusError(GMCP_ERR_CONFIG, "gmcp_set_params: parameters must be resolved (positive stiffnesses)");
    ctx->c.params = *p;
    ctx->c.have_params = true;
    if (ctx->c.ns) derive_sample_fields(ctx->c);  // coef depends on the stiffnesses
    return GMCP_OK;
  });
}

int gmcp_set_surfaces(gmcp_ctx* ctx, const gmcp_surface* slave, const gmcp_surface* master) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    set_surface(ctx->c, ctx->c.slave, slave);
    set_surface(ctx->c, ctx->c.master, master);
    ctx->c.have_pairs = false;
    ctx->c.sync();
    return GMCP_OK;
  });
}

int gmcp_set_vertex_scenes(gmcp_ctx* ctx, const int32_t* scene, int64_t n_vertices) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    Ctx& c = ctx->c;
    c.have_pairs = false;
    if (!scene) {
      c.vscene.resize(0);
      c.n_scenes = 1;
      return GMCP_OK;
    }
    need(n_vertices >= 0, "vertex scenes: negative count");
    int32_t mx = -1;
    for (int64_t v = 0; v < n_vertices; ++v) {
      need(scene[v] >= 0 && scene[v] < (1 << 20), "vertex scenes: ids must lie in [0, 2^20)");
      mx = std::max(mx, scene[v]);
    }
    c.vscene.upload(scene, n_vertices, c.stream);
    c.n_scenes = mx + 1;
    c.sync();
    return GMCP_OK;
  });
}

int gmcp_set_positions(gmcp_ctx* ctx, const double* x, int64_t n_dof) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    need(x != nullptr && n_dof >= 0 && n_dof % 3 == 0, "positions: need 3N doubles");
    Ctx& c = ctx->c;
    if (n_dof != c.n_dof) c.plan.valid = false;
    c.n_dof = n_dof;
    c.x.upload(x, n_dof, c.stream);
    if (c.dx.n != (size_t)n_dof) {
      c.dx.resize(n_dof);
      c.dx.zero(c.stream);
    }
    c.sync();
    return GMCP_OK;
  });
}

int gmcp_set_step(gmcp_ctx* ctx, const double* dx, int64_t n_dof) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    need(dx != nullptr && n_dof == ctx->c.n_dof, "step: size must match positions");
    ctx->c.dx.upload(dx, n_dof, ctx->c.stream);
    ctx->c.sync();
    return GMCP_OK;
  });
}

double* gmcp_positions_device(gmcp_ctx* ctx) { return ctx ? ctx->c.x.p : nullptr; }
double* gmcp_step_device(gmcp_ctx* ctx) { return ctx ? ctx->c.dx.p : nullptr; }

int gmcp_upload_samples(gmcp_ctx* ctx, const gmcp_samples* s) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    need(s != nullptr && s->n >= 0, "null samples");
    Ctx& c = ctx->c;
    need(c.have_params, "gmcp_upload_samples: call gmcp_set_params first");
    const int64_t n = s->n;
    if (n) {
      need(s->type && s->slave && s->master && s->beta_s && s->beta_m && s->eta && s->weight && s->gamma &&
               s->eps && s->g_ref,
           "samples: null field");
      for (int64_t i = 0; i < 3 * n; ++i)
        if (s->slave[i] < 0 || 3 * (int64_t)s->slave[i] >= c.n_dof)
          throw StatusError(GMCP_ERR_ARG, "samples: slave vertex id out of range");
      for (int64_t i = 0; i < n; ++i) {
        const int nm = s->type[i] == GMCP_FACE ? 3 : (s->type[i] == GMCP_EDGE ? 2 : 1);
        for (int j = 0; j < 3; ++j) {
          const int32_t m = s->master[3 * i + j];
          if (j < nm && (m < 0 || 3 * (int64_t)m >= c.n_dof))
            throw StatusError(GMCP_ERR_ARG, "samples: master vertex id out of range");
        }
      }
    }
    c.ns = n;
    c.s_type.upload(s->type, n, c.stream);
    c.s_slave.upload(s->slave, 3 * n, c.stream);
    c.s_master.upload(s->master, 3 * n, c.stream);
    c.s_beta_s.upload(s->beta_s, 3 * n, c.stream);
    c.s_beta_m.upload(s->beta_m, 3 * n, c.stream);
    c.s_eta.upload(s->eta, n, c.stream);
    c.s_weight.upload(s->weight, n, c.stream);
    c.s_gamma.upload(s->gamma, n, c.stream);
    c.s_eps.upload(s->eps, n, c.stream);
    c.s_gref.upload(s->g_ref, n, c.stream);
    derive_sample_fields(c);
    c.sync();
    return GMCP_OK;
  });
}

int64_t gmcp_num_samples(const gmcp_ctx* ctx) { return ctx ? ctx->c.ns : 0; }

int gmcp_download_samples(gmcp_ctx* ctx, gmcp_samples* o) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    Ctx& c = ctx->c;
    const int64_t n = c.ns;
    need(o != nullptr && o->n >= n, "samples out: too small");
    c.s_type.download(o->type, n, c.stream);
    c.s_slave.download(o->slave, 3 * n, c.stream);
    c.s_master.download(o->master, 3 * n, c.stream);
    c.s_beta_s.download(o->beta_s, 3 * n, c.stream);
    c.s_beta_m.download(o->beta_m, 3 * n, c.stream);
    c.s_eta.download(o->eta, n, c.stream);
    c.s_weight.download(o->weight, n, c.stream);
    c.s_gamma.download(o->gamma, n, c.stream);
    c.s_eps.download(o->eps, n, c.stream);
    c.s_gref.download(o->g_ref, n, c.stream);
    c.sync();
    return GMCP_OK;
  });
}

int gmcp_try_energy(gmcp_ctx* ctx, double* energy, double* min_gap, int32_t* feasible) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    const EnergyOut o = run_energy(ctx->c, true);
    if (o.first_degenerate >= 0 && (o.first_bad < 0 || o.first_degenerate < o.first_bad))
      throw StatusError(GMCP_ERR_DEGENERATE, "triangle_normal: degenerate triangle (area below cutoff)",
                        o.first_degenerate);
    *energy = o.energy;
    *min_gap = o.first_bad >= 0 ? o.min_gap_prefix : o.min_gap;
    *feasible = o.first_bad < 0 ? 1 : 0;
    return GMCP_OK;
  });
}

int gmcp_energy(gmcp_ctx* ctx, double* energy, int64_t* bad) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    if (bad) *bad = -1;
    const EnergyOut o = run_energy(ctx->c, false);
    if (o.first_degenerate >= 0 && (o.first_bad < 0 || o.first_degenerate < o.first_bad))
      throw StatusError(GMCP_ERR_DEGENERATE, "triangle_normal: degenerate triangle (area below cutoff)",
                        o.first_degenerate);
    if (o.first_bad >= 0) {
      if (bad) *bad = o.first_bad;
      throw_bad(o.first_bad);
    }
    *energy = o.energy;
    return GMCP_OK;
  });
}

static int grad_common(gmcp_ctx* ctx, int mode, double* grad, double* energy, int64_t* bad) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    Ctx& c = ctx->c;
    int64_t b = -1;
    if (bad) *bad = -1;
    if (grad) {  // the caller's gradient travels up while the assembly runs
      c.ensure_aux();
      c.grad_in.resize(std::max<int64_t>(c.n_dof, 1));
      GMCP_CUDA(cudaMemcpyAsync(c.grad_in.p, grad, c.n_dof * sizeof(double), cudaMemcpyHostToDevice, c.aux));
      GMCP_CUDA(cudaEventRecord(c.aux_done, c.aux));
    }
    try {
      const double e = run_assembly(c, mode, &b);
      if (energy) *energy = e;
    } catch (const StatusError& se) {
      if (grad) GMCP_CUDA(cudaStreamSynchronize(c.aux));
      if (bad) *bad = se.bad;
      throw;
    }
    if (grad) {  // accumulated into the caller's buffer (contact_energy.hpp:126-142): grad += g_c
      GMCP_CUDA(cudaStreamWaitEvent(c.stream, c.aux_done, 0));
      add_into(c, c.grad_in.p, c.grad.p, c.n_dof);
      c.grad_in.download(grad, c.n_dof, c.stream);
      c.sync();
    }
    return GMCP_OK;
  });
}

int gmcp_gradient(gmcp_ctx* ctx, double* grad, double* energy, int64_t* bad) {
  return grad_common(ctx, 0, grad, energy, bad);
}
int gmcp_gradient_hessian(gmcp_ctx* ctx, double* grad, double* energy, int64_t* bad) {
  return grad_common(ctx, 1, grad, energy, bad);
}

static int add_common(gmcp_ctx* ctx, int mode, const double* x, int64_t n_dof, double* grad, double* energy,
                      int64_t* bad) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    need(x != nullptr && n_dof >= 0 && n_dof % 3 == 0, "positions: need 3N doubles");
    Ctx& c = ctx->c;
    if (n_dof != c.n_dof) {
      c.plan.valid = false;
      c.n_dof = n_dof;
    }
    if (c.dx.n != (size_t)n_dof) {
      c.dx.resize(n_dof);
      c.dx.zero(c.stream);
    }
    int64_t b = -1;
    if (bad) *bad = -1;
    try {
      const double e = run_assembly_host(c, mode, x, grad, &b);
      if (energy) *energy = e;
    } catch (const StatusError& se) {
      if (bad) *bad = se.bad;
      throw;
    }
    return GMCP_OK;
  });
}

int gmcp_add_gradient(gmcp_ctx* ctx, const double* x, int64_t n_dof, double* grad, double* energy, int64_t* bad) {
  return add_common(ctx, 0, x, n_dof, grad, energy, bad);
}
int gmcp_add_gradient_hessian(gmcp_ctx* ctx, const double* x, int64_t n_dof, double* grad, double* energy,
                              int64_t* bad) {
  return add_common(ctx, 1, x, n_dof, grad, energy, bad);
}

int gmcp_download_hessian(gmcp_ctx* ctx, int64_t* nnzb, int32_t* rowptr, int32_t* cols, double* vals) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    Ctx& c = ctx->c;
    need(c.plan.valid, "no assembled Hessian (call gmcp_gradient_hessian first)");
    *nnzb = c.plan.nnzb;
    if (rowptr) c.plan.rowptr.download(rowptr, c.plan.n_rows + 1, c.stream);
    if (cols) c.plan.cols.download(cols, c.plan.nnzb, c.stream);
    if (vals) c.plan.vals.download(vals, 9 * c.plan.nnzb, c.stream);
    c.sync();
    return GMCP_OK;
  });
}

int gmcp_step_filter(gmcp_ctx* ctx, double* alpha) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    *alpha = run_step_filter(ctx->c);
    return GMCP_OK;
  });
}

int gmcp_displacement_cap(gmcp_ctx* ctx, double* alpha) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    *alpha = run_displacement_cap(ctx->c);
    return GMCP_OK;
  });
}

int gmcp_pressure_field(gmcp_ctx* ctx, int64_t* n, gmcp_pressure_record* out) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    *n = (int64_t)ctx->c.face_idx.n;
    if (out) run_pressure(ctx->c, out);
    return GMCP_OK;
  });
}

int gmcp_force_summary(gmcp_ctx* ctx, double* out12) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    run_force_summary(ctx->c, out12);
    return GMCP_OK;
  });
}

int gmcp_kinematics(gmcp_ctx* ctx, double* g, int32_t* nv, int32_t* ids, double* dg) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    run_kinematics(ctx->c, g, nv, ids, dg);
    return GMCP_OK;
  });
}

int gmcp_broadphase(gmcp_ctx* ctx, double r, int64_t* counts) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    if (!(r > 0)) throw StatusError(GMCP_ERR_CONFIG, "build_candidate_pairs: detection radius must be positive");
    run_broadphase(ctx->c, r, counts);
    return GMCP_OK;
  });
}

int gmcp_download_pairs(gmcp_ctx* ctx, int which, int64_t* offsets, int32_t* ids) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    Ctx& c = ctx->c;
    need(c.have_pairs, "no candidate pairs");
    need(which >= 0 && which < 3, "which must be 0..2");
    if (offsets) c.pair_off[which].download(offsets, c.slave.n_tris + 1, c.stream);
    if (ids) c.pair_ids[which].download(ids, c.pair_ids[which].n, c.stream);
    c.sync();
    return GMCP_OK;
  });
}

int gmcp_upload_pairs(gmcp_ctx* ctx, const int64_t* to, const int32_t* ti, const int64_t* eo, const int32_t* ei,
                      const int64_t* vo, const int32_t* vi) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    Ctx& c = ctx->c;
    const int32_t nst = c.slave.n_tris;
    const int64_t* offs[3] = {to, eo, vo};
    const int32_t* ids[3] = {ti, ei, vi};
    for (int k = 0; k < 3; ++k) {
      need(offs[k] != nullptr, "null pair offsets");
      c.pair_off[k].upload(offs[k], nst + 1, c.stream);
      c.pair_ids[k].upload(ids[k], offs[k][nst], c.stream);
    }
    c.have_pairs = true;
    c.sync();
    return GMCP_OK;
  });
}

int gmcp_build_samples(gmcp_ctx* ctx, const double* eps_reference, int64_t* n_samples) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    Ctx& c = ctx->c;
    need(c.have_pairs, "gmcp_build_samples: no candidate pairs (call gmcp_broadphase)");
    need(c.have_params, "gmcp_build_samples: call gmcp_set_params first");
    const double* er = nullptr;
    if (eps_reference) {
      c.eps_ref.upload(eps_reference, c.n_dof, c.stream);
      er = c.eps_ref.p;
    }
    *n_samples = run_sampler(c, er);
    return GMCP_OK;
  });
}

int gmcp_time_assembly(gmcp_ctx* ctx, int reps, int flush_l2, double* ms_pass, double* ms_kernel) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    need(reps > 0, "reps must be positive");
    time_assembly(ctx->c, reps, flush_l2, ms_pass, ms_kernel);
    return GMCP_OK;
  });
}


int gmcp_embed_in_surface(gmcp_ctx* ctx, const double* points, int64_t n_points, const double* host_vertices,
                          int64_t n_host_vertices, const int32_t* host_tris, int64_t n_host_tris, int32_t* tri,
                          double* bary, double* offset, int64_t* bad) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    need(n_points >= 0 && n_host_vertices >= 0 && n_host_tris >= 0, "embedding: negative sizes");
    need((points || !n_points) && host_vertices && host_tris && (tri || !n_points) && (bary || !n_points) &&
             (offset || !n_points),
         "embedding: null buffer");
    for (int64_t k = 0; k < 3 * n_host_tris; ++k)
      need(host_tris[k] >= 0 && host_tris[k] < n_host_vertices, "embedding: host triangle vertex out of range");
    int64_t b = -1;
    try {
      run_embed(ctx->c, points, n_points, host_vertices, n_host_vertices, host_tris, n_host_tris, tri, bary, offset,
                &b);
    } catch (const StatusError&) {
      if (bad) *bad = b;
      throw;
    }
    if (bad) *bad = -1;
    return GMCP_OK;
  });
}

int gmcp_apply_embedding(gmcp_ctx* ctx, const int32_t* tri, const double* bary, const double* offset, int64_t n,
                         const int32_t* host_tris, int64_t n_host_tris, const double* host_positions,
                         int64_t n_host_vertices, double* out, int64_t* bad) {
  return guarded([&] {
    check_ctx(ctx);
    const DeviceBind bind_(ctx->c.device, &ctx->c.cub);
    need(n >= 0 && (tri || !n) && (bary || !n) && (offset || !n) && (out || !n) && host_tris && host_positions,
         "apply_embedding: null buffer");
    for (int64_t i = 0; i < n; ++i) need(tri[i] >= 0 && tri[i] < n_host_tris, "apply_embedding: triangle out of range");
    for (int64_t k = 0; k < 3 * n_host_tris; ++k)
      need(host_tris[k] >= 0 && host_tris[k] < n_host_vertices, "apply_embedding: host vertex out of range");
    int64_t b = -1;
    try {
      run_apply_embedding(ctx->c, tri, bary, offset, n, host_tris, n_host_tris, host_positions, n_host_vertices,
                          out, &b);
    } catch (const StatusError&) {
      if (bad) *bad = b;
      throw;
    }
    if (bad) *bad = -1;
    return GMCP_OK;
  });
}

}  // extern "C"
