// C wrapper around the UNMODIFIED reference headers. TEST INFRASTRUCTURE ONLY.
// Built by oracle/Makefile against /root/reference/proj/include and the
// Eigen-API shim in oracle/eigen_shim into oracle/_ref/libgmcp_ref.so. It
// implements oracle/gmcp_oracle_api.h by calling the reference functions
// verbatim, plus ref_* helpers (meshes, scene solves) used to pin the Python
// scene generators and to time the reference CPU path.
#include "gmcp/bench.hpp"
#include "gmcp/embedding.hpp"

#include <chrono>
#include <cstring>
#include <map>

#include "gmcp_oracle_api.h"

using namespace gmcp;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const InfeasibleGapError& e) {
    return fail(GMCP_ERR_INFEASIBLE, e.what());
  } catch (const MeshError& e) {
    return fail(GMCP_ERR_DEGENERATE, e.what());
  } catch (const ConfigError& e) {
    return fail(GMCP_ERR_CONFIG, e.what());
  } catch (const ParseError& e) {
    return fail(GMCP_ERR_PARSE, e.what());
  } catch (const SolverError& e) {
    return fail(GMCP_ERR_SOLVER, e.what());
  } catch (const Error& e) {
    return fail(GMCP_ERR_INFEASIBLE, e.what());  // barrier()/adaptive_eps() domain errors
  } catch (const std::exception& e) {
    return fail(GMCP_ERR_ARG, e.what());
  }
}

ContactSurface to_surface(const gmcp_surface* s) {
  ContactSurface cs;
  cs.tris.resize(s->n_tris);
  cs.tri_edges.resize(s->n_tris);
  for (int t = 0; t < s->n_tris; ++t)
    for (int k = 0; k < 3; ++k) {
      cs.tris[t][k] = s->tris[3 * t + k];
      cs.tri_edges[t][k] = s->tri_edges[3 * t + k];
    }
  cs.edges.resize(s->n_edges);
  for (int e = 0; e < s->n_edges; ++e) cs.edges[e] = {s->edges[2 * e], s->edges[2 * e + 1]};
  cs.verts.assign(s->verts, s->verts + s->n_verts);
  return cs;
}

int64_t max_vertex(const gmcp_surface* s) {
  int64_t m = -1;
  for (int i = 0; i < 3 * s->n_tris; ++i) m = std::max<int64_t>(m, s->tris[i]);
  return m;
}

BarrierParams to_params(const gmcp_barrier_params* p) {
  BarrierParams b;
  b.kappa_face = p->kappa_face;
  b.kappa_edge = p->kappa_edge;
  b.kappa_point = p->kappa_point;
  b.eps_max = p->eps_max;
  b.delta_face = p->delta_face;
  b.delta_edge = p->delta_edge;
  b.detection_radius = p->detection_radius;
  b.quad_order_face = p->quad_order_face;
  b.quad_order_edge = p->quad_order_edge;
  return b;
}

void from_params(const BarrierParams& b, gmcp_barrier_params* p) {
  p->kappa_face = b.kappa_face;
  p->kappa_edge = b.kappa_edge;
  p->kappa_point = b.kappa_point;
  p->eps_max = b.eps_max;
  p->delta_face = b.delta_face;
  p->delta_edge = b.delta_edge;
  p->detection_radius = b.detection_radius;
  p->quad_order_face = b.quad_order_face;
  p->quad_order_edge = b.quad_order_edge;
}

VecX to_vec(const double* x, int64_t n) {
  VecX v(n);
  for (int64_t i = 0; i < n; ++i) v[i] = x[i];
  return v;
}

}  // namespace

struct orc_pairs {
  ContactPairSet set;
};
struct orc_state {
  ContactState state;
  int64_t n_dof = 0;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_is_reference(void) { return 1; }

int orc_resolve_barrier_params(gmcp_barrier_params* p, double mean_slave_edge) {
  return guarded([&] {
    from_params(resolve_barrier_params(to_params(p), mean_slave_edge), p);
    return GMCP_OK;
  });
}

int orc_mean_edge_length(const gmcp_surface* s, const double* x, double* out) {
  return guarded([&] {
    const ContactSurface cs = to_surface(s);
    int64_t nv = 0;
    for (const auto& e : cs.edges) nv = std::max<int64_t>(nv, e[1] + 1);
    *out = mean_edge_length(cs, to_vec(x, 3 * nv));
    return GMCP_OK;
  });
}

int orc_barrier(double g, double eps, double* out) {
  return guarded([&] {
    const BarrierEval b = barrier(g, eps);
    out[0] = b.B;
    out[1] = b.dB;
    out[2] = b.ddB;
    return GMCP_OK;
  });
}

int orc_build_candidate_pairs(const gmcp_surface* slave, const gmcp_surface* master,
                              const double* x, double r, int use_tree, orc_pairs** out) {
  return guarded([&] {
    const int64_t nv = std::max(max_vertex(slave), max_vertex(master)) + 1;
    auto* p = new orc_pairs;
    try {
      p->set = build_candidate_pairs(to_surface(slave), to_surface(master), to_vec(x, 3 * nv), r,
                                     use_tree != 0);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
    return GMCP_OK;
  });
}

int orc_pairs_from_csr(int32_t n_st, const int64_t* tri_off, const int32_t* tri_ids,
                       const int64_t* edge_off, const int32_t* edge_ids, const int64_t* vert_off,
                       const int32_t* vert_ids, orc_pairs** out) {
  auto* p = new orc_pairs;
  p->set.per_slave_tri.resize(n_st);
  for (int st = 0; st < n_st; ++st) {
    auto& c = p->set.per_slave_tri[st];
    c.tris.assign(tri_ids + tri_off[st], tri_ids + tri_off[st + 1]);
    c.edges.assign(edge_ids + edge_off[st], edge_ids + edge_off[st + 1]);
    c.verts.assign(vert_ids + vert_off[st], vert_ids + vert_off[st + 1]);
  }
  *out = p;
  return GMCP_OK;
}

int64_t orc_pairs_size(const orc_pairs* p, int which) {
  int64_t n = 0;
  for (const auto& c : p->set.per_slave_tri)
    n += static_cast<int64_t>(which == 0 ? c.tris.size() : which == 1 ? c.edges.size() : c.verts.size());
  return n;
}
int32_t orc_pairs_slave_tris(const orc_pairs* p) {
  return static_cast<int32_t>(p->set.per_slave_tri.size());
}
void orc_pairs_copy(const orc_pairs* p, int which, int64_t* offsets, int32_t* ids) {
  int64_t k = 0;
  for (size_t st = 0; st < p->set.per_slave_tri.size(); ++st) {
    const auto& c = p->set.per_slave_tri[st];
    const auto& v = which == 0 ? c.tris : which == 1 ? c.edges : c.verts;
    if (offsets) offsets[st] = k;
    for (int id : v) {
      if (ids) ids[k] = id;
      ++k;
    }
  }
  if (offsets) offsets[p->set.per_slave_tri.size()] = k;
}
void orc_pairs_free(orc_pairs* p) { delete p; }

int orc_build_contact_state(const gmcp_surface* slave, const gmcp_surface* master,
                            const orc_pairs* pairs, const double* x, int64_t n_dof,
                            const gmcp_barrier_params* params, const double* eps_reference,
                            orc_state** out) {
  return guarded([&] {
    const VecX xv = to_vec(x, n_dof);
    VecX ref;
    if (eps_reference) ref = to_vec(eps_reference, n_dof);
    auto* s = new orc_state;
    try {
      s->state = build_contact_state(to_surface(slave), to_surface(master), pairs->set, xv,
                                     to_params(params), eps_reference ? &ref : nullptr);
    } catch (...) {
      delete s;
      throw;
    }
    s->n_dof = n_dof;
    *out = s;
    return GMCP_OK;
  });
}

int orc_state_from_samples(const gmcp_samples* in, const double* ref_x, int64_t n_dof,
                           orc_state** out) {
  auto* s = new orc_state;
  s->n_dof = n_dof;
  s->state.reference_positions = to_vec(ref_x, n_dof);
  s->state.samples.resize(in->n);
  for (int64_t i = 0; i < in->n; ++i) {
    ContactSample& c = s->state.samples[i];
    c.type = static_cast<SampleType>(in->type[i]);
    for (int k = 0; k < 3; ++k) {
      c.slave[k] = in->slave[3 * i + k];
      c.master[k] = in->master[3 * i + k];
      c.beta_s[k] = in->beta_s[3 * i + k];
      c.beta_m[k] = in->beta_m[3 * i + k];
    }
    c.eta = in->eta[i];
    c.weight = in->weight[i];
    c.gamma = in->gamma[i];
    c.eps = in->eps[i];
    c.g_ref = in->g_ref[i];
  }
  *out = s;
  return GMCP_OK;
}

int64_t orc_state_size(const orc_state* s) { return static_cast<int64_t>(s->state.samples.size()); }

void orc_state_copy(const orc_state* s, gmcp_samples* o) {
  for (size_t i = 0; i < s->state.samples.size(); ++i) {
    const ContactSample& c = s->state.samples[i];
    o->type[i] = static_cast<int8_t>(c.type);
    for (int k = 0; k < 3; ++k) {
      o->slave[3 * i + k] = c.slave[k];
      o->master[3 * i + k] = c.master[k];
      o->beta_s[3 * i + k] = c.beta_s[k];
      o->beta_m[3 * i + k] = c.beta_m[k];
    }
    o->eta[i] = c.eta;
    o->weight[i] = c.weight;
    o->gamma[i] = c.gamma;
    o->eps[i] = c.eps;
    o->g_ref[i] = c.g_ref;
  }
}
void orc_state_free(orc_state* s) { delete s; }

int orc_sample_gap(const orc_state* s, int64_t i, const double* x, double* g) {
  return guarded([&] {
    *g = sample_gap(s->state.samples.at(i), to_vec(x, s->n_dof));
    return GMCP_OK;
  });
}

int orc_kinematics(const orc_state* s, const double* x, double* g, int32_t* nv, int32_t* ids,
                   double* dg) {
  return guarded([&] {
    const VecX xv = to_vec(x, s->n_dof);
    for (size_t i = 0; i < s->state.samples.size(); ++i) {
      const SampleKinematics k = sample_kinematics(s->state.samples[i], xv);
      g[i] = k.g;
      nv[i] = k.nv;
      for (int v = 0; v < 6; ++v) {
        ids[6 * i + v] = v < k.nv ? k.ids[v] : -1;
        for (int a = 0; a < 3; ++a) dg[18 * i + 3 * v + a] = v < k.nv ? k.dg[v][a] : 0.0;
      }
    }
    return GMCP_OK;
  });
}

int orc_try_contact_energy(const orc_state* s, const gmcp_barrier_params* p, const double* x,
                           double* energy, double* min_gap, int32_t* feasible) {
  return guarded([&] {
    const ContactEnergyResult r = try_contact_energy(s->state, to_params(p), to_vec(x, s->n_dof));
    *energy = r.energy;
    *min_gap = r.min_gap;
    *feasible = r.feasible ? 1 : 0;
    return GMCP_OK;
  });
}

int orc_contact_energy(const orc_state* s, const gmcp_barrier_params* p, const double* x,
                       double* energy, int64_t* bad) {
  *bad = -1;
  try {
    *energy = contact_energy(s->state, to_params(p), to_vec(x, s->n_dof));
    return GMCP_OK;
  } catch (const InfeasibleGapError& e) {
    *bad = e.sample_id;
    return fail(GMCP_ERR_INFEASIBLE, e.what());
  } catch (const std::exception& e) {
    return fail(GMCP_ERR_ARG, e.what());
  }
}

int orc_add_contact_gradient(const orc_state* s, const gmcp_barrier_params* p, const double* x,
                             double* grad, double* energy, int64_t* bad) {
  *bad = -1;
  try {
    VecX gv = to_vec(grad, s->n_dof);
    *energy = add_contact_gradient(s->state, to_params(p), to_vec(x, s->n_dof), gv);
    for (int64_t i = 0; i < s->n_dof; ++i) grad[i] = gv[i];
    return GMCP_OK;
  } catch (const InfeasibleGapError& e) {
    *bad = e.sample_id;
    return fail(GMCP_ERR_INFEASIBLE, e.what());
  } catch (const std::exception& e) {
    return fail(GMCP_ERR_ARG, e.what());
  }
}

int orc_add_contact_gradient_hessian(const orc_state* s, const gmcp_barrier_params* p,
                                     const double* x, double* grad, double* energy,
                                     int64_t* bad, int64_t* n_blocks, int32_t* brow,
                                     int32_t* bcol, double* bval, int64_t* n_triplets) {
  *bad = -1;
  try {
    VecX gv = to_vec(grad, s->n_dof);
    std::vector<Eigen::Triplet<Real>> trips;
    *energy = add_contact_gradient_hessian(s->state, to_params(p), to_vec(x, s->n_dof), gv, trips);
    for (int64_t i = 0; i < s->n_dof; ++i) grad[i] = gv[i];
    if (n_triplets) *n_triplets = static_cast<int64_t>(trips.size());
    // setFromTriplets: duplicates summed in insertion order
    std::map<std::pair<int, int>, std::array<double, 9>> blocks;
    for (const auto& t : trips) {
      auto it = blocks.find({t.row() / 3, t.col() / 3});
      if (it == blocks.end()) {
        std::array<double, 9> z{};
        it = blocks.emplace(std::make_pair(t.row() / 3, t.col() / 3), z).first;
      }
      double& e = it->second[3 * (t.row() % 3) + (t.col() % 3)];
      e = e + t.value();
    }
    *n_blocks = static_cast<int64_t>(blocks.size());
    if (brow) {
      int64_t k = 0;
      for (const auto& [key, v] : blocks) {
        brow[k] = key.first;
        bcol[k] = key.second;
        for (int j = 0; j < 9; ++j) bval[9 * k + j] = v[j];
        ++k;
      }
    }
    return GMCP_OK;
  } catch (const InfeasibleGapError& e) {
    *bad = e.sample_id;
    return fail(GMCP_ERR_INFEASIBLE, e.what());
  } catch (const std::exception& e) {
    return fail(GMCP_ERR_ARG, e.what());
  }
}

int orc_step_filter(const orc_state* s, const double* x, const double* dx, double* alpha) {
  return guarded([&] {
    *alpha = step_filter(s->state, to_vec(x, s->n_dof), to_vec(dx, s->n_dof));
    return GMCP_OK;
  });
}

int orc_displacement_cap(const orc_state* s, const gmcp_barrier_params* p, const double* x,
                         const double* dx, int64_t n_dof, double* alpha) {
  return guarded([&] {
    *alpha = displacement_cap(s->state, to_params(p), to_vec(x, s->n_dof), to_vec(dx, n_dof));
    return GMCP_OK;
  });
}

int orc_pressure_field(const orc_state* s, const gmcp_barrier_params* p, const double* x,
                       int64_t* n, gmcp_pressure_record* out) {
  return guarded([&] {
    const auto f = contact_pressure_field(s->state, to_params(p), to_vec(x, s->n_dof));
    *n = static_cast<int64_t>(f.size());
    if (out)
      for (size_t i = 0; i < f.size(); ++i) {
        out[i].sample = f[i].sample;
        for (int k = 0; k < 3; ++k) out[i].position[k] = f[i].position[k];
        out[i].radius = f[i].radius;
        out[i].gap = f[i].gap;
        out[i].pressure = f[i].pressure;
      }
    return GMCP_OK;
  });
}

int orc_force_summary(const orc_state* s, const gmcp_barrier_params* p, const double* x,
                      double* out) {
  return guarded([&] {
    const ContactForceSummary f = contact_force_summary(s->state, to_params(p), to_vec(x, s->n_dof));
    for (int k = 0; k < 3; ++k) {
      out[k] = f.face[k];
      out[3 + k] = f.edge[k];
      out[6 + k] = f.point[k];
      out[9 + k] = f.total[k];
    }
    return GMCP_OK;
  });
}

int orc_time_assembly(const orc_state* s, const gmcp_barrier_params* p, const double* x, int32_t reps,
                      double* best_seconds, int64_t* n_triplets) {
  return guarded([&] {
    const VecX xv = to_vec(x, s->n_dof);
    const BarrierParams bp = to_params(p);
    double best = 1e300;
    for (int r = 0; r < reps; ++r) {
      VecX grad = VecX::Zero(s->n_dof);
      std::vector<Eigen::Triplet<Real>> trips;
      const auto t0 = std::chrono::steady_clock::now();
      add_contact_gradient_hessian(s->state, bp, xv, grad, trips);
      const auto t1 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
      *n_triplets = static_cast<int64_t>(trips.size());
    }
    *best_seconds = best;
    return GMCP_OK;
  });
}

// ---------------------------------------------------------------------------
// ref_* helpers: mesh generators / boundary extraction (tet_mesh.hpp:56-168,
// contact_sampling.hpp:226-255) and whole-scene solves (solver.hpp:125-228).

int ref_make_block(const double* size, const int32_t* div, const double* origin, int64_t* nv,
                   double* verts, int64_t* nt, int32_t* tets) {
  return guarded([&] {
    const TetMesh m = make_block(Vec3(size[0], size[1], size[2]), {div[0], div[1], div[2]},
                                 Vec3(origin[0], origin[1], origin[2]));
    *nv = static_cast<int64_t>(m.vertices.size());
    *nt = static_cast<int64_t>(m.tets.size());
    if (verts)
      for (size_t v = 0; v < m.vertices.size(); ++v)
        for (int k = 0; k < 3; ++k) verts[3 * v + k] = m.vertices[v][k];
    if (tets)
      for (size_t t = 0; t < m.tets.size(); ++t)
        for (int k = 0; k < 4; ++k) tets[4 * t + k] = m.tets[t][k];
    return GMCP_OK;
  });
}

// Boundary surface of a tet mesh: triangles in surface-local ids + vertex_map.
int ref_boundary_surface(const double* verts, int64_t nv, const int32_t* tets, int64_t nt,
                         int64_t* ntri, int32_t* tris, int64_t* nsv, int32_t* vmap) {
  return guarded([&] {
    TetMesh m;
    m.vertices.resize(nv);
    for (int64_t v = 0; v < nv; ++v) m.vertices[v] = Vec3(verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]);
    m.tets.resize(nt);
    for (int64_t t = 0; t < nt; ++t)
      for (int k = 0; k < 4; ++k) m.tets[t][k] = tets[4 * t + k];
    const SurfaceMesh s = extract_boundary_surface(m);
    *ntri = static_cast<int64_t>(s.triangles.size());
    *nsv = static_cast<int64_t>(s.vertex_map.size());
    if (tris)
      for (size_t t = 0; t < s.triangles.size(); ++t)
        for (int k = 0; k < 3; ++k) tris[3 * t + k] = s.triangles[t][k];
    if (vmap)
      for (size_t v = 0; v < s.vertex_map.size(); ++v) vmap[v] = s.vertex_map[v];
    return GMCP_OK;
  });
}

// make_contact_surface over (tris, vertex_map) with an optional subset.
// counts = {n_tris, n_edges, n_verts}; arrays may be null to count.
int ref_contact_surface(const int32_t* tris_local, int64_t ntri, const int32_t* vmap, int64_t nsv,
                        int32_t vertex_offset, const int32_t* subset, int64_t nsub, int64_t* counts,
                        int32_t* tris, int32_t* edges, int32_t* tri_edges, int32_t* verts) {
  return guarded([&] {
    SurfaceMesh s;
    s.triangles.resize(ntri);
    for (int64_t t = 0; t < ntri; ++t)
      for (int k = 0; k < 3; ++k) s.triangles[t][k] = tris_local[3 * t + k];
    s.vertex_map.assign(vmap, vmap + nsv);
    std::vector<int> sub;
    if (subset) sub.assign(subset, subset + nsub);
    const ContactSurface cs = make_contact_surface(s, vertex_offset, subset ? &sub : nullptr);
    counts[0] = static_cast<int64_t>(cs.tris.size());
    counts[1] = static_cast<int64_t>(cs.edges.size());
    counts[2] = static_cast<int64_t>(cs.verts.size());
    if (tris)
      for (size_t t = 0; t < cs.tris.size(); ++t)
        for (int k = 0; k < 3; ++k) {
          tris[3 * t + k] = cs.tris[t][k];
          tri_edges[3 * t + k] = cs.tri_edges[t][k];
        }
    if (edges)
      for (size_t e = 0; e < cs.edges.size(); ++e) {
        edges[2 * e] = cs.edges[e][0];
        edges[2 * e + 1] = cs.edges[e][1];
      }
    if (verts)
      for (size_t v = 0; v < cs.verts.size(); ++v) verts[v] = cs.verts[v];
    return GMCP_OK;
  });
}

// Patch test (bench.hpp:44-124) solved by the reference System::solve with the
// shim's stand-in LDL^T. out: x (n_dof), stats {newton_iters, rebuilds,
// backtracks, seconds, sigma_zz_err, sigma_spur, force_z}.
int ref_patch_test(double kappa, const int32_t* div_bottom, const int32_t* div_top,
                   int32_t load_steps, int64_t* n_dof, double* x_out, double* stats) {
  return guarded([&] {
    SceneConfig cfg = make_patch_scene(kappa, {div_bottom[0], div_bottom[1], div_bottom[2]},
                                       {div_top[0], div_top[1], div_top[2]});
    cfg.solver.load_steps = load_steps;
    System sys = build_scene(cfg);
    *n_dof = sys.x.size();
    if (!x_out) return GMCP_OK;
    const RunStats rs = sys.solve(cfg.solver);
    for (Eigen::Index d = 0; d < sys.x.size(); ++d) x_out[d] = sys.x[d];
    const PatchReport rep = patch_stress_metrics(sys, cfg.loads[0].pressure);
    const ContactForceSummary sum =
        contact_force_summary(sys.contacts[0].state, sys.contacts[0].params, sys.x);
    stats[0] = rs.total_newton_iters;
    stats[1] = rs.total_rebuilds;
    int bt = 0;
    for (const auto& s : rs.steps) bt += s.backtracks;
    stats[2] = bt;
    stats[3] = rs.wall_seconds;
    stats[4] = rep.sigma_zz_max_rel_err;
    stats[5] = rep.sigma_spur;
    stats[6] = sum.total.z();
    return GMCP_OK;
  });
}

// Hertz indentation meshes (bench.hpp:178-193) at a given refine.
static void put_mesh(const TetMesh& m, int64_t* nv, double* v, int64_t* nt, int32_t* t) {
  *nv = static_cast<int64_t>(m.vertices.size());
  *nt = static_cast<int64_t>(m.tets.size());
  if (v)
    for (size_t i = 0; i < m.vertices.size(); ++i)
      for (int k = 0; k < 3; ++k) v[3 * i + k] = m.vertices[i][k];
  if (t)
    for (size_t i = 0; i < m.tets.size(); ++i)
      for (int k = 0; k < 4; ++k) t[4 * i + k] = m.tets[i][k];
}

int ref_hertz_meshes(double refine, int64_t* nvb, double* vb, int64_t* ntb, int32_t* tb, int64_t* nvh,
                     double* vh, int64_t* nth, int32_t* th) {
  return guarded([&] {
    HertzConfig cfg;
    cfg.refine = refine;
    put_mesh(make_hertz_block(cfg), nvb, vb, ntb, tb);
    put_mesh(make_hertz_ball(cfg), nvh, vh, nth, th);
    return GMCP_OK;
  });
}

// run_hertz (bench.hpp:210-303). out[0..13]: peak, p0, contact_radius,
// alpha_H, outside_max, peak_rel_err, contact_radius_rel_err, applied_force,
// total_newton_iters, steps, kappa_face, wall_seconds, samples, total_rebuilds.
int ref_run_hertz(double refine, int32_t load_steps, double* out) {
  return guarded([&] {
    HertzConfig cfg;
    cfg.refine = refine;
    cfg.load_steps = load_steps;
    const HertzResult r = run_hertz(cfg);
    const double v[14] = {r.peak, r.oracle.p0, r.contact_radius, r.oracle.alpha_H, r.outside_max,
                          r.peak_rel_err, r.contact_radius_rel_err, r.applied_force,
                          (double)r.stats.total_newton_iters, (double)r.steps.size(), r.params.kappa_face,
                          r.stats.wall_seconds, (double)r.profile.size(), (double)r.stats.total_rebuilds};
    for (int k = 0; k < 14; ++k) out[k] = v[k];
    return GMCP_OK;
  });
}

// parse_scene + build_scene + System::solve (scene.hpp:155-449, solver.hpp:125)
// on a scene file. x_out (n_dof) may be null to query n_dof. stats[0..5]:
// total_newton_iters, total_rebuilds, steps, wall_seconds, newton_tol_used,
// final min gap; force_z_out[pair] = contact_force_summary(...).total per pair
// (3 doubles each, up to max_pairs pairs).
int ref_run_scene(const char* path, int64_t* n_dof, double* x_out, double* stats, double* force_out,
                  int32_t max_pairs) {
  return guarded([&] {
    const SceneConfig cfg = parse_scene(path);
    System sys = build_scene(cfg);
    *n_dof = sys.x.size();
    if (!x_out) return GMCP_OK;
    const RunStats rs = sys.solve(cfg.solver);
    for (Eigen::Index d = 0; d < sys.x.size(); ++d) x_out[d] = sys.x[d];
    stats[0] = rs.total_newton_iters;
    stats[1] = rs.total_rebuilds;
    stats[2] = (double)rs.steps.size();
    stats[3] = rs.wall_seconds;
    stats[4] = rs.newton_tol_used;
    stats[5] = rs.steps.empty() ? 0.0 : rs.steps.back().min_gap;
    for (int p = 0; p < (int)sys.contacts.size() && p < max_pairs; ++p) {
      const ContactForceSummary f = contact_force_summary(sys.contacts[p].state, sys.contacts[p].params, sys.x);
      for (int k = 0; k < 3; ++k) force_out[3 * p + k] = f.total[k];
    }
    return GMCP_OK;
  });
}

// build_scene arrays of a scene file (scene.hpp:382-449): f_ext, fixed mask,
// Dirichlet targets and the slave triangle count of each contact pair.
int ref_scene_arrays(const char* path, int64_t* n_dof, double* f_ext, uint8_t* fixed, double* dirichlet,
                     int64_t* slave_tris, int32_t max_pairs) {
  return guarded([&] {
    const SceneConfig cfg = parse_scene(path);
    System sys = build_scene(cfg);
    *n_dof = sys.x.size();
    if (!f_ext) return GMCP_OK;
    for (Eigen::Index d = 0; d < sys.x.size(); ++d) {
      f_ext[d] = sys.f_ext[d];
      fixed[d] = sys.fixed[d];
      dirichlet[d] = sys.dirichlet[d];
    }
    for (int p = 0; p < (int)sys.contacts.size() && p < max_pairs; ++p)
      slave_tris[p] = (int64_t)sys.contacts[p].slave.tris.size();
    return GMCP_OK;
  });
}

// The reference's own writers (vtk_io.hpp) on given arrays, for byte-level
// format pinning: <dir>/vol.vtk (tets + displacement + stress), <dir>/surf.vtk,
// <dir>/p.csv (7 columns as write_step_outputs), <dir>/report.txt.
int ref_write_formats(const char* dir, const double* pts, int64_t np, const int32_t* tets, int64_t nt,
                      const int32_t* tris, int64_t ntri, const double* disp, const double* stress,
                      const double* rows, int64_t nrows) {
  return guarded([&] {
    const std::string d(dir);
    std::vector<Vec3> points(np);
    for (int64_t i = 0; i < np; ++i) points[i] = Vec3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    std::vector<std::array<int, 4>> cells(nt);
    for (int64_t i = 0; i < nt; ++i)
      for (int k = 0; k < 4; ++k) cells[i][k] = tets[4 * i + k];
    std::vector<std::array<int, 3>> tr(ntri);
    for (int64_t i = 0; i < ntri; ++i)
      for (int k = 0; k < 3; ++k) tr[i][k] = tris[3 * i + k];
    GridField dsp{"displacement", 3, std::vector<Real>(disp, disp + 3 * np)};
    GridField sig{"cauchy_stress", 9, std::vector<Real>(stress, stress + 9 * nt)};
    save_vtk_tets(d + "/vol.vtk", points, cells, {dsp}, {sig});
    save_vtk_tris(d + "/surf.vtk", points, tr);
    std::vector<std::vector<Real>> rw(nrows);
    for (int64_t i = 0; i < nrows; ++i) rw[i].assign(rows + 7 * i, rows + 7 * i + 7);
    save_csv(d + "/p.csv", {"pair", "sample", "x", "y", "z", "gap", "pressure"}, rw);
    Report rep;
    rep.set("scene.path", std::string("a b.scene"));
    rep.set("scene.bodies", 3L);
    rep.set("x", 0.1);
    rep.set("y", -2.5e-300);
    rep.set("x", 1.0 / 3.0);
    rep.set("threads", 1);
    rep.save(d + "/report.txt");
    return GMCP_OK;
  });
}

// embedding.hpp:26-106 (the reference's own functions)
static SurfaceMesh host_mesh(const double* host_v, int64_t n_hv, const int32_t* host_t, int64_t n_ht) {
  SurfaceMesh h;
  h.vertices.resize(n_hv);
  for (int64_t v = 0; v < n_hv; ++v) h.vertices[v] = Vec3(host_v[3 * v], host_v[3 * v + 1], host_v[3 * v + 2]);
  h.triangles.resize(n_ht);
  for (int64_t t = 0; t < n_ht; ++t)
    for (int k = 0; k < 3; ++k) h.triangles[t][k] = host_t[3 * t + k];
  return h;
}

int orc_embed_in_surface(const double* points, int64_t n_points, const double* host_v, int64_t n_hv,
                         const int32_t* host_t, int64_t n_ht, int32_t use_tree, int32_t* tri, double* bary,
                         double* offset, int64_t* bad) {
  *bad = -1;
  const SurfaceMesh h = host_mesh(host_v, n_hv, host_t, n_ht);
  for (int64_t t = 0; t < n_ht; ++t) {  // the index the reference's message names
    const auto& tr = h.triangles[t];
    if (!((h.vertices[tr[1]] - h.vertices[tr[0]]).cross(h.vertices[tr[2]] - h.vertices[tr[0]]).norm() > 0)) {
      *bad = t;
      break;
    }
  }
  return guarded([&] {
    std::vector<Vec3> pts(n_points);
    for (int64_t i = 0; i < n_points; ++i) pts[i] = Vec3(points[3 * i], points[3 * i + 1], points[3 * i + 2]);
    const SurfaceEmbedding e = embed_in_surface(pts, h, use_tree != 0);
    for (int64_t i = 0; i < n_points; ++i) {
      tri[i] = e[i].tri;
      for (int k = 0; k < 3; ++k) bary[3 * i + k] = e[i].bary[k];
      offset[i] = e[i].offset;
    }
    return GMCP_OK;
  });
}

int orc_apply_embedding(const int32_t* tri, const double* bary, const double* offset, int64_t n,
                        const int32_t* host_t, int64_t n_ht, const double* host_x, int64_t n_hv, double* out,
                        int64_t* bad) {
  *bad = -1;
  SurfaceEmbedding e(n);
  for (int64_t i = 0; i < n; ++i) {
    e[i].tri = tri[i];
    e[i].bary = Vec3(bary[3 * i], bary[3 * i + 1], bary[3 * i + 2]);
    e[i].offset = offset[i];
  }
  std::vector<std::array<int, 3>> ht(n_ht);
  for (int64_t t = 0; t < n_ht; ++t)
    for (int k = 0; k < 3; ++k) ht[t][k] = host_t[3 * t + k];
  std::vector<Vec3> hx(n_hv);
  for (int64_t v = 0; v < n_hv; ++v) hx[v] = Vec3(host_x[3 * v], host_x[3 * v + 1], host_x[3 * v + 2]);
  return guarded([&] {
    std::vector<Vec3> r;
    try {
      r = apply_embedding(e, ht, hx);
    } catch (const MeshError& me) {
      const std::string m = me.what();  // "host triangle <t> is degenerate ..."
      const auto p = m.find("host triangle ");
      if (p != std::string::npos) *bad = std::atoll(m.c_str() + p + 14);
      throw;
    }
    for (int64_t i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) out[3 * i + k] = r[i][k];
    return GMCP_OK;
  });
}

}  // extern "C"
