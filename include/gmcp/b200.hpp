// Drop-in B200 backend for the reference's contact path (C++ side).
//
// Include AFTER the reference headers (proj/include/gmcp/*.hpp, Eigen 3.3+)
// and link libgmcp_b200.so. Every function exists twice: with the reference
// signature verbatim (runs on the calling thread's default_device(), so a
// call site only gains the gmcp::b200:: qualifier), and with a leading
// gmcp::b200::Device& (explicit device / stream ownership). Both take the
// reference's own types and rethrow the reference exceptions (core.hpp:25-56):
//
//   reference (proj/include/gmcp/)                      here (namespace gmcp::b200)
//   build_candidate_pairs   contact_sampling.hpp:281    build_candidate_pairs
//   build_contact_state     contact_sampling.hpp:382    build_contact_state
//   try_contact_energy      contact_energy.hpp:95       try_contact_energy
//   contact_energy          contact_energy.hpp:110      contact_energy
//   add_contact_gradient    contact_energy.hpp:126      add_contact_gradient
//   add_contact_gradient_hessian contact_energy.hpp:146 add_contact_gradient_hessian
//   step_filter             contact_energy.hpp:184      step_filter
//   displacement_cap        contact_energy.hpp:198      displacement_cap
//   contact_pressure_field  contact_energy.hpp:225      contact_pressure_field
//   contact_force_summary   contact_energy.hpp:253      contact_force_summary
//   System::solve           solver.hpp:125              solve(System&, ...)
//
// The per-call functions copy x / dx / grad between host and device (the
// drop-in compatibility path). solve() runs the whole load-stepping Newton
// loop device-resident and touches the host only at the StepCallback.
#pragma once

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../gmcp_b200.h"
#include "../gmcp_solver.h"

namespace gmcp::b200 {

namespace detail {

[[noreturn]] inline void rethrow(int rc, const char* msg, long bad = -1, Real residual = 0) {
  const std::string m = msg ? msg : "";
  switch (rc) {
    case GMCP_ERR_INFEASIBLE: throw InfeasibleGapError(m, bad);
    case GMCP_ERR_DEGENERATE: throw MeshError(m);
    case GMCP_ERR_CONFIG: throw ConfigError(m);
    case GMCP_ERR_PARSE: throw ParseError(m);
    case GMCP_ERR_SOLVER: throw SolverError(m, residual);
    default: throw Error("gmcp_b200: " + m);
  }
}
inline void check(int rc, long bad = -1) {
  if (rc != GMCP_OK) rethrow(rc, gmcp_last_error(), bad);
}

struct SurfaceArrays {
  std::vector<int32_t> tris, edges, tri_edges, verts;
  gmcp_surface c{};
  explicit SurfaceArrays(const ContactSurface& s) {
    for (const auto& t : s.tris) tris.insert(tris.end(), t.begin(), t.end());
    for (const auto& e : s.edges) edges.insert(edges.end(), e.begin(), e.end());
    for (const auto& t : s.tri_edges) tri_edges.insert(tri_edges.end(), t.begin(), t.end());
    verts.assign(s.verts.begin(), s.verts.end());
    c = gmcp_surface{(int32_t)s.tris.size(), tris.data(),      (int32_t)s.edges.size(),
                     edges.data(),           tri_edges.data(), (int32_t)s.verts.size(),
                     verts.data()};
  }
};

inline gmcp_barrier_params to_c(const BarrierParams& p) {
  return gmcp_barrier_params{p.kappa_face, p.kappa_edge,       p.kappa_point,     p.eps_max,        p.delta_face,
                             p.delta_edge, p.detection_radius, p.quad_order_face, p.quad_order_edge};
}

struct SampleArrays {
  std::vector<int8_t> type;
  std::vector<int32_t> slave, master;
  std::vector<double> beta_s, beta_m, eta, weight, gamma, eps, g_ref;
  gmcp_samples c{};
  void resize(size_t n) {
    type.resize(n);
    slave.resize(3 * n);
    master.resize(3 * n);
    beta_s.resize(3 * n);
    beta_m.resize(3 * n);
    eta.resize(n);
    weight.resize(n);
    gamma.resize(n);
    eps.resize(n);
    g_ref.resize(n);
    c = gmcp_samples{(int64_t)n,    type.data(), slave.data(), master.data(), beta_s.data(), beta_m.data(),
                     eta.data(),    weight.data(), gamma.data(), eps.data(),  g_ref.data()};
  }
  void from(const ContactState& st) {
    resize(st.samples.size());
    for (size_t i = 0; i < st.samples.size(); ++i) {
      const ContactSample& s = st.samples[i];
      type[i] = (int8_t)s.type;
      for (int k = 0; k < 3; ++k) {
        slave[3 * i + k] = s.slave[k];
        master[3 * i + k] = s.master[k];
        beta_s[3 * i + k] = s.beta_s[k];
        beta_m[3 * i + k] = s.beta_m[k];
      }
      eta[i] = s.eta;
      weight[i] = s.weight;
      gamma[i] = s.gamma;
      eps[i] = s.eps;
      g_ref[i] = s.g_ref;
    }
  }
  bool matches(const ContactState& st) const {
    const size_t n = st.samples.size();
    if (c.type == nullptr || type.size() != n) return false;
    auto same = [](double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; };
    for (size_t i = 0; i < n; ++i) {
      const ContactSample& s = st.samples[i];
      if (type[i] != (int8_t)s.type || !same(eta[i], s.eta) || !same(weight[i], s.weight) ||
          !same(gamma[i], s.gamma) || !same(eps[i], s.eps) || !same(g_ref[i], s.g_ref))
        return false;
      for (int k = 0; k < 3; ++k)
        if (slave[3 * i + k] != s.slave[k] || master[3 * i + k] != s.master[k] ||
            !same(beta_s[3 * i + k], s.beta_s[k]) || !same(beta_m[3 * i + k], s.beta_m[k]))
          return false;
    }
    return true;
  }
  void to(ContactState& st) const {
    st.samples.resize(type.size());
    for (size_t i = 0; i < type.size(); ++i) {
      ContactSample& s = st.samples[i];
      s.type = (SampleType)type[i];
      for (int k = 0; k < 3; ++k) {
        s.slave[k] = slave[3 * i + k];
        s.master[k] = master[3 * i + k];
        s.beta_s[k] = beta_s[3 * i + k];
        s.beta_m[k] = beta_m[3 * i + k];
      }
      s.eta = eta[i];
      s.weight = weight[i];
      s.gamma = gamma[i];
      s.eps = eps[i];
      s.g_ref = g_ref[i];
    }
  }
};

}  // namespace detail

// One GPU context (one CUDA stream). Caches the last uploaded ContactState by
// CONTENT: the reference reassigns a pair's state in place on a rebuild
// (solver.hpp:295), so neither the object's address nor its sample count
// identifies it. bind_state compares every field bitwise against the host
// copy of the samples it uploaded last (O(n) host work, no device traffic)
// and re-uploads on any difference.
class Device {
 public:
  explicit Device(int device = 0) { detail::check(gmcp_ctx_create(device, &ctx_)); }
  ~Device() { gmcp_ctx_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  gmcp_ctx* raw() { return ctx_; }

  void positions(const VecX& x) { detail::check(gmcp_set_positions(ctx_, x.data(), (int64_t)x.size())); }
  void step(const VecX& dx) { detail::check(gmcp_set_step(ctx_, dx.data(), (int64_t)dx.size())); }
  void params(const BarrierParams& p) {
    const gmcp_barrier_params c = detail::to_c(p);
    if (have_params_ && std::memcmp(&c, &params_, sizeof c) == 0) return;
    detail::check(gmcp_set_params(ctx_, &c));
    params_ = c;
    have_params_ = true;
  }
  void bind(const ContactState& st, const BarrierParams& p, const VecX& x) {
    positions(x);
    bind_state(st, p);
  }
  // params + samples only (the single-call entries take x themselves)
  void bind_state(const ContactState& st, const BarrierParams& p) {
    params(p);
    bind_samples(st);
  }
  // samples only (step_filter takes no params, contact_energy.hpp:184): keeps
  // the bound params, or binds placeholder stiffnesses the filter never reads
  void bind_samples(const ContactState& st) {
    if (!have_params_) {
      BarrierParams q;
      q.kappa_edge = q.kappa_point = q.kappa_face;
      params(q);
    }
    if (!bound_.matches(st)) {
      bound_.from(st);
      detail::check(gmcp_upload_samples(ctx_, &bound_.c));
      ++uploads_;
    }
  }
  // samples uploaded so far (a test hook for the content cache)
  long uploads() const { return uploads_; }

 private:
  gmcp_ctx* ctx_ = nullptr;
  detail::SampleArrays bound_;
  gmcp_barrier_params params_{};
  bool have_params_ = false;
  long uploads_ = 0;
};

// The device behind the reference-signature overloads below: one per host
// thread, on CUDA device GMCP_B200_DEVICE (default 0).
inline Device& default_device() {
  thread_local std::unique_ptr<Device> d;
  if (!d) {
    const char* e = std::getenv("GMCP_B200_DEVICE");
    d = std::make_unique<Device>(e ? std::atoi(e) : 0);
  }
  return *d;
}

inline ContactPairSet build_candidate_pairs(Device& d, const ContactSurface& slave, const ContactSurface& master,
                                            const VecX& x, Real detection_radius) {
  detail::SurfaceArrays s(slave), m(master);
  detail::check(gmcp_set_surfaces(d.raw(), &s.c, &m.c));
  d.positions(x);
  int64_t counts[3];
  detail::check(gmcp_broadphase(d.raw(), detection_radius, counts));
  ContactPairSet out;
  out.per_slave_tri.resize(slave.tris.size());
  for (int which = 0; which < 3; ++which) {
    std::vector<int64_t> off(slave.tris.size() + 1);
    std::vector<int32_t> ids((size_t)std::max<int64_t>(counts[which], 1));
    detail::check(gmcp_download_pairs(d.raw(), which, off.data(), ids.data()));
    for (size_t st = 0; st < slave.tris.size(); ++st) {
      auto& dst = which == 0 ? out.per_slave_tri[st].tris
                             : (which == 1 ? out.per_slave_tri[st].edges : out.per_slave_tri[st].verts);
      dst.assign(ids.begin() + off[st], ids.begin() + off[st + 1]);
    }
  }
  return out;
}

inline ContactState build_contact_state(Device& d, const ContactSurface& slave, const ContactSurface& master,
                                        const ContactPairSet& pairs, const VecX& x, const BarrierParams& params,
                                        const VecX* eps_reference = nullptr) {
  if (pairs.per_slave_tri.size() != slave.tris.size())
    throw ConfigError("build_contact_state: pair set does not match slave surface");
  detail::SurfaceArrays s(slave), m(master);
  detail::check(gmcp_set_surfaces(d.raw(), &s.c, &m.c));
  d.params(params);
  d.positions(x);
  std::vector<int64_t> off[3];
  std::vector<int32_t> ids[3];
  for (int w = 0; w < 3; ++w) {
    off[w].push_back(0);
    for (const auto& c : pairs.per_slave_tri) {
      const auto& v = w == 0 ? c.tris : (w == 1 ? c.edges : c.verts);
      ids[w].insert(ids[w].end(), v.begin(), v.end());
      off[w].push_back((int64_t)ids[w].size());
    }
  }
  detail::check(gmcp_upload_pairs(d.raw(), off[0].data(), ids[0].data(), off[1].data(), ids[1].data(),
                                  off[2].data(), ids[2].data()));
  int64_t n = 0;
  detail::check(gmcp_build_samples(d.raw(), eps_reference ? eps_reference->data() : nullptr, &n));
  detail::SampleArrays a;
  a.resize((size_t)n);
  detail::check(gmcp_download_samples(d.raw(), &a.c));
  ContactState st;
  st.reference_positions = x;
  a.to(st);
  return st;
}

inline ContactEnergyResult try_contact_energy(Device& d, const ContactState& st, const BarrierParams& p,
                                              const VecX& x) {
  d.bind(st, p, x);
  ContactEnergyResult r;
  int32_t feas = 1;
  detail::check(gmcp_try_energy(d.raw(), &r.energy, &r.min_gap, &feas));
  r.feasible = feas != 0;
  return r;
}

inline Real contact_energy(Device& d, const ContactState& st, const BarrierParams& p, const VecX& x) {
  d.bind(st, p, x);
  Real e = 0;
  int64_t bad = -1;
  const int rc = gmcp_energy(d.raw(), &e, &bad);
  if (rc) detail::rethrow(rc, gmcp_last_error(), (long)bad);
  return e;
}

inline Real add_contact_gradient(Device& d, const ContactState& st, const BarrierParams& p, const VecX& x,
                                 VecX& grad) {
  d.bind_state(st, p);
  Real e = 0;
  int64_t bad = -1;
  const int rc = gmcp_add_gradient(d.raw(), x.data(), (int64_t)x.size(), grad.data(), &e, &bad);
  if (rc) detail::rethrow(rc, gmcp_last_error(), (long)bad);
  return e;
}

// Emits the Gauss-Newton Hessian as triplets (the reference's interface); the
// device keeps the BCSR for the device-resident solver.
inline Real add_contact_gradient_hessian(Device& d, const ContactState& st, const BarrierParams& p, const VecX& x,
                                         VecX& grad, std::vector<Eigen::Triplet<Real>>& H) {
  d.bind_state(st, p);
  Real e = 0;
  int64_t bad = -1;
  const int rc = gmcp_add_gradient_hessian(d.raw(), x.data(), (int64_t)x.size(), grad.data(), &e, &bad);
  if (rc) detail::rethrow(rc, gmcp_last_error(), (long)bad);
  int64_t nnzb = 0;
  detail::check(gmcp_download_hessian(d.raw(), &nnzb, nullptr, nullptr, nullptr));
  std::vector<int32_t> rowptr(x.size() / 3 + 1), cols((size_t)nnzb);
  std::vector<double> vals(9 * (size_t)nnzb);
  detail::check(gmcp_download_hessian(d.raw(), &nnzb, rowptr.data(), cols.data(), vals.data()));
  for (size_t r = 0; r + 1 < rowptr.size(); ++r)
    for (int32_t k = rowptr[r]; k < rowptr[r + 1]; ++k)
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) {
          const double v = vals[9 * (size_t)k + 3 * a + c];
          if (v != 0) H.emplace_back((int)(3 * r + a), 3 * cols[k] + c, v);
        }
  return e;
}

inline Real step_filter(Device& d, const ContactState& st, const VecX& x, const VecX& dx) {
  d.positions(x);
  d.bind_samples(st);
  d.step(dx);
  Real a = 1;
  detail::check(gmcp_step_filter(d.raw(), &a));
  return a;
}

inline Real displacement_cap(Device& d, const ContactState& st, const BarrierParams& p, const VecX& x,
                             const VecX& dx) {
  d.bind(st, p, x);
  d.step(dx);
  Real a = 1;
  detail::check(gmcp_displacement_cap(d.raw(), &a));
  return a;
}

inline std::vector<PressureRecord> contact_pressure_field(Device& d, const ContactState& st, const BarrierParams& p,
                                                          const VecX& x) {
  d.bind(st, p, x);
  int64_t n = 0;
  detail::check(gmcp_pressure_field(d.raw(), &n, nullptr));
  std::vector<gmcp_pressure_record> raw((size_t)n);
  if (n) detail::check(gmcp_pressure_field(d.raw(), &n, raw.data()));
  std::vector<PressureRecord> out((size_t)n);
  for (size_t i = 0; i < raw.size(); ++i) {
    out[i].sample = (long)raw[i].sample;
    out[i].position = Vec3(raw[i].position[0], raw[i].position[1], raw[i].position[2]);
    out[i].radius = raw[i].radius;
    out[i].gap = raw[i].gap;
    out[i].pressure = raw[i].pressure;
  }
  return out;
}

inline ContactForceSummary contact_force_summary(Device& d, const ContactState& st, const BarrierParams& p,
                                                 const VecX& x) {
  d.bind(st, p, x);
  double o[12];
  detail::check(gmcp_force_summary(d.raw(), o));
  ContactForceSummary s;
  s.face = Vec3(o[0], o[1], o[2]);
  s.edge = Vec3(o[3], o[4], o[5]);
  s.point = Vec3(o[6], o[7], o[8]);
  s.total = Vec3(o[9], o[10], o[11]);
  return s;
}

// ---------------------------------------------------------------------------
// Reference signatures, verbatim (contact_sampling.hpp:281,382;
// contact_energy.hpp:95-276): a call site switches by qualifying the call
// with gmcp::b200:: and nothing else. They run on default_device().

inline ContactPairSet build_candidate_pairs(const ContactSurface& slave, const ContactSurface& master, const VecX& x,
                                            Real detection_radius, bool /*use_tree*/ = true) {
  // the tree and brute-force sets are identical (test_sampling.cpp:390-397); the LBVH always runs
  return build_candidate_pairs(default_device(), slave, master, x, detection_radius);
}
inline ContactState build_contact_state(const ContactSurface& slave, const ContactSurface& master,
                                        const ContactPairSet& pairs, const VecX& x, const BarrierParams& params,
                                        const VecX* eps_reference = nullptr) {
  return build_contact_state(default_device(), slave, master, pairs, x, params, eps_reference);
}
inline ContactEnergyResult try_contact_energy(const ContactState& st, const BarrierParams& p, const VecX& x) {
  return try_contact_energy(default_device(), st, p, x);
}
inline Real contact_energy(const ContactState& st, const BarrierParams& p, const VecX& x) {
  return contact_energy(default_device(), st, p, x);
}
inline Real add_contact_gradient(const ContactState& st, const BarrierParams& p, const VecX& x, VecX& grad) {
  return add_contact_gradient(default_device(), st, p, x, grad);
}
inline Real add_contact_gradient_hessian(const ContactState& st, const BarrierParams& p, const VecX& x, VecX& grad,
                                         std::vector<Eigen::Triplet<Real>>& H) {
  return add_contact_gradient_hessian(default_device(), st, p, x, grad, H);
}
inline Real step_filter(const ContactState& st, const VecX& x, const VecX& dx) {
  return step_filter(default_device(), st, x, dx);
}
inline Real displacement_cap(const ContactState& st, const BarrierParams& p, const VecX& x, const VecX& dx) {
  return displacement_cap(default_device(), st, p, x, dx);
}
inline std::vector<PressureRecord> contact_pressure_field(const ContactState& st, const BarrierParams& p,
                                                          const VecX& x) {
  return contact_pressure_field(default_device(), st, p, x);
}
inline ContactForceSummary contact_force_summary(const ContactState& st, const BarrierParams& p, const VecX& x) {
  return contact_force_summary(default_device(), st, p, x);
}

#ifdef GMCP_B200_WITH_SOLVER
// System::solve on the device (solver.hpp:125-228). Bodies are rebuilt from
// the reference System's element operators (tets) and rest positions;
// Dirichlet dofs, loads and contact pairs are copied as configured.
inline RunStats solve(System& sys, const SolverSettings& settings, const System::StepCallback& on_step = nullptr,
                      int device = 0, Real pcg_tol = 1e-10, int pcg_max_iters = 20000) {
  gmcp_system* h = nullptr;
  if (int rc = gmcp_system_create(device, &h)) detail::rethrow(rc, gmcp_system_last_error());
  std::unique_ptr<gmcp_system, void (*)(gmcp_system*)> guard(h, gmcp_system_destroy);
  auto chk = [](int rc, Real res = 0) {
    if (rc) detail::rethrow(rc, gmcp_system_last_error(), -1, res);
  };
  for (const Body& b : sys.bodies) {
    std::vector<double> v(3 * (size_t)b.num_vertices);
    for (int i = 0; i < 3 * b.num_vertices; ++i) v[i] = sys.rest[3 * b.vertex_offset + i];
    std::vector<int32_t> t;
    for (const auto& op : b.ops) t.insert(t.end(), op.verts.begin(), op.verts.end());
    int32_t off = 0;
    chk(gmcp_system_add_body(h, v.data(), b.num_vertices, t.data(), (int64_t)b.ops.size(), b.material.E,
                             b.material.nu, &off));
  }
  std::vector<int64_t> dofs;
  std::vector<double> tg;
  for (size_t d = 0; d < sys.fixed.size(); ++d)
    if (sys.fixed[d]) {
      dofs.push_back((int64_t)d);
      tg.push_back(sys.dirichlet[d]);
    }
  chk(gmcp_system_fix_dofs(h, (int64_t)dofs.size(), dofs.data(), tg.data()));
  chk(gmcp_system_set_external_force(h, sys.f_ext.data(), sys.f_ext.size()));
  chk(gmcp_system_set_positions(h, sys.x.data(), sys.x.size()));
  for (const auto& pair : sys.contacts) {
    detail::SurfaceArrays s(pair.slave), m(pair.master);
    const gmcp_barrier_params c = detail::to_c(pair.params);
    int32_t id = 0;
    chk(gmcp_system_add_contact_pair(h, &s.c, &m.c, &c, &id));
  }
  struct Ctx {
    const System::StepCallback* cb;
    RunStats* rs;
    System* sys;
  };
  RunStats rs;
  Ctx ctx{&on_step, &rs, &sys};
  auto tramp = [](const gmcp_step_stats* s, const double* x, int64_t n, void* user) {
    auto* c = static_cast<Ctx*>(user);
    StepStats ss;
    ss.step = s->step;
    ss.newton_iters = s->newton_iters;
    ss.rebuilds = s->rebuilds;
    ss.backtracks = s->backtracks;
    ss.residual = s->residual;
    ss.energy = s->energy;
    ss.min_gap = s->min_gap;
    ss.energy_monotone = s->energy_monotone != 0;
    c->rs->steps.push_back(ss);
    for (int64_t i = 0; i < n; ++i) c->sys->x[i] = x[i];
    if (*c->cb) (*c->cb)(ss, c->sys->x);
  };
  gmcp_solver_settings st{settings.load_steps, settings.max_newton_iters, settings.newton_tol,
                          settings.max_line_search, pcg_tol, pcg_max_iters};
  gmcp_run_stats out{};
  if (int rc = gmcp_system_solve(h, &st, tramp, &ctx, &out))
    detail::rethrow(rc, gmcp_system_last_error(), -1, out.residual);
  chk(gmcp_system_positions(h, sys.x.data(), sys.x.size()));
  rs.newton_tol_used = out.newton_tol_used;
  rs.wall_seconds = out.wall_seconds;
  rs.total_newton_iters = (int)out.total_newton_iters;
  rs.total_rebuilds = (int)out.total_rebuilds;
  return rs;
}
#endif

}  // namespace gmcp::b200
