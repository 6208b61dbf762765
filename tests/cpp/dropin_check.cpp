// Drop-in check: the reference's own scene/types driven through the B200
// backend (include/gmcp/b200.hpp) next to the reference CPU functions.
// Built by tests/test_cpp_dropin.py against the reference headers + the
// oracle's Eigen shim (test infrastructure). Exit 0 = all checks passed,
// 3 = no CUDA device (nothing to run), 1 = mismatch.
#include "gmcp/bench.hpp"

#define GMCP_B200_WITH_SOLVER
#include "gmcp/b200.hpp"

#include <cstdio>
#include <map>
#include <thread>

using namespace gmcp;

static int fails = 0;
#define CHECK(c, ...)                   \
  do {                                  \
    if (!(c)) {                         \
      std::printf("FAIL: " __VA_ARGS__); \
      std::printf("\n");                \
      ++fails;                          \
    }                                   \
  } while (0)

int main() {
  int ndev = 0;
  if (gmcp_device_count(&ndev) != GMCP_OK || ndev == 0) {
    std::printf("no CUDA device\n");
    return 3;
  }
  b200::Device dev(0);
  System sys = build_scene(make_patch_scene());
  auto& pair = sys.contacts[0];
  VecX x = sys.x;
  for (int v = sys.bodies[1].vertex_offset; v < sys.num_vertices(); ++v) x[3 * v + 2] -= 1.5e-3;

  // broadphase + sampler: bitwise equal
  const ContactPairSet pr = build_candidate_pairs(pair.slave, pair.master, sys.x, pair.params.detection_radius);
  const ContactPairSet pg = b200::build_candidate_pairs(dev, pair.slave, pair.master, sys.x, pair.params.detection_radius);
  for (size_t st = 0; st < pr.per_slave_tri.size(); ++st)
    CHECK(pr.per_slave_tri[st].tris == pg.per_slave_tri[st].tris && pr.per_slave_tri[st].edges == pg.per_slave_tri[st].edges &&
              pr.per_slave_tri[st].verts == pg.per_slave_tri[st].verts,
          "candidate set of slave tri %zu", st);
  const ContactState sr = build_contact_state(pair.slave, pair.master, pr, sys.x, pair.params);
  const ContactState sg = b200::build_contact_state(dev, pair.slave, pair.master, pg, sys.x, pair.params);
  CHECK(sr.samples.size() == sg.samples.size(), "sample count %zu vs %zu", sr.samples.size(), sg.samples.size());
  for (size_t i = 0; i < std::min(sr.samples.size(), sg.samples.size()); ++i) {
    const auto &a = sr.samples[i], &b = sg.samples[i];
    CHECK(a.type == b.type && a.slave == b.slave && a.master == b.master && a.beta_s == b.beta_s &&
              a.beta_m == b.beta_m && a.eta == b.eta && a.weight == b.weight && a.gamma == b.gamma && a.eps == b.eps &&
              a.g_ref == b.g_ref,
          "sample %zu differs", i);
  }
  // per-iteration functions (sg: the GPU-built state, bitwise equal to sr)
  const Real er = contact_energy(sr, pair.params, x), eg = b200::contact_energy(dev, sg, pair.params, x);
  CHECK(std::abs(er - eg) <= 1e-9 * std::abs(er), "energy %.17g vs %.17g", er, eg);
  VecX gr = VecX::Zero(x.size()), gg = VecX::Zero(x.size());
  add_contact_gradient(sr, pair.params, x, gr);
  const Real egg = b200::add_contact_gradient(dev, sr, pair.params, x, gg);
  CHECK((gr - gg).lpNorm<Eigen::Infinity>() <= 1e-9 * gr.lpNorm<Eigen::Infinity>(), "gradient");
  VecX dx = VecX::Zero(x.size());
  for (int v = sys.bodies[1].vertex_offset; v < sys.num_vertices(); ++v) dx[3 * v + 2] = -1e-3;
  CHECK(step_filter(sr, x, dx) == b200::step_filter(dev, sr, x, dx), "step filter");
  CHECK(displacement_cap(sr, pair.params, x, dx) == b200::displacement_cap(dev, sr, pair.params, x, dx),
        "displacement cap");
  {
    const ContactEnergyResult a = try_contact_energy(sr, pair.params, x), b = b200::try_contact_energy(dev, sr, pair.params, x);
    CHECK(a.feasible == b.feasible && a.min_gap == b.min_gap && std::abs(a.energy - b.energy) <= 1e-9 * std::abs(a.energy),
          "try_contact_energy");
  }
  // Gauss-Newton Hessian: the triplets of both sides summed per (row, col)
  // (setFromTriplets semantics, solver.hpp:343) agree to 1e-9 of max |H|
  {
    std::vector<Eigen::Triplet<Real>> Hr, Hg;
    VecX ghr = VecX::Zero(x.size()), ghg = VecX::Zero(x.size());
    const Real ehr = add_contact_gradient_hessian(sr, pair.params, x, ghr, Hr);
    const Real ehg = b200::add_contact_gradient_hessian(dev, sr, pair.params, x, ghg, Hg);
    CHECK(std::abs(ehr - ehg) <= 1e-9 * std::abs(ehr), "hessian-call energy");
    CHECK((ghr - ghg).lpNorm<Eigen::Infinity>() <= 1e-9 * ghr.lpNorm<Eigen::Infinity>(), "hessian-call gradient");
    std::map<std::pair<long, long>, double> mr, mg;
    for (const auto& t : Hr) mr[{(long)t.row(), (long)t.col()}] += t.value();
    for (const auto& t : Hg) mg[{(long)t.row(), (long)t.col()}] += t.value();
    double hmax = 0, err = 0;
    for (const auto& [k, v] : mr) hmax = std::max(hmax, std::abs(v));
    for (const auto& [k, v] : mr) {
      auto it = mg.find(k);
      err = std::max(err, std::abs(v - (it == mg.end() ? 0.0 : it->second)));
    }
    for (const auto& [k, v] : mg)
      if (!mr.count(k)) err = std::max(err, std::abs(v));
    CHECK(!Hr.empty() && err <= 1e-9 * hmax, "hessian entries: max err %.3e of %.3e", err, hmax);
  }
  // pressure field and force summary
  {
    const auto pr_ = contact_pressure_field(sr, pair.params, x);
    const auto pg_ = b200::contact_pressure_field(dev, sr, pair.params, x);
    CHECK(pr_.size() == pg_.size() && !pr_.empty(), "pressure records %zu vs %zu", pr_.size(), pg_.size());
    double pmax = 0, perr = 0;
    for (const auto& r : pr_) pmax = std::max(pmax, std::abs(r.pressure));
    for (size_t i = 0; i < std::min(pr_.size(), pg_.size()); ++i) {
      CHECK(pr_[i].sample == pg_[i].sample && pr_[i].position == pg_[i].position && pr_[i].gap == pg_[i].gap,
            "pressure record %zu", i);
      perr = std::max(perr, std::abs(pr_[i].pressure - pg_[i].pressure));
    }
    CHECK(perr <= 1e-9 * pmax, "pressure values %.3e", perr);
    const ContactForceSummary fr = contact_force_summary(sr, pair.params, x);
    const ContactForceSummary fg = b200::contact_force_summary(dev, sr, pair.params, x);
    const double fs = fr.total.norm() + fr.face.norm() + fr.edge.norm() + fr.point.norm();
    CHECK((fr.face - fg.face).norm() + (fr.edge - fg.edge).norm() + (fr.point - fg.point).norm() +
                  (fr.total - fg.total).norm() <= 1e-9 * fs,
          "force summary");
  }
  // reference signatures verbatim (default device)
  CHECK(std::abs(b200::contact_energy(sr, pair.params, x) - er) <= 1e-9 * std::abs(er), "verbatim contact_energy");
  CHECK(b200::step_filter(sr, x, dx) == step_filter(sr, x, dx), "verbatim step_filter");
  // a state reassigned IN PLACE with the same sample count (the reference's
  // rebuild_pair, solver.hpp:295): the content cache must see the new samples
  {
    ContactState st = build_contact_state(pair.slave, pair.master, pr, sys.x, pair.params);
    const Real e0 = b200::contact_energy(dev, st, pair.params, x);
    CHECK(std::abs(e0 - er) <= 1e-9 * std::abs(er), "bound state energy");
    VecX anchor = sys.x;
    // anchor gap 0.5 mm: eps = 0.9 g_ref = 0.45 mm instead of eps_max = 1 mm (contact_sampling.hpp:471-485)
    for (int v = sys.bodies[1].vertex_offset; v < sys.num_vertices(); ++v) anchor[3 * v + 2] -= 1.5e-3;
    const size_t n0 = st.samples.size();
    st = build_contact_state(pair.slave, pair.master, pr, sys.x, pair.params, &anchor);
    CHECK(st.samples.size() == n0, "in-place rebuild keeps the sample count (%zu vs %zu)", st.samples.size(), n0);
    const Real e1r = contact_energy(st, pair.params, x), e1g = b200::contact_energy(dev, st, pair.params, x);
    CHECK(e1r != er && std::abs(e1g - e1r) <= 1e-9 * std::abs(e1r), "in-place rebuild: %.17g vs %.17g (stale %.17g)",
          e1g, e1r, er);
  }
  // two devices-contexts driven from two host threads at once (per-context
  // CUB scratch and device binding): results equal the single-thread ones
  {
    Real et[2] = {0, 0};
    VecX gt[2] = {VecX::Zero(x.size()), VecX::Zero(x.size())};
    auto work = [&](int k) {
      b200::Device d(0);
      for (int rep = 0; rep < 20; ++rep) {
        const ContactPairSet p2 = b200::build_candidate_pairs(d, pair.slave, pair.master, sys.x, pair.params.detection_radius);
        const ContactState s2 = b200::build_contact_state(d, pair.slave, pair.master, p2, sys.x, pair.params);
        gt[k].setZero();
        et[k] = b200::add_contact_gradient(d, s2, pair.params, x, gt[k]);
      }
    };
    std::thread t0(work, 0), t1(work, 1);
    t0.join();
    t1.join();
    CHECK(et[0] == egg && et[1] == egg, "threaded energies %.17g %.17g vs %.17g", et[0], et[1], egg);
    CHECK(gt[0] == gg && gt[1] == gg, "threaded gradients");
  }
  // infeasible -> InfeasibleGapError with the reference's index
  VecX bad = x;
  for (int v = sys.bodies[1].vertex_offset; v < sys.num_vertices(); ++v) bad[3 * v + 2] -= 0.01;
  long ir = -1, ig = -2;
  try { contact_energy(sr, pair.params, bad); } catch (const InfeasibleGapError& e) { ir = e.sample_id; }
  try { b200::contact_energy(dev, sr, pair.params, bad); } catch (const InfeasibleGapError& e) { ig = e.sample_id; }
  CHECK(ir == ig && ir >= 0, "infeasible index %ld vs %ld", ir, ig);

  // System::solve on the device
  System s2 = build_scene(make_patch_scene());
  const RunStats rs = b200::solve(s2, SolverSettings{});
  const PatchReport rep = patch_stress_metrics(s2, 10.0);
  CHECK(rs.steps.size() == 10, "load steps");
  CHECK(rep.sigma_zz_max_rel_err < 1e-2 && rep.sigma_spur < 1e-1, "patch metrics %g %g", rep.sigma_zz_max_rel_err,
        rep.sigma_spur);
  std::printf("dropin: samples=%zu energy=%.17g newton=%d zz=%.3e spur=%.3e fails=%d\n", sg.samples.size(), eg,
              rs.total_newton_iters, rep.sigma_zz_max_rel_err, rep.sigma_spur, fails);
  return fails ? 1 : 0;
}
