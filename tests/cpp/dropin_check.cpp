// Drop-in check: the reference's own scene/types driven through the B200
// backend (include/gmcp/b200.hpp) next to the reference CPU functions.
// Built by tests/test_cpp_dropin.py against the reference headers + the
// oracle's Eigen shim (test infrastructure). Exit 0 = all checks passed,
// 3 = no CUDA device (nothing to run), 1 = mismatch.
#include "gmcp/bench.hpp"

#define GMCP_B200_WITH_SOLVER
#include "gmcp/b200.hpp"

#include <cstdio>

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
  // per-iteration functions
  const Real er = contact_energy(sr, pair.params, x), eg = b200::contact_energy(dev, sr, pair.params, x);
  CHECK(std::abs(er - eg) <= 1e-9 * std::abs(er), "energy %.17g vs %.17g", er, eg);
  VecX gr = VecX::Zero(x.size()), gg = VecX::Zero(x.size());
  add_contact_gradient(sr, pair.params, x, gr);
  b200::add_contact_gradient(dev, sr, pair.params, x, gg);
  CHECK((gr - gg).lpNorm<Eigen::Infinity>() <= 1e-9 * gr.lpNorm<Eigen::Infinity>(), "gradient");
  VecX dx = VecX::Zero(x.size());
  for (int v = sys.bodies[1].vertex_offset; v < sys.num_vertices(); ++v) dx[3 * v + 2] = -1e-3;
  CHECK(step_filter(sr, x, dx) == b200::step_filter(dev, sr, pair.params, x, dx), "step filter");
  std::vector<Eigen::Triplet<Real>> H;
  VecX gh = VecX::Zero(x.size());
  b200::add_contact_gradient_hessian(dev, sr, pair.params, x, gh, H);
  CHECK(!H.empty(), "hessian triplets");
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
