"""GPU parity: the CUDA contact kernels vs the CPU oracle on identical inputs.

Samples come from the oracle (uploaded through the C-ABI), so these tests pin
the per-iteration kernels independently of the GPU sampler. Tolerances follow
SURVEY.md 8d: energy 1e-9 relative; gradient / pressure / Hessian norm-wise
1e-9 relative; step filter and displacement cap bit-exact (min/max are
order-free and the kernels are compiled without FMA contraction)."""
import numpy as np
import pytest

import fixtures as F
from paper_2605_24339_b200 import scenes as S

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _cases():
    pi = F.patch_interface()
    x = pi["rest"].reshape(-1, 3).copy()
    x[pi["off"]:, 2] -= 1.5e-3
    dx = np.zeros_like(x)
    dx[pi["off"]:, 2] = -1e-3
    yield "patch", pi["slave"], pi["master"], pi["params"], pi["rest"], F.random_active(7, x.ravel()), \
        F.random_active(8, dx.ravel())
    tp = F.tet_pair()
    yield "tetpair", tp["slave"], tp["master"], tp["params"], tp["rest"], F.random_active(3, tp["x"]), \
        F.random_active(4, np.zeros_like(tp["x"]), 1e-3)
    sl = S.slab_scene(20, 16, texture_amp=2e-4, seed=5)
    yield "slab20x16tex", sl.slave, sl.master, sl.params, sl.rest, sl.x_eval, sl.dx
    sl = S.slab_scene(50, 40, seed=11)  # C2: ~106k samples
    yield "C2", sl.slave, sl.master, sl.params, sl.rest, sl.x_eval, sl.dx


CASES = list(_cases())


@pytest.fixture(scope="module")
def gm():
    from paper_2605_24339_b200 import gmcp
    return gmcp


def _setup(gm, orc, case):
    name, slave, master, params, rest, x, dx = case
    pairs = orc.candidate_pairs(slave, master, rest, params.detection_radius)
    ost = orc.contact_state(slave, master, pairs, rest, params)
    ctx = gm.Context(0)
    ctx.set_params(params)
    ctx.set_positions(x)
    ctx.set_step(dx)
    ctx.upload_samples(ost.samples())
    return ctx, ost


def _rel_inf(a, b):
    s = max(np.abs(b).max(), 1e-300)
    return np.abs(a - b).max() / s


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_energy_gradient_hessian_filter(case, gm, orc):
    name, slave, master, params, rest, x, dx = case
    ctx, ost = _setup(gm, orc, case)
    assert ctx.num_samples() == len(ost) > 0

    e_o, mg_o, f_o = ost.try_energy(params, x)
    e_g, mg_g, f_g = ctx.try_energy()
    assert f_o and f_g
    assert abs(e_g - e_o) <= TOL * abs(e_o)
    assert mg_g == mg_o  # min is order-free
    assert abs(ctx.energy() - ost.energy(params, x)) <= TOL * abs(e_o)

    eo, go = ost.gradient(params, x)
    g = np.zeros_like(x)
    eg = ctx.gradient(g)
    assert abs(eg - eo) <= TOL * abs(eo)
    assert _rel_inf(g, go) <= TOL

    eh, gh, brow, bcol, bval, ntrip = ost.gradient_hessian(params, x)
    g2 = np.zeros_like(x)
    ctx.gradient(g2, hessian=True)
    assert _rel_inf(g2, gh) <= TOL
    rowptr, cols, vals = ctx.download_hessian()
    rows = np.repeat(np.arange(rowptr.size - 1), np.diff(rowptr))
    # every oracle block present in the GPU pattern, values within tolerance
    key_g = {(int(r), int(c)): k for k, (r, c) in enumerate(zip(rows, cols))}
    scale = np.abs(bval).max()
    dense_err = 0.0
    seen = np.zeros(len(cols), bool)
    for k in range(len(brow)):
        j = key_g[(int(brow[k]), int(bcol[k]))]
        seen[j] = True
        dense_err = max(dense_err, np.abs(vals[j] - bval[k]).max())
    if (~seen).any():  # pattern blocks the oracle never emitted must be zero-valued within tol
        dense_err = max(dense_err, np.abs(vals[~seen]).max())
    assert dense_err <= TOL * scale
    # exact symmetry (test_contact.cpp:125)
    for (r, c), j in key_g.items():
        assert np.array_equal(vals[j], vals[key_g[(c, r)]].T)

    a_o = ost.step_filter(x, dx)
    a_g = ctx.step_filter()
    assert a_g == a_o  # bit-exact
    assert ctx.displacement_cap() == ost.displacement_cap(params, x, dx)

    po, pg = ost.pressure(params, x), ctx.pressure_field()
    assert np.array_equal(po["sample"], pg["sample"])
    assert np.array_equal(po["gap"], pg["gap"]) and np.array_equal(po["position"], pg["position"])
    assert _rel_inf(pg["pressure"], po["pressure"]) <= TOL
    assert _rel_inf(pg["gap"], po["gap"]) <= TOL
    assert _rel_inf(pg["position"], po["position"]) <= TOL

    fo, fg = ost.force_summary(params, x), ctx.force_summary()
    assert _rel_inf(fg, fo) <= 1e-8

    ko, kg = ost.kinematics(x), ctx.kinematics()
    for u, v in zip(ko, kg):  # no-FMA translation unit: bitwise
        assert np.array_equal(u, v)


def test_assembly_is_bitwise_deterministic(gm, orc):
    ctx, ost = _setup(gm, orc, CASES[2])
    g1, g2 = np.zeros(ctx.n_dof), np.zeros(ctx.n_dof)
    e1 = ctx.gradient(g1, hessian=True)
    v1 = ctx.download_hessian()[2].copy()
    e2 = ctx.gradient(g2, hessian=True)
    v2 = ctx.download_hessian()[2]
    assert e1 == e2 and np.array_equal(g1, g2) and np.array_equal(v1, v2)


def test_single_call_host_path_equals_two_calls(gm, orc):
    """gmcp_add_gradient_hessian (x and grad in one call, transfers overlapped)
    gives bitwise the energy, accumulated gradient and Hessian of
    set_positions + gradient_hessian; the caller's buffer is accumulated into."""
    name, slave, master, params, rest, x, dx = CASES[3]
    ctx, ost = _setup(gm, orc, CASES[3])
    g0 = np.random.default_rng(5).standard_normal(x.size)
    g1 = g0.copy()
    ctx.set_positions(x)
    e1 = ctx.gradient(g1, hessian=True)
    v1 = ctx.download_hessian()[2].copy()
    ctx.set_positions(rest)  # the single call must install x itself
    g2 = g0.copy()
    e2 = ctx.add_gradient(x, g2, hessian=True)
    v2 = ctx.download_hessian()[2]
    assert e1 == e2 and np.array_equal(g1, g2) and np.array_equal(v1, v2)
    g3 = g0.copy()
    e3 = ctx.add_gradient(x, g3, hessian=False)
    assert e3 == e1 and np.array_equal(g3, g1)
    eo, go = ost.gradient(params, x)
    assert _rel_inf(g2 - g0, go) <= 1e-8


def test_single_call_infeasible_leaves_grad(gm, orc):
    tp = F.tet_pair()
    case = ("tp", tp["slave"], tp["master"], tp["params"], tp["rest"], tp["rest"], np.zeros_like(tp["rest"]))
    ctx, ost = _setup(gm, orc, case)
    bad = tp["rest"].copy()
    bad[3 * 4 + 2::3][:4] -= 0.004  # test_contact.cpp:239-260
    from pyoracle import OracleError
    with pytest.raises(OracleError) as eo:
        ost.energy(tp["params"], bad)
    g = np.arange(bad.size, dtype=np.float64)
    with pytest.raises(gm.InfeasibleGapError) as ei:
        ctx.add_gradient(bad, g, hessian=True)
    assert ei.value.sample_id == eo.value.bad and "non-positive gap" in str(ei.value)
    assert np.array_equal(g, np.arange(bad.size, dtype=np.float64))


def test_infeasible_names_first_sample(gm, orc):
    tp = F.tet_pair()
    case = ("tp", tp["slave"], tp["master"], tp["params"], tp["rest"], tp["rest"], np.zeros_like(tp["rest"]))
    ctx, ost = _setup(gm, orc, case)
    bad = tp["rest"].copy()
    bad[3 * 4 + 2::3][:4] -= 0.004  # test_contact.cpp:239-260
    ctx.set_positions(bad)
    e, mg, feas = ctx.try_energy()
    e_o, mg_o, feas_o = ost.try_energy(tp["params"], bad)
    assert not feas and mg == mg_o and mg <= 0
    from pyoracle import OracleError
    with pytest.raises(OracleError) as eo:
        ost.energy(tp["params"], bad)
    with pytest.raises(gm.InfeasibleGapError) as ei:
        ctx.energy()
    assert ei.value.sample_id == eo.value.bad and "non-positive gap" in str(ei.value)
    with pytest.raises(gm.InfeasibleGapError) as ei2:
        ctx.gradient(np.zeros_like(bad))
    assert ei2.value.sample_id == eo.value.bad


def _point_state(gm, beta_s, eps, x, masters=(3,), betas=None, grefs=None):
    n = len(masters)
    s = {k: np.zeros((n, w) if w > 1 else n, dtype=dt) for k, dt, w in gm.SAMPLE_FIELDS}
    s["type"][:] = gm.POINT
    s["slave"][:] = [0, 1, 2]
    s["master"][:] = -1
    s["master"][:, 0] = masters
    s["beta_s"][:] = beta_s if betas is None else betas
    s["weight"][:] = 1
    s["gamma"][:] = 1
    s["eps"][:] = eps
    s["g_ref"][:] = eps if grefs is None else grefs
    return s


def test_step_filter_known_answers(gm):
    """test_contact.cpp:164-214 / acceptance.cpp criterion 3."""
    p = S.resolve_barrier_params(S.BarrierParams(), 1.0)
    x = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 0.25, 0.25, 0.01], float)
    st = gm.state_from_samples(_point_state(gm, [0.5, 0.25, 0.25], 0.01, x), p, x)
    dx = np.zeros_like(x)
    dx[3 * 3 + 2] = -0.02
    a = gm.step_filter(st, x, dx)
    assert abs(a - 0.45) <= 1e-12
    x6 = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 0.25, 0.25, 0.01, 0.5, 0.25, 0.012, 0.25, 0.5, 0.012], float)
    st3 = gm.state_from_samples(_point_state(gm, None, 0.01, x6, masters=(3, 4, 5),
                                             betas=[[0.5, 0.25, 0.25], [0.25, 0.5, 0.25], [0.25, 0.25, 0.5]]),
                                p, x6)
    dx = np.zeros_like(x6)
    dx[3 * 3 + 2], dx[3 * 4 + 2], dx[3 * 5 + 2] = -0.02, -0.036, -0.009
    assert abs(gm.step_filter(st3, x6, dx) - 0.3) <= 1e-12
    dx[:] = 0
    dx[3 * 3 + 2] = dx[3 * 4 + 2] = dx[3 * 5 + 2] = 0.5
    assert gm.step_filter(st3, x6, dx) == 1.0


def test_displacement_cap_known_answers(gm):
    """test_contact.cpp:216-237."""
    p = S.resolve_barrier_params(S.BarrierParams(eps_max=0.002), 1.0)
    x = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 0.25, 0.25, 0.001], float)
    st = gm.state_from_samples(_point_state(gm, [0.5, 0.25, 0.25], 0.002, x), p, x)
    dx = np.zeros_like(x)
    dx[9] = 0.01
    assert abs(gm.displacement_cap(st, p, x, dx) - 0.1) <= 1e-15
    dx[9] = 0.0009
    assert gm.displacement_cap(st, p, x, dx) == 1.0
    far = x.copy()
    far[11] = 0.5
    dx[9] = 100.0
    assert gm.displacement_cap(st, p, far, dx) == 1.0


def test_pressure_known_answer(gm, orc):
    """test_contact.cpp:262-302."""
    gap, eps = 0.0005, 0.001
    s0 = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    x = np.concatenate([s0.ravel(), (s0 + [0, 0, gap]).ravel()])
    smp = {k: np.zeros((1, w) if w > 1 else 1, dtype=dt) for k, dt, w in gm.SAMPLE_FIELDS}
    smp["type"][:] = gm.FACE
    smp["slave"][:] = [0, 1, 2]
    smp["master"][:] = [3, 4, 5]
    smp["beta_s"][:] = [0.2, 0.5, 0.3]
    smp["beta_m"][:] = [0.2, 0.5, 0.3]
    smp["weight"][:] = 0.2
    smp["gamma"][:] = 0.7
    smp["eps"][:] = eps
    smp["g_ref"][:] = gap
    p = S.resolve_barrier_params(S.BarrierParams(eps_max=eps), 1.0)
    st = gm.state_from_samples(smp, p, x)
    rec = gm.contact_pressure_field(st, p, x)
    assert rec.size == 1 and rec["sample"][0] == 0
    assert abs(rec["gap"][0] - gap) <= 1e-12 * gap
    B = orc.barrier(gap, eps)
    expected = p.kappa_face * 0.7 * (-B[1])
    assert expected > 0 and abs(rec["pressure"][0] - expected) <= 1e-12 * expected
    x2 = x.copy()
    x2[[11, 14, 17]] = 0.002
    assert gm.contact_pressure_field(st, p, x2)["pressure"][0] == 0.0


def test_rest_state_is_silent(gm, orc):
    """test_contact.cpp:155-162 / acceptance criterion 8: exactly zero at build."""
    pi = F.patch_interface()
    case = ("patch", pi["slave"], pi["master"], pi["params"], pi["rest"], pi["rest"], np.zeros_like(pi["rest"]))
    ctx, ost = _setup(gm, orc, case)
    assert ctx.energy() == 0.0
    g = np.zeros_like(pi["rest"])
    ctx.gradient(g, hessian=True)
    assert not g.any()
    assert not ctx.download_hessian()[2].any()
