"""GPU parity for the rebuild path: LBVH broadphase candidate sets and the
mortar sampler are BIT-EXACT with the oracle (after the reference's own
canonical ordering, which both produce directly)."""
import numpy as np
import pytest

import fixtures as F
from paper_2605_24339_b200 import scenes as S

pytestmark = pytest.mark.gpu


def _cases():
    pi = F.patch_interface()
    x = pi["rest"].reshape(-1, 3).copy()
    x[pi["off"]:, 2] -= 1.0e-3
    yield "patch", pi["slave"], pi["master"], pi["params"], pi["rest"], F.random_active(21, x.ravel(), 2e-4)
    tp = F.tet_pair()
    yield "tetpair", tp["slave"], tp["master"], tp["params"], tp["rest"], tp["x"]
    sl = S.slab_scene(20, 16, texture_amp=2e-4, seed=5)
    yield "slab20x16tex", sl.slave, sl.master, sl.params, sl.rest, sl.rest + 0.5 * (sl.x_eval - sl.rest)
    sl = S.slab_scene(37, 29, seed=9)
    yield "slab37x29", sl.slave, sl.master, sl.params, sl.rest, sl.rest + 0.3 * (sl.x_eval - sl.rest)
    sl = S.slab_scene(50, 40, seed=11)  # C2
    yield "C2", sl.slave, sl.master, sl.params, sl.rest, None


CASES = list(_cases())


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_broadphase_and_sampler_bit_exact(case, orc):
    from paper_2605_24339_b200 import gmcp as gm
    name, slave, master, params, rest, x_later = case
    for x, eps_ref in ((rest, None),) + (((x_later, rest),) if x_later is not None else ()):
        ctx = gm.Context(0)
        ctx.set_params(params)
        ctx.set_surfaces(slave, master)
        ctx.set_positions(x)
        counts = ctx.broadphase(params.detection_radius)
        pg = ctx.download_pairs()
        po = orc.candidate_pairs(slave, master, x, params.detection_radius)
        for k in ("tris", "edges", "verts"):
            assert np.array_equal(pg[k][0], po[k][0]) and np.array_equal(pg[k][1], po[k][1]), k
        assert list(counts) == [po[k][1].size for k in ("tris", "edges", "verts")]
        n = ctx.build_samples(eps_ref)
        so = orc.contact_state(slave, master, po, x, params, eps_reference=eps_ref).samples()
        sg = ctx.download_samples()
        assert n == so["type"].size
        for k in so:
            assert np.array_equal(so[k], sg[k]), f"{name}: sample field {k}"


def test_self_contact_rejected():
    from paper_2605_24339_b200 import gmcp as gm
    sl = S.slab_scene(4, 3)
    ctx = gm.Context(0)
    ctx.set_params(sl.params)
    ctx.set_surfaces(sl.master, sl.master)
    ctx.set_positions(sl.rest)
    with pytest.raises(gm.ConfigError):
        ctx.broadphase(0.01)


def test_distant_bodies_no_candidates():
    """test_sampling.cpp:334-346."""
    from paper_2605_24339_b200 import gmcp as gm
    a = S.make_block((1, 1, 1), (1, 1, 1))
    b = S.make_block((1, 1, 1), (1, 1, 1), (0, 0, 5))
    rest = np.concatenate([a.vertices.ravel(), b.vertices.ravel()])
    sa = S.make_contact_surface(S.extract_boundary_surface(a), 0)
    sb = S.make_contact_surface(S.extract_boundary_surface(b), a.vertices.shape[0])
    pairs = gm.build_candidate_pairs(sa, sb, rest, 0.01)
    assert pairs.total_candidates() == 0


def test_empty_contact_state_through_every_entry():
    """No candidates -> no samples: every per-iteration entry is well defined
    on the empty state (the reference's loops simply do nothing): zero energy,
    the caller's gradient unchanged, an all-zero Hessian, alpha = 1, no
    pressure records, a zero force summary."""
    from paper_2605_24339_b200 import gmcp as gm
    a = S.make_block((1, 1, 1), (1, 1, 1))
    b = S.make_block((1, 1, 1), (1, 1, 1), (0, 0, 5))
    rest = np.concatenate([a.vertices.ravel(), b.vertices.ravel()])
    sa = S.make_contact_surface(S.extract_boundary_surface(a), 0)
    sb = S.make_contact_surface(S.extract_boundary_surface(b), a.vertices.shape[0])
    params = S.resolve_barrier_params(S.BarrierParams(), S.mean_edge_length(sa, rest))
    ctx = gm.Context(0)
    ctx.set_params(params)
    ctx.set_surfaces(sa, sb)
    ctx.set_positions(rest)
    ctx.broadphase(0.01)
    assert ctx.build_samples() == 0
    g0 = np.arange(rest.size, dtype=np.float64)
    g = g0.copy()
    assert ctx.add_gradient(rest, g, hessian=True) == 0.0
    assert np.array_equal(g, g0)
    g = g0.copy()
    ctx.set_positions(rest)
    assert ctx.gradient(g, hessian=True) == 0.0 and np.array_equal(g, g0)
    _, _, vals = ctx.download_hessian()
    assert not np.any(vals)
    e, mg, feas = ctx.try_energy()
    assert e == 0.0 and feas
    ctx.set_step(np.full(rest.size, -0.1))
    assert ctx.step_filter() == 1.0
    assert ctx.pressure_field()["pressure"].size == 0
    assert not np.any(ctx.force_summary())
