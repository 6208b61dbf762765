"""Pins the plain-C restated oracle (oracle/gmcp_oracle.c) against the
compiled reference (oracle/_ref, the unmodified reference headers): every
output is compared BITWISE on identical inputs. CPU only."""
import numpy as np
import pytest

import fixtures as F
from paper_2605_24339_b200 import scenes as S


def _scenes():
    pi = F.patch_interface()
    x = pi["rest"].reshape(-1, 3).copy()
    x[pi["off"]:, 2] -= 1.5e-3
    x_eval = F.random_active(7, x.ravel())
    dx = np.zeros_like(x)
    dx[pi["off"]:, 2] = -1e-3
    yield "patch", pi["slave"], pi["master"], pi["params"], pi["rest"], x_eval, F.random_active(8, dx.ravel())

    tp = F.tet_pair()
    yield "tetpair", tp["slave"], tp["master"], tp["params"], tp["rest"], F.random_active(3, tp["x"]), \
        F.random_active(4, np.zeros_like(tp["x"]), 1e-3)

    sl = S.slab_scene(12, 10, texture_amp=2e-4, seed=5)
    yield "slab12x10tex", sl.slave, sl.master, sl.params, sl.rest, sl.x_eval, sl.dx


SCENES = list(_scenes())


def _same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b)) or \
        (np.asarray(a).dtype.kind == "f" and np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True))


@pytest.mark.parametrize("scene", SCENES, ids=[s[0] for s in SCENES])
def test_restated_matches_reference_bitwise(scene, orc, ref):
    name, slave, master, params, rest, x, dx = scene
    pr = ref.candidate_pairs(slave, master, rest, params.detection_radius)
    po = orc.candidate_pairs(slave, master, rest, params.detection_radius)
    for k in ("tris", "edges", "verts"):
        assert _same(pr[k][0], po[k][0]) and _same(pr[k][1], po[k][1]), k
    sr = ref.contact_state(slave, master, pr, rest, params)
    so = orc.contact_state(slave, master, po, rest, params)
    a, b = sr.samples(), so.samples()
    assert len(sr) == len(so) > 0
    for k in a:
        assert _same(a[k], b[k]), f"sample field {k}"
    # anchored rebuild at the evaluation state (solver.hpp:146,153)
    x_near = rest + 0.3 * (x - rest)
    pr2 = ref.candidate_pairs(slave, master, x_near, params.detection_radius)
    sr2 = ref.contact_state(slave, master, pr2, x_near, params, eps_reference=rest)
    so2 = orc.contact_state(slave, master, pr2, x_near, params, eps_reference=rest)
    a2, b2 = sr2.samples(), so2.samples()
    for k in a2:
        assert _same(a2[k], b2[k]), f"anchored sample field {k}"

    assert sr.try_energy(params, x) == so.try_energy(params, x)
    assert sr.energy(params, x) == so.energy(params, x)
    er, gr = sr.gradient(params, x)
    eo, go = so.gradient(params, x)
    assert er == eo and _same(gr, go)
    hr, ho = sr.gradient_hessian(params, x), so.gradient_hessian(params, x)
    assert hr[0] == ho[0] and _same(hr[1], ho[1]) and hr[5] == ho[5]
    for i in (2, 3, 4):
        assert _same(hr[i], ho[i])
    assert sr.step_filter(x, dx) == so.step_filter(x, dx)
    assert sr.displacement_cap(params, x, dx) == so.displacement_cap(params, x, dx)
    assert _same(sr.pressure(params, x).view(np.uint8), so.pressure(params, x).view(np.uint8))
    assert _same(sr.force_summary(params, x), so.force_summary(params, x))
    kr, ko = sr.kinematics(x), so.kinematics(x)
    for u, v in zip(kr, ko):
        assert _same(u, v)


ORDERS = [(qf, qe) for qf in (1, 2, 3, 4) for qe in (1, 2, 3, 4, 5)]


@pytest.mark.parametrize("qf,qe", ORDERS, ids=[f"f{a}e{b}" for a, b in ORDERS])
@pytest.mark.parametrize("scene", [SCENES[0], SCENES[2]], ids=["patch", "slab12x10tex"])
def test_restated_matches_reference_every_quadrature_order(scene, qf, qe, orc, ref):
    """Every accepted (quad_order_face, quad_order_edge) pair (barrier.hpp:44-45,
    quadrature.hpp:20-81): samples, energy, gradient and summed Hessian blocks
    bitwise."""
    name, slave, master, p0, rest, x, dx = scene
    params = S.BarrierParams(**p0.__dict__)
    params.quad_order_face, params.quad_order_edge = qf, qe
    pr = ref.candidate_pairs(slave, master, rest, params.detection_radius)
    sr = ref.contact_state(slave, master, pr, rest, params)
    so = orc.contact_state(slave, master, pr, rest, params)
    a, b = sr.samples(), so.samples()
    assert len(sr) == len(so) > 0
    for k in a:
        assert _same(a[k], b[k]), f"sample field {k}"
    hr, ho = sr.gradient_hessian(params, x), so.gradient_hessian(params, x)
    assert hr[0] == ho[0] and _same(hr[1], ho[1]) and hr[5] == ho[5]
    for i in (2, 3, 4):
        assert _same(hr[i], ho[i])
    assert sr.step_filter(x, dx) == so.step_filter(x, dx)
    assert _same(sr.pressure(params, x).view(np.uint8), so.pressure(params, x).view(np.uint8))


def test_brute_force_equals_tree(ref):
    sl = S.slab_scene(9, 7, seed=1)
    a = ref.candidate_pairs(sl.slave, sl.master, sl.x_eval, sl.params.detection_radius, True)
    b = ref.candidate_pairs(sl.slave, sl.master, sl.x_eval, sl.params.detection_radius, False)
    for k in a:
        assert _same(a[k][1], b[k][1])


def test_infeasible_reports_first_sample(orc, ref):
    tp = F.tet_pair()
    p = tp["params"]
    pr = orc.candidate_pairs(tp["slave"], tp["master"], tp["rest"], p.detection_radius)
    so = orc.contact_state(tp["slave"], tp["master"], pr, tp["rest"], p)
    sr = ref.contact_state(tp["slave"], tp["master"], pr, tp["rest"], p)
    bad = tp["rest"].copy()
    bad[3 * 4 + 2::3][:4] -= 0.004  # test_contact.cpp:239-260
    from pyoracle import OracleError
    ids = []
    for st in (so, sr):
        e, mg, feas = st.try_energy(p, bad)
        assert not feas and mg <= 0
        with pytest.raises(OracleError) as ei:
            st.energy(p, bad)
        assert ei.value.code == 1 and "non-positive gap" in str(ei.value)
        ids.append(ei.value.bad)
    assert ids[0] == ids[1] >= 0


def test_python_generators_match_reference(ref):
    """scenes.py (numpy) reproduces make_block / extract_boundary_surface /
    make_contact_surface orderings of the reference."""
    import ctypes as C
    L = ref.lib
    for size, div, org in (((1, 1, 0.5), (5, 5, 2), (0, 0, 0)), ((1, 1, 0.1), (7, 6, 1), (0, 0, 0.102)),
                           ((0.3, 2, 1), (2, 3, 4), (1, -1, 0.5))):
        m = S.make_block(size, div, org)
        nv, nt = C.c_int64(), C.c_int64()
        sz, dv, og = np.array(size, float), np.array(div, np.int32), np.array(org, float)
        L.ref_make_block(C.c_void_p(sz.ctypes.data), C.c_void_p(dv.ctypes.data), C.c_void_p(og.ctypes.data), C.byref(nv), None, C.byref(nt), None)
        v = np.zeros((nv.value, 3))
        t = np.zeros((nt.value, 4), np.int32)
        L.ref_make_block(C.c_void_p(sz.ctypes.data), C.c_void_p(dv.ctypes.data), C.c_void_p(og.ctypes.data), C.byref(nv), C.c_void_p(v.ctypes.data),
                         C.byref(nt), C.c_void_p(t.ctypes.data))
        assert _same(v, m.vertices) and _same(t, m.tets)
        sm = S.extract_boundary_surface(m)
        ntri, nsv = C.c_int64(), C.c_int64()
        L.ref_boundary_surface(C.c_void_p(v.ctypes.data), nv, C.c_void_p(t.ctypes.data), nt, C.byref(ntri), None, C.byref(nsv), None)
        tris = np.zeros((ntri.value, 3), np.int32)
        vmap = np.zeros(nsv.value, np.int32)
        L.ref_boundary_surface(C.c_void_p(v.ctypes.data), nv, C.c_void_p(t.ctypes.data), nt, C.byref(ntri), C.c_void_p(tris.ctypes.data),
                               C.byref(nsv), C.c_void_p(vmap.ctypes.data))
        assert _same(tris, sm.triangles) and _same(vmap, sm.vertex_map)
        sub = np.arange(0, ntri.value, 3, dtype=np.int32)
        cs = S.make_contact_surface(sm, 17, sub)
        counts = np.zeros(3, np.int64)
        L.ref_contact_surface(C.c_void_p(tris.ctypes.data), ntri, C.c_void_p(vmap.ctypes.data), nsv, 17, C.c_void_p(sub.ctypes.data),
                              C.c_int64(sub.size), C.c_void_p(counts.ctypes.data), None, None, None, None)
        ct = np.zeros((counts[0], 3), np.int32)
        ce = np.zeros((counts[1], 2), np.int32)
        cte = np.zeros((counts[0], 3), np.int32)
        cv = np.zeros(counts[2], np.int32)
        L.ref_contact_surface(C.c_void_p(tris.ctypes.data), ntri, C.c_void_p(vmap.ctypes.data), nsv, 17, C.c_void_p(sub.ctypes.data),
                              C.c_int64(sub.size), C.c_void_p(counts.ctypes.data), C.c_void_p(ct.ctypes.data), C.c_void_p(ce.ctypes.data),
                              C.c_void_p(cte.ctypes.data), C.c_void_p(cv.ctypes.data))
        assert _same(ct, cs.tris) and _same(ce, cs.edges) and _same(cte, cs.tri_edges) and _same(cv, cs.verts)


def test_resolve_params_match(ref):
    pi = F.patch_interface()
    m = S.mean_edge_length(pi["slave"], pi["rest"])
    cp = ref.resolve_params(S.BarrierParams(kappa_face=1e6, eps_max=1e-3), m)
    p = pi["params"]
    assert (cp.kappa_edge, cp.kappa_point, cp.detection_radius) == (p.kappa_edge, p.kappa_point, p.detection_radius)


def test_hertz_generators_match_reference(ref):
    """graded lattices, cylinder sector, sphere octant and the Hertz meshes
    (mesh_gen.hpp, bench.hpp:178-193) bitwise against the reference."""
    import ctypes as C
    L = ref.lib
    for refine in (0.7, 1.0):
        n = [C.c_int64() for _ in range(4)]
        L.ref_hertz_meshes(C.c_double(refine), C.byref(n[0]), None, C.byref(n[1]), None, C.byref(n[2]), None,
                           C.byref(n[3]), None)
        vb, tb = np.zeros((n[0].value, 3)), np.zeros((n[1].value, 4), np.int32)
        vh, th = np.zeros((n[2].value, 3)), np.zeros((n[3].value, 4), np.int32)
        assert L.ref_hertz_meshes(C.c_double(refine), C.byref(n[0]), C.c_void_p(vb.ctypes.data), C.byref(n[1]),
                                  C.c_void_p(tb.ctypes.data), C.byref(n[2]), C.c_void_p(vh.ctypes.data),
                                  C.byref(n[3]), C.c_void_p(th.ctypes.data)) == 0
        cfg = S.HertzConfig(refine=refine)
        b, h = S.make_hertz_block(cfg), S.make_hertz_ball(cfg)
        assert _same(vb, b.vertices) and _same(tb, b.tets) and _same(vh, h.vertices) and _same(th, h.tets)


@pytest.mark.parametrize("refine,count", [(0.7, 4112), (1.0, 9495)])
def test_c1_hertz_sample_anchor(orc, refine, count):
    """Hertz at refine 0.7 -> 4,112 samples (9,495 at refine 1.0);
    kappa_face and the oracle constants as the reference's run_hertz."""
    sc = S.hertz_scene(S.HertzConfig(refine=refine))
    assert (sc.rest.size // 3, sc.slave.tris.shape[0], sc.master.tris.shape[0]) == \
        ((1253, 72, 720) if refine == 0.7 else (sc.rest.size // 3, sc.slave.tris.shape[0], sc.master.tris.shape[0]))
    st = orc.contact_state(sc.slave, sc.master, orc.candidate_pairs(sc.slave, sc.master, sc.rest,
                                                                    sc.params.detection_radius), sc.rest, sc.params)
    assert len(st) == count
    g = F.golden("hertz_ref.json")[str(refine)]
    assert sc.params.kappa_face == g["kappa_face"] and sc.oracle.p0 == g["p0"] and sc.oracle.alpha_H == g["alpha_H"]
    assert sc.applied_force == pytest.approx(g["applied_force"], rel=1e-14)
