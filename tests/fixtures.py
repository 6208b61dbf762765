"""Shared scene fixtures mirroring the reference tests' geometry."""
import numpy as np

from paper_2605_24339_b200 import scenes as S


def patch_interface(kappa=1e6, div_bottom=(5, 5, 2), div_top=(4, 4, 2)):
    """make_patch_scene geometry (bench.hpp:44-99): slave = bottom face of the
    top block, master = whole boundary of the bottom block."""
    bottom = S.make_block((1, 1, 0.5), div_bottom)
    top = S.make_block((1, 1, 0.5), div_top, (0, 0, 0.502))
    off = bottom.vertices.shape[0]
    rest = np.concatenate([bottom.vertices.ravel(), top.vertices.ravel()])
    sb, st = S.extract_boundary_surface(bottom), S.extract_boundary_surface(top)
    z = top.vertices[st.vertex_map[st.triangles], 2]
    sel = np.nonzero(np.all((z >= 0.5019) & (z <= 0.5021), axis=1))[0]
    slave = S.make_contact_surface(st, off, sel)
    master = S.make_contact_surface(sb, 0)
    p = S.resolve_barrier_params(S.BarrierParams(kappa_face=kappa, eps_max=1e-3),
                                 S.mean_edge_length(slave, rest))
    return dict(rest=rest, off=off, slave=slave, master=master, params=p)


def tet_pair():
    """TetPair of test_contact.cpp:32-66: two single tets 2 mm apart; master
    pushed 0.8 mm closer so face, edge and point samples are active."""
    sv = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.3, 0.3, -1]], float)
    mv = np.array([[0, 0, 0.002], [1, 0, 0.002], [0, 1, 0.002], [0.3, 0.3, 1.002]], float)
    slave_m = S.TetMesh(sv, S.orient_tets_positive(sv, np.array([[0, 1, 2, 3]])).astype(np.int32))
    master_m = S.TetMesh(mv, S.orient_tets_positive(mv, np.array([[0, 1, 2, 3]])).astype(np.int32))
    rest = np.concatenate([sv.ravel(), mv.ravel()])
    slave = S.make_contact_surface(S.extract_boundary_surface(slave_m), 0)
    master = S.make_contact_surface(S.extract_boundary_surface(master_m), 4)
    p = S.resolve_barrier_params(S.BarrierParams(eps_max=0.01, detection_radius=0.05),
                                 S.mean_edge_length(slave, rest))
    x = rest.copy()
    x[3 * 4 + 2::3][:4] -= 0.0008
    return dict(rest=rest, x=x, slave=slave, master=master, params=p)


def random_active(seed, x, amp=1e-4):
    rng = np.random.default_rng(seed)
    return x + rng.uniform(-amp, amp, size=x.size)
