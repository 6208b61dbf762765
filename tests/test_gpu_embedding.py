"""Dual-mesh embedding on the device against the restated oracle (itself
pinned bitwise to the reference in test_embedding_oracle.py): bindings,
barycentrics, offsets and reconstructions BITWISE, including equidistant
ties and degenerate-triangle errors; plus a large visual mesh."""
import numpy as np
import pytest

from paper_2605_24339_b200 import embedding as EM
from paper_2605_24339_b200 import gmcp as gm
from paper_2605_24339_b200 import scenes as S

pytestmark = pytest.mark.gpu


def _host(div=(6, 5, 3), size=(1.0, 0.8, 0.5)):
    m = S.make_block(size, div)
    sm = S.extract_boundary_surface(m)
    return m.vertices[sm.vertex_map], sm.triangles


def test_embed_and_apply_bitwise(orc):
    V, T = _host()
    rng = np.random.default_rng(11)
    P = np.concatenate([rng.uniform(V.min(0) - 0.05, V.max(0) + 0.05, size=(3000, 3)), V + 0.0,
                        0.5 * (V[T[:, 0]] + V[T[:, 1]])])  # vertices / edge midpoints: exact ties
    e = EM.embed_in_surface(P, V, T)
    o = orc.embed_in_surface(P, V, T)
    assert np.array_equal(e.tri, o[0]) and np.array_equal(e.bary, o[1]) and np.array_equal(e.offset, o[2])
    X = V * np.array([1.1, 0.9, 1.05]) + 0.01 * np.sin(7 * V)
    assert np.array_equal(EM.apply_embedding(e, T, X), orc.apply_embedding(*o, T, X))
    assert np.max(np.abs(EM.apply_embedding(e, T, V) - P)) < 1e-12  # rest reconstruction


def test_large_visual_mesh_matches_oracle(orc):
    sl = S.slab_scene(40, 32)  # host: the pad surface
    m = sl.meshes[1]
    sm = S.extract_boundary_surface(m)
    V, T = m.vertices[sm.vertex_map], sm.triangles
    rng = np.random.default_rng(5)
    P = V[rng.integers(0, V.shape[0], 20000)] + rng.normal(0, 2e-3, size=(20000, 3))
    e = EM.embed_in_surface(P, V, T)
    o = orc.embed_in_surface(P[:2000], V, T)
    assert np.array_equal(e.tri[:2000], o[0]) and np.array_equal(e.bary[:2000], o[1])
    assert np.array_equal(e.offset[:2000], o[2])


def test_degenerate_errors_name_the_triangle(orc):
    from pyoracle import OracleError
    V, T = _host()
    Vd = V.copy()
    Vd[T[7, 2]] = Vd[T[7, 0]]
    with pytest.raises(gm.MeshError):
        EM.embed_in_surface(V[:5], Vd, T)
    with pytest.raises(OracleError) as oe:
        orc.embed_in_surface(V[:5], Vd, T)
    ctx = gm.Context(0)
    import ctypes as C
    bad = C.c_int64(-1)
    P = np.ascontiguousarray(V[:5])
    tri, bary, off = np.zeros(5, np.int32), np.zeros((5, 3)), np.zeros(5)
    rc = ctx.L.gmcp_embed_in_surface(ctx.h, gm._p(P), C.c_int64(5), gm._p(Vd), C.c_int64(Vd.shape[0]),
                                     gm._p(np.ascontiguousarray(T, np.int32)), C.c_int64(T.shape[0]), gm._p(tri),
                                     gm._p(bary), gm._p(off), C.byref(bad))
    assert rc == gm.GMCP_ERR_DEGENERATE and bad.value == oe.value.bad
    e = EM.embed_in_surface(V[:40] + 1e-3, V, T)
    X = V.copy()
    k = int(e.tri[3])
    X[T[k, 1]] = X[T[k, 0]]
    with pytest.raises(gm.MeshError) as me:
        EM.apply_embedding(e, T, X)
    with pytest.raises(OracleError) as oe2:
        orc.apply_embedding(e.tri, e.bary, e.offset, T, X)
    assert f"host triangle {oe2.value.bad} " in str(me.value)
