"""Dual-mesh embedding (embedding.hpp:26-106): the restated oracle against
the compiled reference, BITWISE (tree and brute-force reference paths), on
the reference's own test situations (test_embedding.cpp): off-surface points,
equidistant ties -> lowest index, rigid / affine host motion, degenerate
triangles reported by index. CPU only."""
import numpy as np
import pytest

from paper_2605_24339_b200 import scenes as S


def _host(div=(6, 5, 3), size=(1.0, 0.8, 0.5)):
    m = S.make_block(size, div)
    sm = S.extract_boundary_surface(m)
    return m.vertices[sm.vertex_map], sm.triangles


def _points(V, seed, n=400, spread=0.05):
    rng = np.random.default_rng(seed)
    lo, hi = V.min(0) - spread, V.max(0) + spread
    return rng.uniform(lo, hi, size=(n, 3))


def test_embed_restated_equals_reference(orc, ref):
    V, T = _host()
    P = np.concatenate([_points(V, 1), V[:37] + 1e-3, 0.5 * (V[T[:20, 0]] + V[T[:20, 1]])])  # incl. edge midpoints
    o = orc.embed_in_surface(P, V, T)
    for use_tree in (True, False):
        r = ref.embed_in_surface(P, V, T, use_tree)
        for a, b in zip(o, r):
            assert np.array_equal(a, b)


def test_equidistant_ties_lowest_index(orc, ref):  # test_embedding.cpp:90-99
    V, T = _host((2, 2, 1), (1.0, 1.0, 1.0))
    P = V.copy()  # every vertex touches several triangles at distance 0
    o = orc.embed_in_surface(P, V, T)
    r = ref.embed_in_surface(P, V, T, True)
    assert np.array_equal(o[0], r[0])
    for i, p in enumerate(P):
        touching = [t for t in range(T.shape[0]) if np.any(np.all(V[T[t]] == p, axis=1))]
        assert o[0][i] == min(touching)


def test_apply_rest_rigid_affine(orc, ref):  # test_embedding.cpp:72-155
    V, T = _host()
    P = _points(V, 2, 300, 0.02)
    tri, bary, off = orc.embed_in_surface(P, V, T)
    rest = orc.apply_embedding(tri, bary, off, T, V)
    assert np.array_equal(rest, ref.apply_embedding(tri, bary, off, T, V))
    assert np.max(np.abs(rest - P)) < 1e-12
    th = 0.3
    R = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1.0]])
    X = V @ R.T + np.array([0.1, -0.2, 0.3])
    o = orc.apply_embedding(tri, bary, off, T, X)
    assert np.array_equal(o, ref.apply_embedding(tri, bary, off, T, X))
    assert np.max(np.abs(o - (P @ R.T + np.array([0.1, -0.2, 0.3])))) < 1e-12


def test_degenerate_triangles_reported(orc, ref):  # test_embedding.cpp:200-227
    from pyoracle import OracleError
    V, T = _host()
    Vd = V.copy()
    Vd[T[7, 2]] = Vd[T[7, 0]]  # collapse triangle 7 (and its neighbours sharing the vertex)
    bads = []
    for o in (orc, ref):
        with pytest.raises(OracleError) as e:
            o.embed_in_surface(_points(V, 3, 10), Vd, T)
        bads.append(e.value.bad)
    assert bads[0] == bads[1] >= 0
    P = _points(V, 4, 200, 0.0)
    tri, bary, off = orc.embed_in_surface(P, V, T)
    X = V.copy()
    k = int(tri[5])
    X[T[k, 1]] = X[T[k, 0]]
    bads = []
    for o in (orc, ref):
        with pytest.raises(OracleError) as e:
            o.apply_embedding(tri, bary, off, T, X)
        bads.append(e.value.bad)
    assert bads[0] == bads[1] >= 0
