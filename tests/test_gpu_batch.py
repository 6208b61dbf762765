"""C5 batched scenes: independent Hertz scenes packed into one
context with per-vertex scene ids. The packed broadphase and sampler must
equal the concatenation of the per-scene oracle results BITWISE (no pair
crosses scenes, although the scenes overlap in space), and the packed
energy / gradient / Hessian blocks must match the per-scene oracle sums."""
import numpy as np
import pytest

from paper_2605_24339_b200 import scenes as S

pytestmark = pytest.mark.gpu


def _per_scene(orc, b, k, x):
    N = b.v_off[1] - b.v_off[0]
    xs = x[3 * b.v_off[k]:3 * b.v_off[k + 1]]
    rest = b.rest[3 * b.v_off[k]:3 * b.v_off[k + 1]]
    sl, ms = b.base.slave, b.base.master
    po = orc.candidate_pairs(sl, ms, rest, b.params.detection_radius)
    st = orc.contact_state(sl, ms, po, rest, b.params)
    return N, po, st, xs


def test_batched_scenes_bitwise_per_scene(orc):
    from paper_2605_24339_b200 import gmcp as gm
    b = S.c5_batch(1024, first=5, count=4)
    ctx = gm.Context(0)
    ctx.set_params(b.params)
    ctx.set_surfaces(b.slave, b.master)
    ctx.set_positions(b.rest)
    ctx.set_vertex_scenes(b.vscene)
    ctx.broadphase(b.params.detection_radius)
    pg = ctx.download_pairs()
    n = ctx.build_samples()
    sg = ctx.download_samples()
    nst = b.base.slave.tris.shape[0]
    n_mt, n_me = b.base.master.tris.shape[0], b.base.master.edges.shape[0]
    n_mv = b.base.master.verts.shape[0]
    s0 = 0
    E = 0.0
    ctx.set_positions(b.x_eval)
    g = np.zeros(b.rest.size)
    e_gpu = ctx.gradient(g, hessian=True)
    for k in range(4):
        N, po, st, xs = _per_scene(orc, b, k, b.x_eval)
        # candidate sets: scene k's slave tris, ids shifted into the packed surfaces
        for key, shift in (("tris", n_mt * k), ("edges", n_me * k), ("verts", n_mv * k)):
            off, ids = pg[key]
            o0, o1 = off[nst * k], off[nst * (k + 1)]
            assert np.array_equal(off[nst * k:nst * (k + 1) + 1] - o0, po[key][0]), key
            assert np.array_equal(ids[o0:o1] - shift, po[key][1]), key
        so = st.samples()
        m = so["type"].size
        for f in so:
            a = sg[f][s0:s0 + m]
            if f in ("slave", "master"):
                a = np.where(a >= 0, a - b.v_off[k], a)
            assert np.array_equal(a, so[f]), f"scene {k}: field {f}"
        s0 += m
        ek, gk = st.gradient(b.params, xs)
        E += ek
        gs = g[3 * b.v_off[k]:3 * b.v_off[k + 1]]
        assert np.max(np.abs(gs - gk)) <= 1e-9 * np.max(np.abs(gk))
    assert n == s0
    assert e_gpu == pytest.approx(E, rel=1e-9)


def test_single_scene_ids_match_plain_context():
    """scene ids all zero == no scene ids (same candidate sets)."""
    from paper_2605_24339_b200 import gmcp as gm
    b = S.c5_batch(1024, first=0, count=1)
    out = []
    for sc in (None, b.vscene):
        ctx = gm.Context(0)
        ctx.set_params(b.params)
        ctx.set_surfaces(b.slave, b.master)
        ctx.set_positions(b.rest)
        ctx.set_vertex_scenes(sc)
        ctx.broadphase(b.params.detection_radius)
        out.append(ctx.download_pairs())
    for key in ("tris", "edges", "verts"):
        assert all(np.array_equal(x, y) for x, y in zip(out[0][key], out[1][key]))
