"""CPU study (scipy, no GPU): PCG iteration counts on the C2/C3-style slab Newton
matrix with the current block-Jacobi preconditioner vs a two-level additive
preconditioner (block-Jacobi + an aggregation coarse space of rigid-body modes).
It informs DESIGN.md 9 "next"; nothing here is on the product path.

The matrix is the one the device solver builds at the first Newton iteration of
build_slab_system (system.py): linear elastic K (E = 1000, nu = 0) + the contact
Gauss-Newton Hessian from the oracle at the slab's evaluation state, Dirichlet
dofs eliminated by the mask (P H P + I - P).

  python tools/precond_study.py [nb nt [agg ...]]  (default 50 40 = C2, agg 5 10)
  python tools/precond_study.py hertz [g ...]      (C1 / one C5 scene, g^3 grid aggregates)
"""
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2605_24339_b200 import scenes as S  # noqa: E402
from paper_2605_24339_b200.system import material, shape_gradients  # noqa: E402
from pyoracle import Oracle  # noqa: E402


def elastic_K(mesh, off, n_dof, E=1000.0, nu=0.0):
    lam, mu = material(E, nu)
    g, vol = shape_gradients(mesh.vertices, mesh.tets)  # (nt,4,3)
    nt = g.shape[0]
    # K_ab^{ij} = vol (lam g_a^i g_b^j + mu g_a^j g_b^i + mu delta_ij g_a . g_b)
    gg = np.einsum("tak,tbk->tab", g, g)
    K = (lam * np.einsum("tai,tbj->taibj", g, g) + mu * np.einsum("taj,tbi->taibj", g, g)
         + mu * np.einsum("tab,ij->taibj", gg, np.eye(3))) * np.abs(vol)[:, None, None, None, None]
    dof = 3 * (off + mesh.tets)[:, :, None] + np.arange(3)[None, None, :]  # (nt,4,3)
    rows = np.broadcast_to(dof[:, :, :, None, None], (nt, 4, 3, 4, 3)).ravel()
    cols = np.broadcast_to(dof[:, None, None, :, :], (nt, 4, 3, 4, 3)).ravel()
    return sp.csr_matrix((K.ravel(), (rows, cols)), shape=(n_dof, n_dof))


def build(nb, nt):
    sl = S.slab_scene(nb, nt)
    n = sl.rest.size
    H = elastic_K(sl.meshes[0], sl.offsets[0], n) + elastic_K(sl.meshes[1], sl.offsets[1], n)
    orc = Oracle("restated")
    pairs = orc.candidate_pairs(sl.slave, sl.master, sl.rest, sl.params.detection_radius)
    st = orc.contact_state(sl.slave, sl.master, pairs, sl.rest, sl.params)
    _, _, brow, bcol, bval, _ = st.gradient_hessian(sl.params, sl.x_eval)
    bval = np.asarray(bval).reshape(-1, 3, 3)
    r = (3 * np.asarray(brow)[:, None, None] + np.arange(3)[None, :, None]).repeat(3, 2).ravel()
    c = (3 * np.asarray(bcol)[:, None, None] + np.arange(3)[None, None, :]).repeat(3, 1).ravel()
    H = H + sp.csr_matrix((bval.ravel(), (r, c)), shape=(n, n))
    # Dirichlet: indenter bottom face clamped, pad u_x = u_y = 0 (system.build_slab_system)
    r3 = sl.rest.reshape(-1, 3)
    mask = np.ones((n // 3, 3))
    nb0 = sl.offsets[1]
    mask[:nb0][r3[:nb0, 2] < 1e-9] = 0
    mask[nb0:, 0:2] = 0
    m = mask.ravel()
    Pm = sp.diags(m)
    A = (Pm @ H @ Pm + sp.diags(1 - m)).tocsr()
    return sl, A, m


def build_hertz(refine=0.7):
    """C1 (one C5 scene): block + ball, the ball lowered so its pole gap is
    eps_max / 2 (scenes.c5_batch), Dirichlet dofs from the scene."""
    sc = S.hertz_scene(S.HertzConfig(refine=refine))
    n = sc.rest.size
    H = elastic_K(sc.block, 0, n, sc.cfg.E, sc.cfg.nu) + elastic_K(sc.ball, sc.ball_offset, n, sc.cfg.E, sc.cfg.nu)
    x = sc.rest.reshape(-1, 3).copy()
    x[sc.ball_offset:, 2] -= sc.cfg.initial_gap - 0.5 * sc.cfg.eps_max
    x = x.ravel()
    orc = Oracle("restated")
    pairs = orc.candidate_pairs(sc.slave, sc.master, sc.rest, sc.params.detection_radius)
    st = orc.contact_state(sc.slave, sc.master, pairs, sc.rest, sc.params)
    _, _, brow, bcol, bval, _ = st.gradient_hessian(sc.params, x)
    bval = np.asarray(bval).reshape(-1, 3, 3)
    r = (3 * np.asarray(brow)[:, None, None] + np.arange(3)[None, :, None]).repeat(3, 2).ravel()
    c = (3 * np.asarray(bcol)[:, None, None] + np.arange(3)[None, None, :]).repeat(3, 1).ravel()
    H = H + sp.csr_matrix((bval.ravel(), (r, c)), shape=(n, n))
    m = np.ones(n)
    m[3 * sc.fixed[:, 0] + sc.fixed[:, 1]] = 0
    Pm = sp.diags(m)
    A = (Pm @ H @ Pm + sp.diags(1 - m)).tocsr()
    bodies = [(sc.block, 0), (sc.ball, sc.ball_offset)]
    return bodies, sc.rest, A, m


def grid_coarse_space(bodies, rest, m, g):
    """Rigid-body modes per aggregate = one cell of a g x g x g grid over each
    body's bounding box (graded meshes), masked."""
    r3 = rest.reshape(-1, 3)
    cols, rows, vals = [], [], []
    k = 0
    for mesh, off in bodies:
        vs_all = off + np.arange(mesh.vertices.shape[0])
        p = r3[vs_all]
        lo, hi = p.min(0), p.max(0)
        cell = np.minimum(((p - lo) / np.maximum(hi - lo, 1e-30) * g).astype(int), g - 1)
        key = (cell[:, 0] * g + cell[:, 1]) * g + cell[:, 2]
        for u in np.unique(key):
            vs = vs_all[key == u]
            d = r3[vs] - r3[vs].mean(axis=0)
            modes = [np.tile(np.eye(3)[a], (vs.size, 1)) for a in range(3)]
            modes += [np.cross(np.eye(3)[a], d) for a in range(3)]
            for md in modes:
                dof = (3 * vs[:, None] + np.arange(3)).ravel()
                val = md.ravel() * m[dof]
                if np.abs(val).max() > 0:
                    rows.append(dof)
                    cols.append(np.full(dof.size, k))
                    vals.append(val)
                    k += 1
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(m.size, k))


def block_jacobi(A):
    n = A.shape[0] // 3
    D = np.zeros((n, 3, 3))
    Ac = A.tocoo()
    sel = (Ac.row // 3) == (Ac.col // 3)
    np.add.at(D, (Ac.row[sel] // 3, Ac.row[sel] % 3, Ac.col[sel] % 3), Ac.data[sel])
    Di = np.linalg.inv(D)
    return lambda r: np.einsum("vab,vb->va", Di, r.reshape(-1, 3)).ravel()


def coarse_space(sl, m, agg):
    """Rigid-body modes (3 translations + 3 rotations) per aggregate = agg x agg
    lattice cells in x/y of one body (both vertex layers), masked."""
    r3 = sl.rest.reshape(-1, 3)
    cols, rows, vals = [], [], []
    k = 0
    for b, mesh in enumerate(sl.meshes):
        off = sl.offsets[b]
        v = mesh.vertices
        h = np.min(np.diff(np.unique(np.round(v[:, 0], 12))))
        ix = np.floor(v[:, 0] / (agg * h) + 1e-9).astype(int)
        iy = np.floor(v[:, 1] / (agg * h) + 1e-9).astype(int)
        key = ix * 100000 + iy
        for u in np.unique(key):
            vs = off + np.nonzero(key == u)[0]
            cen = r3[vs].mean(axis=0)
            d = r3[vs] - cen
            modes = []
            for a in range(3):
                t = np.zeros((vs.size, 3))
                t[:, a] = 1
                modes.append(t)
            for a in range(3):  # rotation about axis a: e_a x d
                e = np.zeros(3)
                e[a] = 1
                modes.append(np.cross(e, d))
            for md in modes:
                dof = (3 * vs[:, None] + np.arange(3)).ravel()
                val = md.ravel() * m[dof]
                if np.abs(val).max() > 0:
                    rows.append(dof)
                    cols.append(np.full(dof.size, k))
                    vals.append(val)
                    k += 1
    P = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(m.size, k))
    return P


def pcg(A, b, prec, tol=1e-8, maxit=20000):
    x = np.zeros_like(b)
    r = b.copy()
    z = prec(r)
    p = z.copy()
    rz = r @ z
    bb = b @ b
    for it in range(1, maxit + 1):
        q = A @ p
        a = rz / (p @ q)
        x += a * p
        r -= a * q
        if r @ r <= tol * tol * bb:
            return it, x
        z = prec(r)
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
    return maxit, x


def main_hertz(gs):
    bodies, rest, A, m = build_hertz()
    print(f"Hertz C1 (refine 0.7): {A.shape[0]} dofs, {A.nnz} nonzeros")
    b = m * np.random.default_rng(1).standard_normal(A.shape[0])
    Dj = block_jacobi(A)
    print(f"block-Jacobi: {pcg(A, b, Dj)[0]} iterations")
    for g in gs:
        P = grid_coarse_space(bodies, rest, m, g)
        lam, Q = np.linalg.eigh((P.T @ A @ P).toarray())
        keep = lam > 1e-12 * lam.max()
        Ci = (Q[:, keep] / lam[keep]) @ Q[:, keep].T
        it2 = pcg(A, b, lambda r, P=P, Ci=Ci: Dj(r) + P @ (Ci @ (P.T @ r)))[0]
        print(f"two-level additive, {g}^3 grid cells per body ({P.shape[1]} coarse dofs): {it2} iterations")


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "hertz":
        return main_hertz([int(a) for a in sys.argv[2:]] or [4, 6])
    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    nt = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    aggs = [int(a) for a in sys.argv[3:]] or [5, 10]
    t0 = time.time()
    sl, A, m = build(nb, nt)
    print(f"slab({nb},{nt}): {A.shape[0]} dofs, {A.nnz} nonzeros, built in {time.time() - t0:.1f} s")
    rng = np.random.default_rng(1)
    b = m * rng.standard_normal(A.shape[0])
    Dj = block_jacobi(A)
    it, _ = pcg(A, b, Dj)
    print(f"block-Jacobi: {it} iterations")
    for agg in aggs:
        P = coarse_space(sl, m, agg)
        Ac = (P.T @ A @ P).toarray()
        lam, Q = np.linalg.eigh(Ac)  # masked modes can be dependent: pseudo-inverse
        keep = lam > 1e-12 * lam.max()
        Ci = (Q[:, keep] / lam[keep]) @ Q[:, keep].T

        def two_level(r, P=P, Ci=Ci):
            return Dj(r) + P @ (Ci @ (P.T @ r))

        it2, _ = pcg(A, b, two_level)
        print(f"two-level additive, {agg}x{agg}-cell aggregates ({P.shape[1]} coarse dofs, factor "
              f"{8 * P.shape[1] ** 2 / 2e6:.2f} MB): {it2} iterations")


if __name__ == "__main__":
    main()


def pair_jacobi(A):
    """6x6 block-Jacobi over vertex pairs from a greedy matching of the strongest
    normalized couplings (generic; on the thin slabs it pairs stacked vertices)."""
    n = A.shape[0] // 3
    B = A.tocoo()
    v, w = B.row // 3, B.col // 3
    sel = v != w
    s = np.zeros(0)
    keys = v[sel] * n + w[sel]
    uk, inv = np.unique(keys, return_inverse=True)
    s = np.bincount(inv, weights=B.data[sel] ** 2)
    dsel = ~sel
    dn = np.bincount(v[dsel], weights=B.data[dsel] ** 2, minlength=n)
    pv, pw = uk // n, uk % n
    score = s / np.sqrt(dn[pv] * dn[pw])
    mate = -np.ones(n, int)
    for k in np.argsort(-score):
        a, b = pv[k], pw[k]
        if mate[a] < 0 and mate[b] < 0 and a != b:
            mate[a], mate[b] = b, a
    groups = [(a, mate[a]) for a in range(n) if mate[a] > a] + [(a,) for a in range(n) if mate[a] < 0]
    Ad = A.tocsr()
    blocks = []
    for gidx in groups:
        dof = np.concatenate([3 * g + np.arange(3) for g in gidx])
        blocks.append((dof, np.linalg.inv(Ad[dof][:, dof].toarray())))

    def apply(r):
        z = np.zeros_like(r)
        for dof, Mi in blocks:
            z[dof] = Mi @ r[dof]
        return z
    return apply


if __name__ == "__main__" and os.environ.get("PAIR_STUDY"):
    nb, nt = int(os.environ.get("NB", 20)), int(os.environ.get("NT", 16))
    sl, A, m = build(nb, nt)
    b = m * np.random.default_rng(1).standard_normal(A.shape[0])
    print(f"slab({nb},{nt}) block-Jacobi {pcg(A, b, block_jacobi(A))[0]}, vertex-pair 6x6 Jacobi "
          f"{pcg(A, b, pair_jacobi(A))[0]} iterations")
