"""GPU re-expression of the reference's analytic checks on the contact path
(test_contact.cpp:94-135), run on the CUDA kernels through the C-ABI:

* the gradient matches central finite differences of the energy over 50
  seeded random active states (h = 1e-7, inf-norm error / max(|g|, 1) < 1e-5);
* the Gauss-Newton Hessian is exactly symmetric and positive semi-definite
  (lambda_min >= -1e-10 max|H|), and the gradient written with it equals the
  plain gradient bitwise.

The samples are built by the GPU sampler (gmcp_broadphase + gmcp_build_samples)
at rest, as make_active_pair does (test_contact.cpp:54-66)."""
import numpy as np
import pytest

import fixtures as F

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gm():
    from paper_2605_24339_b200 import gmcp
    return gmcp


def _ctx(gm, scene, x):
    ctx = gm.Context(0)
    ctx.set_params(scene["params"])
    ctx.set_surfaces(scene["slave"], scene["master"])
    ctx.set_positions(scene["rest"])
    ctx.broadphase(scene["params"].detection_radius)
    assert ctx.build_samples() > 0
    ctx.set_positions(x)
    return ctx


def _energy(ctx, x):
    ctx.set_positions(x)
    return ctx.energy()


def _dense_hessian(ctx, n):
    rowptr, cols, vals = ctx.download_hessian()
    H = np.zeros((n, n))
    for r in range(rowptr.size - 1):
        for k in range(rowptr[r], rowptr[r + 1]):
            H[3 * r:3 * r + 3, 3 * cols[k]:3 * cols[k] + 3] += vals[k].reshape(3, 3)
    return H


def test_gradient_matches_finite_differences(gm):
    tp = F.tet_pair()
    ctx = _ctx(gm, tp, tp["x"])
    assert ctx.try_energy()[1] < tp["params"].eps_max  # some sample is active
    rng = np.random.default_rng(101)
    h = 1e-7
    for cfg in range(50):
        x = tp["x"] + rng.uniform(-1e-4, 1e-4, size=tp["x"].size)
        ctx.set_positions(x)
        g = np.zeros_like(x)
        ctx.gradient(g)
        fd = np.zeros_like(x)
        xp = x.copy()
        for i in range(x.size):
            xp[i] = x[i] + h
            ep = _energy(ctx, xp)
            xp[i] = x[i] - h
            em = _energy(ctx, xp)
            xp[i] = x[i]
            fd[i] = (ep - em) / (2 * h)
        scale = max(np.abs(g).max(), 1.0)
        assert np.abs(fd - g).max() / scale < 1e-5, cfg
        assert np.abs(g).max() > 1.0  # contact really is active


@pytest.mark.parametrize("which", ["tetpair", "patch"])
def test_gauss_newton_hessian_symmetric_psd(gm, which):
    if which == "tetpair":
        sc = F.tet_pair()
        x = sc["x"]
    else:
        sc = F.patch_interface()
        xv = sc["rest"].reshape(-1, 3).copy()
        xv[sc["off"]:, 2] -= 1.5e-3
        x = F.random_active(7, xv.ravel())
    ctx = _ctx(gm, sc, x)
    g = np.zeros_like(x)
    ctx.gradient(g, hessian=True)
    H = _dense_hessian(ctx, x.size)
    assert np.abs(H).max() > 0
    assert np.array_equal(H, H.T)  # exact symmetry
    lam = np.linalg.eigvalsh(H)
    assert lam.min() >= -1e-10 * np.abs(H).max()
    g2 = np.zeros_like(x)
    ctx.gradient(g2)
    assert np.array_equal(g, g2)  # the combined routine's gradient is the plain one
