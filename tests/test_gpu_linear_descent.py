"""Standalone Newton linear solve (gmcp_system_linear_solve /
system.solve_descent): the drop-in for the reference's System::solve_descent
(solver.hpp:325-375) under its own CPU System, on a caller-assembled BCSR.

* A captured Hertz C1 Newton system (operand BCSR, Dirichlet mask, gradient;
  tests/test_gpu_linear_solve.py's capture) solved through the standalone
  entry reaches the reference's acceptance test (||H dx - rhs||_inf <= 1e-6
  ||rhs||_inf, solver.hpp:349-356), matches LAPACK's dense solution of the same
  system to the accuracy its condition allows, and matches the System's own
  device solve of it.
* The same matrix without its Dirichlet dofs (global rigid modes) and a net
  force fails the plain solve and is accepted after the reference's
  regularization (1e-8 x the mean free diagonal entry, solver.hpp:352-361), as
  the reference's LDL^T path does.
* Malformed input returns the reference's error types."""
import numpy as np
import pytest

from paper_2605_24339_b200 import gmcp as G
from paper_2605_24339_b200 import scenes as S
from paper_2605_24339_b200 import system as SY

pytestmark = pytest.mark.gpu


def _hertz_capture():
    sys_, _ = SY.build_hertz_system(S.HertzConfig(refine=0.7))
    sys_.capture_linear_system(True)
    sys_.time_newton(SY.SolverSettings(pcg_tol=1e-10), n_iters=2)  # the second system: no shift
    cap = sys_.captured_linear_system()
    return sys_, cap


def test_captured_newton_system_solves_like_lapack_and_the_system():
    sys_, cap = _hertz_capture()
    assert cap["shift"] == 0
    m = cap["mask"]
    rhs = -m * cap["grad"]
    fixed = (m == 0).astype(np.uint8)
    for positions in (None, sys_.rest):  # smoother only / two-level
        r = SY.solve_descent(cap["rowptr"], cap["cols"], cap["vals"], rhs, fixed=fixed, positions=positions,
                             pcg_tol=1e-10)
        assert not r.regularized
        assert r.residual_inf_rel <= 1e-6
        nv = cap["rowptr"].size - 1
        rows = np.repeat(np.arange(nv), np.diff(cap["rowptr"]))
        H = np.zeros((3 * nv, 3 * nv))
        for a in range(3):
            for c in range(3):
                H[3 * rows + a, 3 * cap["cols"] + c] += cap["vals"][:, a, c]
        A = (m[:, None] * H) * m[None, :] + np.diag(1.0 - m)
        res = m * (H @ r.dx) - rhs
        assert np.abs(res).max() <= 1e-6 * np.abs(rhs).max()
        assert np.all(r.dx[m == 0] == 0)
        xd = np.linalg.solve(A, rhs)
        err = np.sqrt((r.dx - xd) @ (A @ (r.dx - xd)) / (xd @ (A @ xd)))  # energy norm
        assert err <= 1e-6, err
        assert np.linalg.norm(r.dx - cap["dx"]) <= 1e-6 * np.linalg.norm(cap["dx"])
        assert r.iterations > 0


def test_floating_system_is_accepted_after_regularization():
    # the captured Newton matrix without its Dirichlet dofs: elastic and contact
    # terms are translation invariant, so H has the global rigid modes, and a net
    # force along x is inconsistent -> the plain PCG is not accepted, the
    # regularized retry is (the reference's LDL^T path: solver.hpp:352-361)
    _, cap = _hertz_capture()
    nv = cap["rowptr"].size - 1
    rhs = np.zeros(3 * nv)
    rhs[0::3] = 1.0
    r = SY.solve_descent(cap["rowptr"], cap["cols"], cap["vals"], rhs, pcg_tol=1e-10)
    assert r.regularized and r.residual_inf_rel <= 1e-6
    assert np.all(np.isfinite(r.dx))
    with pytest.raises(G.SolverError):  # no iterations to reach the tolerance: SolverError
        SY.solve_descent(cap["rowptr"], cap["cols"], cap["vals"], rhs, pcg_tol=1e-10, max_iters=1)


def test_bad_input_raises_reference_errors():
    rp = np.array([0, 1, 2], np.int32)
    cl = np.array([1, 0], np.int32)
    vals = np.tile(np.eye(3), (2, 1, 1))
    with pytest.raises(G.ConfigError):
        SY.solve_descent(rp, cl, vals, np.zeros(5))  # rhs size
    bad = np.array([0, 2, 2], np.int32)
    with pytest.raises(G.Error):
        SY.solve_descent(bad, np.array([1, 0], np.int32), vals, np.ones(6))  # columns not ascending
    with pytest.raises(G.Error):
        SY.solve_descent(rp, cl, vals, np.ones(6), fixed=np.ones(6, np.uint8))  # no free dofs
