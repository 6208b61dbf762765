"""The single-system PCG under every preconditioner the runtime switches
select (GMCP_PAIR_JACOBI / GMCP_COARSE are read when a System is
created): 3x3 block-Jacobi, vertex-pair 6x6 block-Jacobi, and either with the
two-level rigid-mode coarse space. Every mode must reach the same
load-stepped equilibrium (the reference's System::solve result does not
depend on how the Newton system is solved), report the mode it ran, and keep
the reference's acceptance test on every linear solve (solver.hpp:349-356)."""
import os

import numpy as np
import pytest

from paper_2605_24339_b200 import scenes as S
from paper_2605_24339_b200 import system as SY

pytestmark = pytest.mark.gpu

MODES = [(0, 0), (1, 0), (0, 1), (1, 1)]


def _solve(build, pair, coarse):
    old = {k: os.environ.get(k) for k in ("GMCP_PAIR_JACOBI", "GMCP_COARSE")}
    os.environ["GMCP_PAIR_JACOBI"], os.environ["GMCP_COARSE"] = str(pair), str(coarse)
    try:
        s = build()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    st = s.solve(SY.SolverSettings(load_steps=4))
    return s, st


@pytest.mark.parametrize("scene", ["patch", "hertz"])
def test_every_preconditioner_reaches_the_same_equilibrium(scene):
    if scene == "patch":
        build = SY.build_patch_scene
    else:
        def build():
            return SY.build_hertz_system(S.HertzConfig(refine=0.7))[0]
    runs = {}
    for pair, coarse in MODES:
        s, st = _solve(build, pair, coarse)
        info = s.precond_info()
        assert info["pair_jacobi"] == bool(pair) and info["coarse"] == bool(coarse)
        lin = s.linear_stats()
        assert lin["solves"] >= st.total_newton_iters and lin["max_relinf"] <= 1e-6
        runs[(pair, coarse)] = (s.x.copy(), s.rest, st)
    x0, rest, st0 = runs[(1, 1)]
    umax = np.abs(x0 - rest).max()
    for mode, (x, _, st) in runs.items():
        assert np.abs(x - x0).max() <= 1e-8 * umax, mode
        assert abs(st.total_newton_iters - st0.total_newton_iters) <= 4, mode
    # the two-level preconditioner needs fewer PCG iterations than its smoother alone
    assert runs[(1, 1)][2].total_pcg_iters < runs[(1, 0)][2].total_pcg_iters
    assert runs[(0, 1)][2].total_pcg_iters < runs[(0, 0)][2].total_pcg_iters
