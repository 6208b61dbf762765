"""Scene files solved on the device (parse_scene + build_scene + System::solve
on B200) against the reference's own solve of the same file
(tests/golden/<scene>_ref.npz, made by tests/golden/make_scene_golden.py):
the patch test and C4, the two-pad fingertip squeeze (2 contact pairs, 20
load steps)."""
import os

import numpy as np
import pytest

import fixtures as F  # noqa: F401  (sys.path set-up)
from paper_2605_24339_b200 import scene as SC

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("name,tol", [("patch_test", 1e-4), ("fingertip", 1e-9)])
def test_scene_matches_reference_solve(name, tol):
    g = np.load(os.path.join(ROOT, "tests", "golden", name + "_ref.npz"))
    sys_, st = SC.run_scene(os.path.join(ROOT, "scenes", name + ".scene"))
    x_ref = g["x"]
    u_ref = x_ref - sys_.rest
    # same equilibrium up to the Newton tolerance's slack (residual <= tol_N;
    # patch test: 6.25e-7 N against a soft interface -> ~1e-4 of u; measured
    # 8.7e-5. Fingertip: measured 1e-13)
    assert np.max(np.abs(sys_.x - x_ref)) <= tol * np.max(np.abs(u_ref))
    assert len(st.steps) == int(g["stats"][2])
    assert abs(st.total_newton_iters - int(g["stats"][0])) <= 3
    assert st.newton_tol_used == g["stats"][4]
    assert all(s.min_gap > 0 for s in st.steps)
    for p in range(len(sys_.contacts)):
        tot = sys_.contact_force_summary(p)[3]
        assert np.allclose(tot, g["force"][3 * p:3 * p + 3], rtol=tol, atol=tol * np.max(np.abs(g["force"])))


@pytest.mark.gpu
def test_scene_outputs_deterministic(tmp_path):
    """bench.hpp:374-402 run_scene with per-step files, twice in sequential
    mode: every file byte-identical (the reference's determinism criterion);
    pressure tables list each pair's face samples with positive pressures."""
    from paper_2605_24339_b200 import outputs as O
    import shutil
    d = tmp_path / "out"
    snaps = []
    for k in range(2):  # same output directory both times (it is echoed in the report)
        if d.exists():
            shutil.rmtree(d)
        cfg = SC.parse_scene(os.path.join(ROOT, "scenes", "patch_test.scene"))
        rep = O.run_scene(cfg, out_override=str(d), sequential=True)
        snaps.append({p.name: p.read_bytes() for p in d.iterdir()})
    names = sorted(snaps[0])
    assert names == sorted(snaps[1])
    assert "report.txt" in names and "step_10_pressure.csv" in names and "step_01_volume.vtk" in names
    for n in names:
        assert snaps[0][n] == snaps[1][n], n
    assert rep.find("total_newton_iters") is not None and rep.find("wall_seconds") is None
    rows = np.loadtxt(d / "step_10_pressure.csv", delimiter=",", skiprows=1)
    assert rows.shape[1] == 7 and np.all(rows[:, 0] == 0) and np.max(rows[:, 6]) > 0
