"""C1: Hertz sphere-on-block indentation solved on the device (System on
B200) -- the reference's acceptance criterion (acceptance.cpp:280-301) and
agreement with the reference's own run_hertz (tests/golden/hertz_ref.json)."""
import numpy as np
import pytest

import fixtures as F
from paper_2605_24339_b200 import scenes as S
from paper_2605_24339_b200 import system as SY


@pytest.mark.gpu
@pytest.mark.parametrize("refine", [0.7, 1.0])
def test_hertz_acceptance_and_reference_agreement(refine):
    res = SY.run_hertz(S.HertzConfig(refine=refine))
    g = F.golden("hertz_ref.json")[str(refine)]
    # acceptance.cpp:296-300
    assert len(res.stats.steps) == 10
    assert res.peak_rel_err <= 0.20
    assert res.contact_radius_rel_err <= 0.20
    assert res.outside_max <= 0.02 * res.peak
    # same problem, same discretisation as the reference run
    assert res.params.kappa_face == g["kappa_face"]
    assert res.applied_force == pytest.approx(g["applied_force"], rel=1e-12)
    # the device solve (PCG) converges to the reference's (LDL^T) equilibrium:
    # measured agreement is ~3e-13 on the peak at refine 0.7
    assert res.peak == pytest.approx(g["peak"], rel=1e-7)
    assert res.contact_radius == pytest.approx(g["contact_radius"], rel=1e-7)
    assert abs(res.stats.total_newton_iters - g["total_newton_iters"]) <= 3
    assert res.face_samples == g["face_samples"]
    assert all(s.min_gap > 0 for s in res.stats.steps)
