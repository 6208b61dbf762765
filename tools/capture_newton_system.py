"""Capture a steady Newton iteration's linear system from the device solver
(gmcp_system_capture_linear_system) for the offline preconditioner study
(tools/precond_study.py). Writes gpurun_out/newton_<case>.npz.

  python tools/capture_newton_system.py c2|hertz|c3 [iteration]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_24339_b200 import scenes as S  # noqa: E402
from paper_2605_24339_b200 import system as SY  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c2"
it = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if case == "hertz":
    sys_, _ = SY.build_hertz_system(S.HertzConfig(refine=0.7))
elif case == "c3":
    sys_ = SY.build_slab_system(155, 124, texture_amp=2e-4)
else:
    sys_ = SY.build_slab_system(50, 40, texture_amp=2e-4)
sys_.capture_linear_system(True)
ms, pcg = sys_.time_newton(SY.SolverSettings(pcg_tol=1e-10), n_iters=it)
cap = sys_.captured_linear_system()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
out = os.path.join(ROOT, "gpurun_out", f"newton_{case}.npz")
np.savez_compressed(out, rest=sys_.rest, pcg=pcg, ms=ms, **cap)
print(case, "pcg per iteration", pcg.tolist(), "ms", np.round(ms, 2).tolist(), "->", out)
