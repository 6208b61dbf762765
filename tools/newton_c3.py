"""C3 Newton iterations on the device (for profiling the PCG kernels):
  python tools/newton_c3.py [n_iters] [pcg_tol]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24339_b200 import system as SY  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-10
s = SY.build_slab_system(155, 124, texture_amp=2e-4)
ms, pcg = s.time_newton(SY.SolverSettings(pcg_tol=tol, pcg_max_iters=50000), n)
ps = s.pcg_stats()
print("ms/iter", [round(float(v), 2) for v in ms], "pcg", list(pcg),
      "us/pcg-iter %.2f" % (1e3 * ps["ms"] / max(ps["iters"], 1)), flush=True)
