"""C3 Newton iterations on the device (for profiling the PCG kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24339_b200 import system as SY
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = SY.build_slab_system(155, 124, texture_amp=2e-4)
ms, pcg = s.time_newton(SY.SolverSettings(pcg_tol=1e-8, pcg_max_iters=50000), n)
print("ms/iter", [round(float(v), 2) for v in ms], "pcg", list(pcg), flush=True)
