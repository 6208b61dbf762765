"""Full C3 load-stepped solve on the device (dev tool): wall time, Newton and
PCG totals, first Newton step PCG count per load step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24339_b200 import system as SY
s = SY.build_slab_system(155, 124, texture_amp=2e-4)
t = time.time()
st = s.solve(SY.SolverSettings(pcg_tol=1e-8, pcg_max_iters=50000))
print(f"C3 solve {time.time()-t:.2f}s newton {st.total_newton_iters} pcg {st.total_pcg_iters} rebuilds {st.total_rebuilds}",
      [(ss.newton_iters, ss.pcg_iters) for ss in st.steps], flush=True)
