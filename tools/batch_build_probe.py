import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_24339_b200 import scenes as S, system as SY
cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
t = time.time(); b = S.c5_batch(1024, first=0, count=cnt); t1 = time.time()
bs = SY.build_hertz_batch_system(b); t2 = time.time()
ms, pcg = bs.time_newton(SY.SolverSettings(load_steps=10), 6); t3 = time.time()
act = bs.timed_active_scenes(len(ms))
print(f"{cnt}: c5_batch {t1-t:.1f}s build {t2-t1:.1f}s time_newton(6) {t3-t2:.1f}s per-iter ms {np.round(ms,1)} pcg {pcg} "
      f"active {act} -> {act[1:].sum() / (ms[1:].sum() / 1e3):.0f} scene-Newton-steps/s (passes 2..)", flush=True)
