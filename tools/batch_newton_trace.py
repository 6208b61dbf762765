"""Batched C5 Newton passes with per-phase trace (GMCP_TRACE=1) for the
library named by GMCP_B200_LIB (dev tool)."""
import os, sys, time
os.environ.setdefault("GMCP_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24339_b200 import scenes as S, system as SY

b = S.c5_batch(int(sys.argv[1]) if len(sys.argv) > 1 else 1024)
bs = SY.build_hertz_batch_system(b)
ms, pcg = bs.time_newton(SY.SolverSettings(load_steps=10), 8)
print("per pass ms", [round(float(v), 1) for v in ms], "pcg", list(pcg), flush=True)
