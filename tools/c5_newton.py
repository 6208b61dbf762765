"""C5 batched Newton passes on the device (dev tool):
  python tools/c5_newton.py [n_scenes] [passes]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24339_b200 import scenes as S  # noqa: E402
from paper_2605_24339_b200 import system as SY  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 8
b = S.c5_batch(1024, 0, n)
s = SY.build_hertz_batch_system(b)
ms, pcg = s.time_newton(SY.SolverSettings(load_steps=10), passes)
act = s.timed_active_scenes(len(ms))
print("pass ms", [round(float(v), 1) for v in ms], "pcg", [int(v) for v in pcg], "active", [int(v) for v in act])
print("scene-Newton-steps/s (passes 3..) %.0f" % (act[2:].sum() / (ms[2:].sum() / 1e3)), flush=True)
