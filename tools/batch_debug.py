import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24339_b200 import scenes as S, system as SY
bb = S.c5_batch(1024, first=0, count=256)
try:
    bs = SY.build_hertz_batch_system(bb)
    st = bs.solve(SY.SolverSettings(load_steps=10))
    print("batch 256 ok", flush=True)
except Exception as e:
    print("batch 256 FAIL", e, flush=True)
    import re
    k = int(re.search(r"scene (\d+)", str(e)).group(1))
    one = SY.build_hertz_scene_system(bb, k)
    try:
        so = one.solve(SY.SolverSettings(load_steps=10))
        print("single", k, "ok", so.total_newton_iters, [s.newton_iters for s in so.steps], flush=True)
    except Exception as e2:
        print("single", k, "FAIL", e2, flush=True)
