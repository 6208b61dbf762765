"""Batched C5 Newton solve: agreement with individual solves and timing vs batch size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_24339_b200 import scenes as S, system as SY

b = S.c5_batch(1024, first=3, count=3)
bs = SY.build_hertz_batch_system(b)
st = bs.solve(SY.SolverSettings(load_steps=4))
N = b.base.rest.size // 3
for k in range(3):
    one = SY.build_hertz_scene_system(b, k)
    so = one.solve(SY.SolverSettings(load_steps=4))
    xb = bs.x[3 * k * N:3 * (k + 1) * N]
    print(f"scene {k}: max|dx| rel {np.max(np.abs(xb - one.x)) / np.max(np.abs(one.x - one.rest)):.2e} "
          f"iters batch {bs.scene_newton_iters()[k]} single {so.total_newton_iters}", flush=True)
for cnt in [int(a) for a in sys.argv[1:]] or [16, 64, 256]:
    t = time.time()
    b = S.c5_batch(1024, first=0, count=cnt)
    bs = SY.build_hertz_batch_system(b)
    t1 = time.time()
    st = bs.solve(SY.SolverSettings(load_steps=10))
    it = bs.scene_newton_iters()
    print(f"{cnt} scenes: build {t1-t:.1f}s solve {st.wall_seconds:.2f}s loops {sum(s.newton_iters for s in st.steps)} "
          f"scene-iters {it.sum()} -> {it.sum()/st.wall_seconds:.0f} scene-Newton-steps/s, pcg {st.total_pcg_iters}, "
          f"rebuilds {st.total_rebuilds}", flush=True)
