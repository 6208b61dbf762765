"""Times the C3 rebuild (broadphase + sampler through the public API): the
first (cold: buffers allocated) and the following (warm) rebuilds, wall clock
around each call pair (the calls synchronize). Dev tool."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24339_b200 import gmcp as gm, scenes

sc = scenes.slab_scene(155, 124, texture_amp=2e-4)
ctx = gm.Context(0)
ctx.set_params(sc.params)
ctx.set_surfaces(sc.slave, sc.master)
ctx.set_positions(sc.rest)
ts = []
for _ in range(6):
    t0 = time.perf_counter()
    ctx.broadphase(sc.params.detection_radius)
    n = ctx.build_samples()
    ts.append((time.perf_counter() - t0) * 1e3)
print("samples", n, "rebuild ms cold %.2f warm" % ts[0], " ".join("%.2f" % t for t in ts[1:]), flush=True)
