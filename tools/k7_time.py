"""Times the C3 assembly pass for the library named by GMCP_B200_LIB (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_24339_b200 import gmcp as gm, scenes

sc = scenes.slab_scene(155, 124, texture_amp=2e-4)
ctx = gm.Context(0)
ctx.set_params(sc.params)
ctx.set_surfaces(sc.slave, sc.master)
ctx.set_positions(sc.rest)
ctx.broadphase(sc.params.detection_radius)
n = ctx.build_samples()
ctx.set_positions(sc.x_eval)
g = np.zeros(sc.rest.size)
e = ctx.gradient(g, hessian=True)
_, _, vals = ctx.download_hessian()
ctx.time_assembly(5, True)
best = min((ctx.time_assembly(20, True) for _ in range(3)), key=lambda t: t[0])
print(f"{os.environ.get('GMCP_B200_LIB', 'default')}: n={n} pass {best[0]*1e3:.1f} us  k7 {best[1]*1e3:.1f} us  "
      f"E={e!r} |g|={np.linalg.norm(g)!r} |H|={np.linalg.norm(vals)!r}", flush=True)
