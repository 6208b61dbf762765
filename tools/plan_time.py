"""Host assembly-plan build time (per rebuild) on C3: first gradient call minus a steady call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_24339_b200 import gmcp as gm, scenes

sc = scenes.slab_scene(155, 124, texture_amp=2e-4)
ctx = gm.Context(0)
ctx.set_params(sc.params); ctx.set_surfaces(sc.slave, sc.master); ctx.set_positions(sc.rest)
t = time.perf_counter(); ctx.broadphase(sc.params.detection_radius); n = ctx.build_samples(); t1 = time.perf_counter()
ctx.set_positions(sc.x_eval)
g = np.zeros(sc.rest.size)
t2 = time.perf_counter(); ctx.gradient(g, hessian=True); t3 = time.perf_counter()
ctx.gradient(g, hessian=True); t4 = time.perf_counter()
ctx.set_positions(sc.rest)
t5 = time.perf_counter(); ctx.broadphase(sc.params.detection_radius); t6 = time.perf_counter(); ctx.build_samples(); t7 = time.perf_counter()
ctx.set_positions(sc.x_eval)
t8 = time.perf_counter(); ctx.gradient(g, hessian=True); t9 = time.perf_counter()
print(f"second rebuild: broadphase {1e3*(t6-t5):.1f} ms sampler {1e3*(t7-t6):.1f} ms plan+grad {1e3*(t9-t8):.1f} ms")
print(f"rebuild (broadphase+sampler) {1e3*(t1-t):.1f} ms; first gradient (plan) {1e3*(t3-t2):.1f} ms; steady {1e3*(t4-t3):.2f} ms")
