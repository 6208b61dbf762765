"""Breakdown of the e2e step (public API with pinned host buffers) on C3."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_24339_b200 import gmcp as gm, scenes

sc = scenes.slab_scene(155, 124, texture_amp=2e-4)
ctx = gm.Context(0)
ctx.set_params(sc.params); ctx.set_surfaces(sc.slave, sc.master); ctx.set_positions(sc.rest)
ctx.broadphase(sc.params.detection_radius); n = ctx.build_samples()
xh = torch.empty(sc.rest.size, dtype=torch.float64, pin_memory=True).numpy(); xh[:] = sc.x_eval
gh = torch.empty(sc.rest.size, dtype=torch.float64, pin_memory=True).numpy()
for _ in range(5):
    ctx.set_positions(xh); ctx.gradient(gh, hessian=True)
K = 50
def t(f):
    t0 = time.perf_counter()
    for _ in range(K): f()
    return (time.perf_counter() - t0) / K * 1e6
print("zero gh        %.1f us" % t(lambda: gh.__setitem__(slice(None), 0)))
print("set_positions  %.1f us" % t(lambda: ctx.set_positions(xh)))
print("gradient(None) %.1f us" % t(lambda: ctx.gradient(None, hessian=True)))
print("gradient(gh)   %.1f us" % t(lambda: ctx.gradient(gh, hessian=True)))
def step():
    gh[:] = 0; ctx.set_positions(xh); ctx.gradient(gh, hessian=True)
print("full step      %.1f us  (n=%d -> %.3g samples/s)" % (t(step), n, n / (t(step) * 1e-6)))
