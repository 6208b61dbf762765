import sys, time
sys.path.insert(0, '/root/repo')
from paper_2605_24339_b200 import system as SY
for nb, nt, tex in ((50, 40, 0.0), (155, 124, 2e-4)):
    t = time.time()
    s = SY.build_slab_system(nb, nt, texture_amp=tex)
    t1 = time.time()
    for tol in (1e-8, 1e-6):
        ms, pcg = s.time_newton(SY.SolverSettings(pcg_tol=tol, pcg_max_iters=50000), 4)
        print(f"slab({nb},{nt}) tol {tol}: setup {t1-t:.1f}s  ms/iter {list(ms.round(2))} pcg {list(pcg)}", flush=True)
