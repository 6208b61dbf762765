"""Runs the Hertz indentation (C1) on the device and prints the metrics."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24339_b200 import scenes as S, system as SY

for refine in [float(a) for a in sys.argv[1:]] or [0.7]:
    t = time.time()
    r = SY.run_hertz(S.HertzConfig(refine=refine))
    st = r.stats
    print(f"refine {refine}: {time.time()-t:.2f}s wall (solve {st.wall_seconds:.2f}s) steps {len(st.steps)} newton {st.total_newton_iters} "
          f"rebuilds {st.total_rebuilds} pcg {st.total_pcg_iters} peak {r.peak!r} (p0 {r.oracle.p0!r}, err {r.peak_rel_err:.4f}) "
          f"radius {r.contact_radius!r} (aH {r.oracle.alpha_H!r}, err {r.contact_radius_rel_err:.4f}) outside {r.outside_max!r} "
          f"face samples {r.face_samples} min gaps {[round(s.min_gap, 9) for s in st.steps]}", flush=True)
