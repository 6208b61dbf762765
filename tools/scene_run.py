"""Runs a scene file on the device System (parse_scene + build_scene + solve)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_24339_b200 import scene as SC

for path in sys.argv[1:]:
    t = time.time()
    sys_, st = SC.run_scene(path)
    f = [sys_.contact_force_summary(p)[3] if False else sys_.contact_force_summary(p) for p in range(len(sys_.contacts))]
    print(f"{path}: {time.time()-t:.2f}s (solve {st.wall_seconds:.2f}s) steps {len(st.steps)} newton {st.total_newton_iters} "
          f"rebuilds {st.total_rebuilds} pcg {st.total_pcg_iters} min_gap {st.steps[-1].min_gap!r} dofs {sys_.rest.size}", flush=True)
    for p, fs in enumerate(f):
        print("  pair", p, "force summary", np.round(fs, 6).tolist())
    np.save(os.path.join("gpurun_out", os.path.basename(path) + ".x.npy"), sys_.x)
