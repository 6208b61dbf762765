"""A/B of the single-system PCG preconditioners on the device Newton solve
(same box, same scene): env GMCP_PAIR_JACOBI / GMCP_COARSE / GMCP_COARSE_AGGS
are read per System, so each configuration runs in its own subprocess.

  python tools/precond_ab.py c3|c2|hertz [n_iters]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = [("bj", {"GMCP_PAIR_JACOBI": "0", "GMCP_COARSE": "0"}),
           ("pair", {"GMCP_PAIR_JACOBI": "1", "GMCP_COARSE": "0"})] + \
          [(f"pair+coarse{a}", {"GMCP_PAIR_JACOBI": "1", "GMCP_COARSE": "1", "GMCP_COARSE_AGGS": str(a)})
           for a in (32, 64, 128, 256)] + \
          [("bj+coarse128", {"GMCP_PAIR_JACOBI": "0", "GMCP_COARSE": "1", "GMCP_COARSE_AGGS": "128"})]

CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
from paper_2605_24339_b200 import scenes as S, system as SY
case, n = sys.argv[1], int(sys.argv[2])
if case == "hertz":
    s, _ = SY.build_hertz_system(S.HertzConfig(refine=0.7))
elif case == "c2":
    s = SY.build_slab_system(50, 40, texture_amp=2e-4)
else:
    s = SY.build_slab_system(155, 124, texture_amp=2e-4)
ms, pcg = s.time_newton(SY.SolverSettings(pcg_tol=1e-10), n_iters=n)
ps = s.pcg_stats()
ls = s.linear_stats()
print(json.dumps({"ms": [round(float(v), 3) for v in ms], "pcg": [int(v) for v in pcg],
                  "us_per_pcg_iter": 1e3 * ps["ms"] / max(ps["iters"], 1), "max_rel2": ls["max_rel2"]}))
''' % ROOT

case = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = sys.argv[2] if len(sys.argv) > 2 else "6"
for name, env in CONFIGS:
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", CHILD, case, n], env=e, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip()[-400:]
    print(f"{case} {name}: {line}", flush=True)
