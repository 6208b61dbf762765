"""Generates tests/golden/hertz_ref.json: the reference's own run_hertz
(bench.hpp:210-303, compiled from /root/reference with the oracle's Eigen
shim -- its SimplicialLDLT stand-in is a natural-order LDL^T) at refine 0.7
(C1) and 1.0 (the acceptance default). Run here, where /root/reference
exists:  python tests/golden/make_hertz_golden.py
The GPU test compares run_hertz on the device against these numbers."""
import ctypes as C
import json
import os
import subprocess
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
LIB = os.path.join(ROOT, "oracle", "_ref", "libgmcp_ref.so")
KEYS = ("peak", "p0", "contact_radius", "alpha_H", "outside_max", "peak_rel_err", "contact_radius_rel_err",
        "applied_force", "total_newton_iters", "steps", "kappa_face", "wall_seconds", "face_samples",
        "total_rebuilds")


def main():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "ref"])
    L = C.CDLL(LIB)
    out = {}
    for refine in (0.7, 1.0):
        v = np.zeros(len(KEYS))
        t = time.time()
        rc = L.ref_run_hertz(C.c_double(refine), C.c_int32(10), C.c_void_p(v.ctypes.data))
        assert rc == 0, rc
        out[str(refine)] = dict(zip(KEYS, v.tolist()))
        print(refine, f"{time.time() - t:.1f}s", out[str(refine)], flush=True)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "hertz_ref.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
