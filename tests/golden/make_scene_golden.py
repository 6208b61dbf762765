"""Generates tests/golden/<scene>_ref.npz: the reference's own parse_scene +
build_scene + System::solve (scene.hpp, solver.hpp; compiled from
/root/reference with the oracle's Eigen shim, whose SimplicialLDLT stand-in
is a natural-order LDL^T) on the repo's scene files. Run here, where
/root/reference exists:  python tests/golden/make_scene_golden.py
Stores the final positions, run statistics and per-pair contact force totals."""
import ctypes as C
import os
import subprocess
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
LIB = os.path.join(ROOT, "oracle", "_ref", "libgmcp_ref.so")
SCENES = ("patch_test", "fingertip")


def main():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "ref"])
    L = C.CDLL(LIB)
    for name in SCENES:
        path = os.path.join(ROOT, "scenes", name + ".scene").encode()
        n = C.c_int64()
        assert L.ref_run_scene(C.c_char_p(path), C.byref(n), None, None, None, C.c_int32(0)) == 0
        x, st, fo = np.zeros(n.value), np.zeros(6), np.zeros(3 * 8)
        t = time.time()
        rc = L.ref_run_scene(C.c_char_p(path), C.byref(n), C.c_void_p(x.ctypes.data), C.c_void_p(st.ctypes.data),
                             C.c_void_p(fo.ctypes.data), C.c_int32(8))
        assert rc == 0, rc
        print(name, f"{time.time() - t:.1f}s", st, flush=True)
        np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), name + "_ref.npz"),
                            x=x, stats=st, force=fo)


if __name__ == "__main__":
    main()
