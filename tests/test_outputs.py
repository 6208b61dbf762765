"""Run-output formats (vtk_io.hpp) byte-for-byte against the reference's own
writers on the same arrays, including awkward doubles (format_real "%.17g").
CPU only."""
import ctypes as C

import numpy as np

from paper_2605_24339_b200 import outputs as O


def test_writers_byte_identical_to_reference(ref, tmp_path):
    rng = np.random.default_rng(3)
    np_, nt, ntri, nr = 17, 9, 11, 13
    pts = rng.normal(size=(np_, 3)) * np.array([1e-3, 1.0, 1e7])
    pts[0] = [0.0, -0.0, 1.0 / 3.0]
    pts[1] = [1e-320, 5e-324, 123456789.123456789]
    tets = rng.integers(0, np_, size=(nt, 4)).astype(np.int32)
    tris = rng.integers(0, np_, size=(ntri, 3)).astype(np.int32)
    disp = rng.normal(size=(np_, 3))
    stress = rng.normal(size=(nt, 9)) * 1e9
    rows = rng.normal(size=(nr, 7))
    rows[:, 0] = rng.integers(0, 3, nr)
    rows[:, 1] = np.arange(nr)
    rows[2, 6] = -0.0
    a, b = tmp_path / "ref", tmp_path / "ours"
    a.mkdir()
    b.mkdir()
    p = lambda v: C.c_void_p(np.ascontiguousarray(v).ctypes.data)  # noqa: E731
    keep = [np.ascontiguousarray(v) for v in (pts, tets, tris, disp, stress, rows)]
    assert ref.lib.ref_write_formats(C.c_char_p(str(a).encode()), p(keep[0]), C.c_int64(np_), p(keep[1]),
                                     C.c_int64(nt), p(keep[2]), C.c_int64(ntri), p(keep[3]), p(keep[4]), p(keep[5]),
                                     C.c_int64(nr)) == 0
    O.save_vtk_tets(str(b / "vol.vtk"), pts, tets, [("displacement", 3, disp)], [("cauchy_stress", 9, stress)])
    O.save_vtk_tris(str(b / "surf.vtk"), pts, tris)
    O.save_csv(str(b / "p.csv"), ["pair", "sample", "x", "y", "z", "gap", "pressure"], rows.tolist())
    rep = O.Report()
    rep.set("scene.path", "a b.scene")
    rep.set("scene.bodies", 3)
    rep.set("x", 0.1)
    rep.set("y", -2.5e-300)
    rep.set("x", 1.0 / 3.0)
    rep.set("threads", 1)
    rep.save(str(b / "report.txt"))
    for f in ("vol.vtk", "surf.vtk", "p.csv", "report.txt"):
        assert (a / f).read_bytes() == (b / f).read_bytes(), f
