"""Scene files (scene.hpp, mesh_io.hpp) restated in paper_2605_24339_b200/scene.py:
the reference's own parser cases (test_scene.cpp:40-190) re-expressed, and the
host arrays build_scene hands to System (f_ext, Dirichlet mask/targets, slave
selections) compared BITWISE with the compiled reference. CPU only."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2605_24339_b200 import scene as SC
from paper_2605_24339_b200.gmcp import ConfigError, ParseError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCENE_FILES = [os.path.join(ROOT, "scenes", f) for f in ("patch_test.scene", "fingertip.scene")]


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def _expect(tmp_path, text, line, what):
    p = _write(tmp_path, "bad.scene", text)
    with pytest.raises(ParseError) as e:
        SC.parse_scene(p)
    assert str(e.value) == f"{p}:{line}: {what}"


def test_minimal_scene_defaults(tmp_path):  # test_scene.cpp:40-69
    p = _write(tmp_path, "minimal.scene", "[body]\nname = solo\nyoungs = 250\n")
    cfg = SC.parse_scene(p)
    assert cfg.path == p and len(cfg.bodies) == 1
    b = cfg.bodies[0]
    assert (b.name, b.generator, b.size, b.divisions, b.origin, b.youngs, b.poisson, b.line) == \
        ("solo", "block", (1.0, 1.0, 1.0), (1, 1, 1), (0.0, 0.0, 0.0), 250.0, 0.0, 1)
    assert not cfg.bcs and not cfg.loads and not cfg.contacts and cfg.body_force is None
    assert (cfg.solver.load_steps, cfg.solver.max_newton_iters) == (10, 200)
    assert cfg.output.directory == "out" and cfg.output.volume_meshes and cfg.output.pressure_csv


def test_comments_and_directions(tmp_path):  # test_scene.cpp:71-112
    p = _write(tmp_path, "loads.scene",
               "# leading comment\n\n[body]\nname = a  # trailing comment\nyoungs = 10\n\n[bc]\nbody = a\n"
               "axes = zx\nvalue = 0 0 -0.25\n\n[load]\nbody = a\npressure = 3.5\n\n[load]\nbody = a\n"
               "pressure = 1\ndirection = 0 0 -2\n\n[body_force]\nforce = 0 0 -9.8\n")
    cfg = SC.parse_scene(p)
    assert cfg.bodies[0].name == "a" and cfg.bcs[0].axes == [True, False, True]
    assert cfg.bcs[0].value == (0.0, 0.0, -0.25)
    assert cfg.loads[0].direction is None and cfg.loads[0].pressure == 3.5
    assert cfg.loads[1].direction == (0.0, 0.0, -1.0)
    assert cfg.body_force == (0.0, 0.0, -9.8)


@pytest.mark.parametrize("text,line,what", [  # test_scene.cpp:114-134
    ("[body\n", 1, "unterminated section header"),
    ("[frobnicate]\n", 1, "unknown section [frobnicate]"),
    ("name = x\n", 1, "key 'name' outside any section"),
    ("[body]\njust some text\n", 2, "expected key = value"),
    ("[body]\n= 3\n", 2, "empty key"),
    ("[body]\nyoungs =\n", 2, "key 'youngs' has no value"),
    ("[body]\nname = a\nyoungs = 1\nwobble = 3\n", 4, "unknown key 'wobble' in [body]"),
    ("[body]\nname = a\nsize = 1 2\n", 3, "key 'size' expects 3 number(s)"),
    ("[body]\nname = a\nsize = 1 2 3 4\n", 3, "key 'size' expects 3 number(s)"),
    ("[solver]\nload_steps = 2.5\n", 2, "key 'load_steps' expects an integer"),
    ("[output]\nvolume_meshes = maybe\n", 2, "key 'volume_meshes' expects true or false"),
    ("[body]\nname = a\ndivisions = 0 2 2\n", 3, "divisions must be positive integers"),
    ("[body]\nname = a\ngenerator = tets\n", 3, "generator must be 'block' or 'mesh'"),
    ("[bc]\naxes = xq\n", 2, "axes must be a subset of xyz"),
    ("[bc]\nbox = 0 0 0 -1 1 1\n", 2, "key 'box' has min > max"),
])
def test_parse_failures_carry_file_line_reason(tmp_path, text, line, what):
    _expect(tmp_path, text, line, what)


ONE = "[body]\nname = a\nyoungs = 5\n\n"


@pytest.mark.parametrize("text,line,what", [  # test_scene.cpp:136-163
    ("[body]\nyoungs = 5\n", 1, "[body] requires a name"),
    ("[body]\nname = a\n", 1, "body 'a': youngs must be positive"),
    ("[body]\nname = a\nyoungs = 5\npoisson = 0.5\n", 1, "body 'a': poisson must lie in (-1, 0.5)"),
    ("[body]\nname = a\nyoungs = 5\nsize = 1 0 1\n", 1, "body 'a': size must be positive"),
    ("[body]\nname = a\nyoungs = 5\ngenerator = mesh\n", 1, "body 'a': mesh generator requires node and ele paths"),
    (ONE + "[body]\nname = a\nyoungs = 5\n", 5, "duplicate body name 'a'"),
    (ONE + "[bc]\nbody = ghost\naxes = z\n", 5, "[bc] key 'body' references absent body 'ghost'"),
    (ONE + "[bc]\nbody = a\n", 5, "[bc] constrains no axes"),
    (ONE + "[bc]\nbody = a\naxes = z\n\n[load]\nbody = ghost\n", 9, "[load] key 'body' references absent body 'ghost'"),
    (ONE + "[contact]\nslave = ghost\nmaster = a\n", 5, "[contact] key 'slave' references absent body 'ghost'"),
    (ONE + "[contact]\nslave = a\nmaster = ghost\n", 5, "[contact] key 'master' references absent body 'ghost'"),
    (ONE + "[contact]\nslave = a\nmaster = a\nkappa_face = -1\n", 5, "[contact] kappa_face must be positive"),
    (ONE + "[contact]\nslave = a\nmaster = a\neps_max = 0\n", 5, "[contact] eps_max must be positive"),
])
def test_validation_points_at_section_header(tmp_path, text, line, what):
    _expect(tmp_path, text, line, what)


def test_loads_need_a_boundary_condition(tmp_path):  # test_scene.cpp:165-191
    p = _write(tmp_path, "l.scene", ONE + "[load]\nbody = a\npressure = 1\n")
    with pytest.raises(ConfigError):
        SC.parse_scene(p)
    p = _write(tmp_path, "l2.scene", ONE + "[body_force]\nforce = 0 0 -1\n")
    with pytest.raises(ConfigError):
        SC.parse_scene(p)


def test_selectors_that_miss_fail_at_build(tmp_path):  # test_scene.cpp:193-256
    base = ONE + "[bc]\nbody = a\nbox = -1 -1 -1 2 2 1e-9\naxes = xyz\n\n"
    for extra, line, what in (("[bc]\nbody = a\nbox = 5 5 5 6 6 6\naxes = z\n", 10, "[bc] box selects no vertices"),
                              ("[load]\nbody = a\nbox = 5 5 5 6 6 6\npressure = 1\n", 10,
                               "[load] box selects no boundary faces"),
                              ("[contact]\nslave = a\nmaster = a\nslave_box = 5 5 5 6 6 6\n", 10,
                               "[contact] slave_box selects no faces")):
        p = _write(tmp_path, "m.scene", base + extra)
        cfg = SC.parse_scene(p)
        with pytest.raises(ParseError) as e:
            SC.assemble_scene(cfg)
        assert str(e.value) == f"{p}:{line}: {what}"


def test_tet_mesh_files(tmp_path):
    node = _write(tmp_path, "m.node", "# tetgen\n5 3 0 0\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n5 1 1 1\n")
    ele = _write(tmp_path, "m.ele", "2 4 0\n1 1 2 3 4\n2 2 3 4 5\n")
    m = SC.load_tet_mesh(node, ele)
    assert m.vertices.shape == (5, 3) and m.tets.shape == (2, 4)
    from paper_2605_24339_b200 import scenes as S
    assert np.all(S.tet_signed_volume(m.vertices, m.tets.astype(np.int64)) > 0)  # repaired orientation
    bad = _write(tmp_path, "b.ele", "1 4 0\n1 1 2 3 9\n")
    with pytest.raises(ParseError) as e:
        SC.load_tet_mesh(node, bad)
    assert str(e.value) == f"{bad}:2: element 0: vertex reference out of range: 9"


@pytest.mark.parametrize("path", SCENE_FILES, ids=[os.path.basename(p) for p in SCENE_FILES])
def test_scene_arrays_match_reference_bitwise(ref, path):
    """f_ext, Dirichlet mask and targets, slave selections == the reference's build_scene."""
    cfg = SC.parse_scene(path)
    A = SC.assemble_scene(cfg)
    L = ref.lib
    n = C.c_int64()
    pb = path.encode()
    assert L.ref_scene_arrays(C.c_char_p(pb), C.byref(n), None, None, None, None, C.c_int32(0)) == 0
    f, fx, dr, ns = np.zeros(n.value), np.zeros(n.value, np.uint8), np.zeros(n.value), np.zeros(8, np.int64)
    assert L.ref_scene_arrays(C.c_char_p(pb), C.byref(n), C.c_void_p(f.ctypes.data), C.c_void_p(fx.ctypes.data),
                              C.c_void_p(dr.ctypes.data), C.c_void_p(ns.ctypes.data), C.c_int32(8)) == 0
    assert n.value == A.rest.size
    assert np.array_equal(f, A.f_ext) and np.array_equal(fx, A.fixed) and np.array_equal(dr, A.dirichlet)
    assert [int(v) for v in ns[:len(A.contacts)]] == [int(c[3].size) for c in A.contacts]
