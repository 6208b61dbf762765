"""Declarative scene files on the device System: parse_scene / validate_scene /
build_scene (proj/include/gmcp/scene.hpp:19-449) and load_tet_mesh
(mesh_io.hpp:12-105), restated in Python with the reference's keys, defaults,
validation order and error messages ("<path>:<line>: <what>").

The file format is the reference's: line oriented, [section] headers start an
entry, "key = value" lines fill it, '#' starts a comment. Sections: [body]
(generator block | mesh), [bc], [load], [body_force], [contact], [solver],
[output]. build_scene returns a device System (system.py) whose solve() runs
the whole load-stepping Newton loop on the GPU.

Host-side set-up only: nothing here is on the per-iteration
path. Force lumping reproduces the reference's IEEE op order so f_ext is
bitwise the reference's.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import scenes as S
from .gmcp import ConfigError, ParseError


@dataclass
class SelectorBox:
    """scene.hpp:20-34: inclusive axis-aligned selector over rest positions."""
    lo: tuple = (-1e30, -1e30, -1e30)
    hi: tuple = (1e30, 1e30, 1e30)

    def contains(self, p) -> bool:
        return (p[0] >= self.lo[0] and p[0] <= self.hi[0] and p[1] >= self.lo[1] and p[1] <= self.hi[1]
                and p[2] >= self.lo[2] and p[2] <= self.hi[2])

    def contains_all(self, P: np.ndarray) -> np.ndarray:
        lo, hi = np.asarray(self.lo, float), np.asarray(self.hi, float)
        return np.all((P >= lo) & (P <= hi), axis=-1)


@dataclass
class BodySpec:
    name: str = ""
    generator: str = "block"
    size: tuple = (1.0, 1.0, 1.0)
    divisions: tuple = (1, 1, 1)
    origin: tuple = (0.0, 0.0, 0.0)
    node_path: str = ""
    ele_path: str = ""
    youngs: float = -1.0
    poisson: float = 0.0
    translate: tuple = (0.0, 0.0, 0.0)
    line: int = 0


@dataclass
class BcSpec:
    body: str = ""
    box: SelectorBox = field(default_factory=SelectorBox)
    axes: list = field(default_factory=lambda: [False, False, False])
    value: tuple = (0.0, 0.0, 0.0)
    line: int = 0


@dataclass
class LoadSpec:
    body: str = ""
    box: SelectorBox = field(default_factory=SelectorBox)
    pressure: float = 0.0
    direction: tuple | None = None
    line: int = 0


@dataclass
class ContactSpec:
    slave: str = ""
    master: str = ""
    slave_box: SelectorBox | None = None
    params: S.BarrierParams = field(default_factory=S.BarrierParams)
    line: int = 0


@dataclass
class OutputSpec:
    directory: str = "out"
    volume_meshes: bool = True
    surface_meshes: bool = True
    pressure_csv: bool = True


@dataclass
class SolverSpec:
    load_steps: int = 10
    max_newton_iters: int = 200
    newton_tol: float = -1.0
    max_line_search: int = 40


@dataclass
class SceneConfig:
    path: str = "<builtin>"
    bodies: list = field(default_factory=list)
    bcs: list = field(default_factory=list)
    loads: list = field(default_factory=list)
    body_force: tuple | None = None
    contacts: list = field(default_factory=list)
    solver: SolverSpec = field(default_factory=SolverSpec)
    output: OutputSpec = field(default_factory=OutputSpec)


def _fail(path, line, what):
    raise ParseError(f"{path}:{line}: {what}")


def _reals(path, line, key, value, n):
    toks = value.split()
    out = []
    for i in range(n):
        try:
            out.append(float(toks[i]))
        except (IndexError, ValueError):
            _fail(path, line, f"key '{key}' expects {n} number(s)")
    if len(toks) > n:
        _fail(path, line, f"key '{key}' expects {n} number(s)")
    return out


def _real(path, line, key, value):
    return _reals(path, line, key, value, 1)[0]


def _int(path, line, key, value):
    r = _real(path, line, key, value)
    if not math.isfinite(r) or float(int(r)) != r:
        _fail(path, line, f"key '{key}' expects an integer")
    return int(r)


def _bool(path, line, key, value):
    if value in ("true", "1"):
        return True
    if value in ("false", "0"):
        return False
    _fail(path, line, f"key '{key}' expects true or false")


def _vec3(path, line, key, value):
    return tuple(_reals(path, line, key, value, 3))


def _normalized(v):
    """Eigen normalized() as in the shim: divide by sqrt(squaredNorm) if > 0."""
    z = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]
    if z > 0:
        n = math.sqrt(z)
        return (v[0] / n, v[1] / n, v[2] / n)
    return tuple(v)


def _box(path, line, key, value):
    v = _reals(path, line, key, value, 6)
    b = SelectorBox(tuple(v[:3]), tuple(v[3:]))
    for k in range(3):
        if b.lo[k] > b.hi[k]:
            _fail(path, line, f"key '{key}' has min > max")
    return b


def parse_scene(path: str) -> SceneConfig:
    """scene.hpp:155-328."""
    try:
        f = open(path)
    except OSError:
        raise ParseError(f"{path}: cannot open")
    cfg = SceneConfig(path=path)
    section = ""
    with f:
        for line, raw in enumerate(f, start=1):
            raw = raw.split("#", 1)[0]
            s = raw.strip(" \t\r\n")
            if not s:
                continue
            if s[0] == "[":
                if s[-1] != "]":
                    _fail(path, line, "unterminated section header")
                section = s[1:-1].strip(" \t\r\n")
                if section == "body":
                    cfg.bodies.append(BodySpec(line=line))
                elif section == "bc":
                    cfg.bcs.append(BcSpec(line=line))
                elif section == "load":
                    cfg.loads.append(LoadSpec(line=line))
                elif section == "contact":
                    cfg.contacts.append(ContactSpec(line=line))
                elif section not in ("body_force", "solver", "output"):
                    _fail(path, line, f"unknown section [{section}]")
                continue
            eq = s.find("=")
            if eq < 0:
                _fail(path, line, "expected key = value")
            key, value = s[:eq].strip(" \t\r\n"), s[eq + 1:].strip(" \t\r\n")
            if not key:
                _fail(path, line, "empty key")
            if not value:
                _fail(path, line, f"key '{key}' has no value")
            if not section:
                _fail(path, line, f"key '{key}' outside any section")
            if section == "body":
                b = cfg.bodies[-1]
                if key == "name":
                    b.name = value
                elif key == "generator":
                    if value not in ("block", "mesh"):
                        _fail(path, line, "generator must be 'block' or 'mesh'")
                    b.generator = value
                elif key == "size":
                    b.size = _vec3(path, line, key, value)
                elif key == "divisions":
                    v = _reals(path, line, key, value, 3)
                    d = []
                    for x in v:
                        i = int(x) if math.isfinite(x) else 0
                        if float(i) != x or i < 1:
                            _fail(path, line, "divisions must be positive integers")
                        d.append(i)
                    b.divisions = tuple(d)
                elif key == "origin":
                    b.origin = _vec3(path, line, key, value)
                elif key == "node":
                    b.node_path = value
                elif key == "ele":
                    b.ele_path = value
                elif key == "youngs":
                    b.youngs = _real(path, line, key, value)
                elif key == "poisson":
                    b.poisson = _real(path, line, key, value)
                elif key == "translate":
                    b.translate = _vec3(path, line, key, value)
                else:
                    _fail(path, line, f"unknown key '{key}' in [body]")
            elif section == "bc":
                bc = cfg.bcs[-1]
                if key == "body":
                    bc.body = value
                elif key == "box":
                    bc.box = _box(path, line, key, value)
                elif key == "axes":
                    bc.axes = [False, False, False]
                    for ch in value:
                        if ch not in "xyz":
                            _fail(path, line, "axes must be a subset of xyz")
                        bc.axes["xyz".index(ch)] = True
                elif key == "value":
                    bc.value = _vec3(path, line, key, value)
                else:
                    _fail(path, line, f"unknown key '{key}' in [bc]")
            elif section == "load":
                ld = cfg.loads[-1]
                if key == "body":
                    ld.body = value
                elif key == "box":
                    ld.box = _box(path, line, key, value)
                elif key == "pressure":
                    ld.pressure = _real(path, line, key, value)
                elif key == "direction":
                    ld.direction = _normalized(_vec3(path, line, key, value))
                else:
                    _fail(path, line, f"unknown key '{key}' in [load]")
            elif section == "body_force":
                if key == "force":
                    cfg.body_force = _vec3(path, line, key, value)
                else:
                    _fail(path, line, f"unknown key '{key}' in [body_force]")
            elif section == "contact":
                c = cfg.contacts[-1]
                p = c.params
                if key == "slave":
                    c.slave = value
                elif key == "master":
                    c.master = value
                elif key == "slave_box":
                    c.slave_box = _box(path, line, key, value)
                elif key in ("kappa_face", "kappa_edge", "kappa_point", "eps_max", "delta_face", "delta_edge",
                             "detection_radius"):
                    setattr(p, key, _real(path, line, key, value))
                elif key in ("quad_order_face", "quad_order_edge"):
                    setattr(p, key, _int(path, line, key, value))
                else:
                    _fail(path, line, f"unknown key '{key}' in [contact]")
            elif section == "solver":
                sv = cfg.solver
                if key in ("load_steps", "max_newton_iters", "max_line_search"):
                    setattr(sv, key, _int(path, line, key, value))
                elif key == "newton_tol":
                    sv.newton_tol = _real(path, line, key, value)
                else:
                    _fail(path, line, f"unknown key '{key}' in [solver]")
            elif section == "output":
                o = cfg.output
                if key == "directory":
                    o.directory = value
                elif key in ("volume_meshes", "surface_meshes", "pressure_csv"):
                    setattr(o, key, _bool(path, line, key, value))
                else:
                    _fail(path, line, f"unknown key '{key}' in [output]")
    validate_scene(cfg)
    return cfg


def find_body(cfg: SceneConfig, name: str) -> int:
    for i, b in enumerate(cfg.bodies):
        if b.name == name:
            return i
    return -1


def validate_scene(cfg: SceneConfig):
    """scene.hpp:336-380."""
    path = cfg.path
    for i, b in enumerate(cfg.bodies):
        if not b.name:
            _fail(path, b.line, "[body] requires a name")
        if any(cfg.bodies[j].name == b.name for j in range(i)):
            _fail(path, b.line, f"duplicate body name '{b.name}'")
        if b.youngs <= 0:
            _fail(path, b.line, f"body '{b.name}': youngs must be positive")
        if b.poisson <= -1 or b.poisson >= 0.5:
            _fail(path, b.line, f"body '{b.name}': poisson must lie in (-1, 0.5)")
        if b.generator == "block":
            if not (min(b.size) > 0):
                _fail(path, b.line, f"body '{b.name}': size must be positive")
        elif not b.node_path or not b.ele_path:
            _fail(path, b.line, f"body '{b.name}': mesh generator requires node and ele paths")
    for bc in cfg.bcs:
        if find_body(cfg, bc.body) < 0:
            _fail(path, bc.line, f"[bc] key 'body' references absent body '{bc.body}'")
        if not any(bc.axes):
            _fail(path, bc.line, "[bc] constrains no axes")
    for ld in cfg.loads:
        if find_body(cfg, ld.body) < 0:
            _fail(path, ld.line, f"[load] key 'body' references absent body '{ld.body}'")
    for c in cfg.contacts:
        if find_body(cfg, c.slave) < 0:
            _fail(path, c.line, f"[contact] key 'slave' references absent body '{c.slave}'")
        if find_body(cfg, c.master) < 0:
            _fail(path, c.line, f"[contact] key 'master' references absent body '{c.master}'")
        if c.params.kappa_face <= 0:
            _fail(path, c.line, "[contact] kappa_face must be positive")
        if c.params.eps_max <= 0:
            _fail(path, c.line, "[contact] eps_max must be positive")
    if (cfg.loads or cfg.body_force is not None) and not cfg.bcs:
        raise ConfigError(f"{path}: loads require at least one boundary condition")
    if cfg.solver.load_steps < 1:
        raise ConfigError(f"{path}: load_steps must be >= 1")


def _next_data_line(lines, i):
    while i < len(lines):
        s = lines[i].split("#", 1)[0]
        i += 1
        if s.strip(" \t\r\n"):
            return s, i
    return None, i


def load_tet_mesh(node_path: str, ele_path: str) -> S.TetMesh:
    """mesh_io.hpp:30-105: TetGen-style .node / .ele (0- or 1-based)."""
    def read(p):
        try:
            with open(p) as f:
                return f.read().split("\n")
        except OSError:
            raise ParseError(f"{p}: cannot open")

    lines = read(node_path)
    s, i = _next_data_line(lines, 0)
    if s is None:
        _fail(node_path, i, "missing header")
    t = s.split()
    try:
        n, dim = int(t[0]), int(t[1])
    except (IndexError, ValueError):
        _fail(node_path, i, "malformed header")
    if dim != 3:
        _fail(node_path, i, "expected dimension 3")
    if n < 0:
        _fail(node_path, i, "negative vertex count")
    verts, base = [], -1
    for k in range(n):
        s, i = _next_data_line(lines, i)
        if s is None:
            _fail(node_path, i, "unexpected end of file")
        t = s.split()
        try:
            idx, x, y, z = int(t[0]), float(t[1]), float(t[2]), float(t[3])
        except (IndexError, ValueError):
            _fail(node_path, i, "malformed vertex line")
        if k == 0:
            if idx not in (0, 1):
                _fail(node_path, i, "first vertex index must be 0 or 1")
            base = idx
        if idx != base + k:
            _fail(node_path, i, "non-consecutive vertex index")
        verts.append((x, y, z))
    lines = read(ele_path)
    s, i = _next_data_line(lines, 0)
    if s is None:
        _fail(ele_path, i, "missing header")
    t = s.split()
    try:
        n, npt = int(t[0]), int(t[1])
    except (IndexError, ValueError):
        _fail(ele_path, i, "malformed header")
    if npt != 4:
        _fail(ele_path, i, "expected 4 nodes per tet")
    if n < 0:
        _fail(ele_path, i, "negative tet count")
    nv = len(verts)
    tets = []
    for k in range(n):
        s, i = _next_data_line(lines, i)
        if s is None:
            _fail(ele_path, i, "unexpected end of file")
        t = s.split()
        try:
            v = [int(t[0])] + [int(t[j]) for j in range(1, 5)]
        except (IndexError, ValueError):
            _fail(ele_path, i, "malformed tet line")
        tet = []
        for r in v[1:]:
            ref = r - base
            if ref < 0 or ref >= nv:
                _fail(ele_path, i, f"element {k}: vertex reference out of range: {r}")
            tet.append(ref)
        tets.append(tet)
    V = np.asarray(verts, np.float64).reshape(-1, 3)
    T = np.asarray(tets, np.int64).reshape(-1, 4)
    return S.TetMesh(V, S.orient_tets_positive(V, T).astype(np.int32))


def _tet_volumes(V: np.ndarray, T: np.ndarray) -> np.ndarray:
    """elasticity.hpp:40-48: det([b-a | c-a | d-a]) / 6 in the reference's cofactor order."""
    a = V[T[:, 0]]
    d0, d1, d2 = V[T[:, 1]] - a, V[T[:, 2]] - a, V[T[:, 3]] - a  # columns of D
    m = lambda r, c: (d0, d1, d2)[c][:, r]  # noqa: E731  D(r, c)
    det = (m(0, 0) * (m(1, 1) * m(2, 2) - m(2, 1) * m(1, 2)) - m(1, 0) * (m(0, 1) * m(2, 2) - m(2, 1) * m(0, 2))) + \
        m(2, 0) * (m(0, 1) * m(1, 2) - m(1, 1) * m(0, 2))
    return det / 6.0


@dataclass
class SceneArrays:
    """Everything build_scene hands to System, assembled on the host."""
    meshes: list
    names: list
    youngs: list
    poisson: list
    offsets: list
    boundaries: list
    rest: np.ndarray
    fixed: np.ndarray       # (3N,) uint8
    dirichlet: np.ndarray   # (3N,)
    f_ext: np.ndarray       # (3N,)
    contacts: list          # (slave body, master body, raw params, slave tri subset or None)


def assemble_scene(cfg: SceneConfig) -> SceneArrays:
    """scene.hpp:382-449 up to the System calls: meshes, Dirichlet targets,
    pressure and body-force loads (bitwise the reference's f_ext), contact
    slave selections. Selector errors surface here, as in the reference."""
    meshes, offsets = [], []
    n = 0
    for b in cfg.bodies:
        mesh = S.make_block(b.size, b.divisions, b.origin) if b.generator == "block" else \
            load_tet_mesh(b.node_path, b.ele_path)
        if tuple(b.translate) != (0.0, 0.0, 0.0):
            mesh = S.TetMesh(mesh.vertices + np.asarray(b.translate, np.float64), mesh.tets)
        meshes.append(mesh)
        offsets.append(n)
        n += mesh.vertices.shape[0]
    rest = np.concatenate([m.vertices.ravel() for m in meshes]).astype(np.float64) if meshes else np.zeros(0)
    bnds = [S.extract_boundary_surface(m) for m in meshes]
    fixed = np.zeros(rest.size, np.uint8)
    dirichlet = rest.copy()
    r3 = rest.reshape(-1, 3)
    for bc in cfg.bcs:
        bi = find_body(cfg, bc.body)
        gv = offsets[bi] + np.arange(meshes[bi].vertices.shape[0])
        sel = gv[bc.box.contains_all(r3[gv])]
        if sel.size == 0:
            _fail(cfg.path, bc.line, "[bc] box selects no vertices")
        for k in range(3):
            if bc.axes[k]:
                fixed[3 * sel + k] = 1
                dirichlet[3 * sel + k] = r3[sel, k] + bc.value[k]
    f_ext = np.zeros_like(rest)
    for ld in cfg.loads:
        bi = find_body(cfg, ld.body)
        gtris = offsets[bi] + bnds[bi].vertex_map[bnds[bi].triangles]
        faces = gtris[np.all(ld.box.contains_all(r3[gtris]), axis=1)]
        if faces.shape[0] == 0:
            _fail(cfg.path, ld.line, "[load] box selects no boundary faces")
        S.add_pressure_forces(faces, rest, ld.pressure, ld.direction, f_ext)
    if cfg.body_force is not None:  # elasticity.hpp:162-168, bodies then tets in order
        bf = cfg.body_force
        for m, off in zip(meshes, offsets):
            vol4 = _tet_volumes(m.vertices, m.tets.astype(np.int64)) / 4.0
            for t, tet in enumerate(m.tets.tolist()):
                w = float(vol4[t])
                for v in tet:
                    g = 3 * (off + v)
                    f_ext[g] += w * bf[0]
                    f_ext[g + 1] += w * bf[1]
                    f_ext[g + 2] += w * bf[2]
    contacts = []
    for c in cfg.contacts:
        si, mi = find_body(cfg, c.slave), find_body(cfg, c.master)
        subset = None
        if c.slave_box is not None:
            gtris = offsets[si] + bnds[si].vertex_map[bnds[si].triangles]
            subset = np.nonzero(np.all(c.slave_box.contains_all(r3[gtris]), axis=1))[0]
            if subset.size == 0:
                _fail(cfg.path, c.line, "[contact] slave_box selects no faces")
        contacts.append((si, mi, c.params, subset))
    return SceneArrays(meshes, [b.name for b in cfg.bodies], [b.youngs for b in cfg.bodies],
                       [b.poisson for b in cfg.bodies], offsets, bnds, rest, fixed, dirichlet, f_ext, contacts)


def build_scene(cfg: SceneConfig, device: int = 0):
    """scene.hpp:382-449 onto the device System."""
    from . import system as SY
    A = assemble_scene(cfg)
    sys_ = SY.System(device)
    for m, name, E, nu in zip(A.meshes, A.names, A.youngs, A.poisson):
        sys_.add_body(m, E, nu, name)
    sys_.fixed[:] = A.fixed
    sys_.dirichlet[:] = A.dirichlet
    sys_.f_ext[:] = A.f_ext
    for si, mi, params, subset in A.contacts:
        sys_.add_contact_pair(si, mi, params, subset, None)
    return sys_


def solver_settings(cfg: SceneConfig, **pcg):
    """SolverSettings from the scene's [solver] section (+ PCG controls)."""
    from . import system as SY
    sv = cfg.solver
    return SY.SolverSettings(load_steps=sv.load_steps, max_newton_iters=sv.max_newton_iters,
                             newton_tol=sv.newton_tol, max_line_search=sv.max_line_search, **pcg)


def run_scene(path: str, device: int = 0, on_step=None, **pcg):
    """parse_scene + build_scene + System::solve (the CLI's `run` path without
    file output). Returns (System, RunStats)."""
    cfg = parse_scene(path)
    sys_ = build_scene(cfg, device)
    stats = sys_.solve(solver_settings(cfg, **pcg), on_step)
    return sys_, stats


SCENE_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scenes")
