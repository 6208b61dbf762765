"""Run outputs of a scene: per-step legacy-ASCII VTK volume / surface meshes,
pressure CSV tables read back from the device, and the ordered key=value run
report -- vtk_io.hpp:1-144, bench.hpp:310-402 (write_step_outputs, run_scene)
and scene.hpp:451-530 (echo_scene), restated with the reference's layouts and
number formatting (format_real = "%.17g", core.hpp:116-120).

Files of a repeated run are byte-identical (the device solve is deterministic
and sequential mode leaves wall-clock time out of the report), which is the
reference's determinism criterion 10. Host-side I/O around the hot path.
"""
from __future__ import annotations

import os

import numpy as np

from . import scene as SC
from .gmcp import ParseError


def format_real(v: float) -> str:
    return "%.17g" % float(v)


def _write(path: str, text: str):
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError:
        raise ParseError(f"{path}: cannot open for writing")


def _fields(fields, count, path, out):
    for name, comps, data in fields:
        data = np.asarray(data, np.float64).ravel()
        if data.size != count * comps:
            raise ParseError(f"{path}: field '{name}' size mismatch")
        if comps == 1:
            out.append(f"SCALARS {name} double 1\nLOOKUP_TABLE default\n")
            out.extend(format_real(v) + "\n" for v in data.tolist())
        elif comps == 3:
            out.append(f"VECTORS {name} double\n")
            d = data.tolist()
            out.extend(f"{format_real(d[3 * i])} {format_real(d[3 * i + 1])} {format_real(d[3 * i + 2])}\n"
                       for i in range(count))
        elif comps == 9:
            out.append(f"TENSORS {name} double\n")
            d = data.tolist()
            for i in range(count):
                for r in range(3):
                    b = 9 * i + 3 * r
                    out.append(f"{format_real(d[b])} {format_real(d[b + 1])} {format_real(d[b + 2])}\n")
                out.append("\n")
        else:
            raise ParseError(f"{path}: field '{name}' has unsupported component count")


def _write_grid(path, points, cells, cell_type, point_fields=(), cell_fields=()):
    """vtk_io.hpp:55-83."""
    P = np.asarray(points, np.float64).reshape(-1, 3)
    Cc = np.asarray(cells, np.int64)
    N = Cc.shape[1] if Cc.ndim == 2 and Cc.size else (4 if cell_type == 10 else 3)
    out = ["# vtk DataFile Version 3.0\ngmcp output\nASCII\nDATASET UNSTRUCTURED_GRID\n",
           f"POINTS {P.shape[0]} double\n"]
    out.extend(f"{format_real(x)} {format_real(y)} {format_real(z)}\n" for x, y, z in P.tolist())
    out.append(f"CELLS {Cc.shape[0]} {Cc.shape[0] * (N + 1)}\n")
    out.extend(f"{N} " + " ".join(str(k) for k in c) + "\n" for c in Cc.tolist())
    out.append(f"CELL_TYPES {Cc.shape[0]}\n")
    out.extend(f"{cell_type}\n" for _ in range(Cc.shape[0]))
    if point_fields:
        out.append(f"POINT_DATA {P.shape[0]}\n")
        _fields(point_fields, P.shape[0], path, out)
    if cell_fields:
        out.append(f"CELL_DATA {Cc.shape[0]}\n")
        _fields(cell_fields, Cc.shape[0], path, out)
    _write(path, "".join(out))


def save_vtk_tets(path, points, tets, point_fields=(), cell_fields=()):
    """vtk_io.hpp:87-92. fields: (name, components, data)."""
    _write_grid(path, points, tets, 10, point_fields, cell_fields)


def save_vtk_tris(path, points, tris, point_fields=(), cell_fields=()):
    """vtk_io.hpp:94-99."""
    _write_grid(path, points, tris, 5, point_fields, cell_fields)


def save_csv(path, header, rows):
    """vtk_io.hpp:101-115."""
    out = [",".join(header) + "\n"]
    for row in rows:
        if len(row) != len(header):
            raise ParseError(f"{path}: row width does not match header")
        out.append(",".join(format_real(v) for v in row) + "\n")
    _write(path, "".join(out))


class Report:
    """vtk_io.hpp:117-142: ordered key=value report."""

    def __init__(self):
        self.entries: list[list[str]] = []

    def set(self, key: str, value):
        if isinstance(value, bool):
            value = "true" if value else "false"
        elif isinstance(value, (int, np.integer)):
            value = str(int(value))
        elif isinstance(value, (float, np.floating)):
            value = format_real(value)
        for e in self.entries:
            if e[0] == key:
                e[1] = value
                return
        self.entries.append([key, value])

    def find(self, key: str):
        for k, v in self.entries:
            if k == key:
                return v
        return None

    def save(self, path: str):
        _write(path, "".join(f"{k}={v}\n" for k, v in self.entries))


def step_name(step: int, what: str, ext: str) -> str:
    return f"step_{step:02d}_{what}.{ext}"


def _elem_stress(mesh, E, nu, x, rest, off):
    """bench.hpp:18-25 per element (small-strain Cauchy stress)."""
    from .system import body_stresses, Body
    b = Body(mesh, E, nu, "", off, None)
    return body_stresses(b, x, rest)


def write_step_outputs(sys_, cfg: SC.SceneConfig, x: np.ndarray, step: int):
    """bench.hpp:322-372: volume mesh (displacement + Cauchy stress), surface
    mesh and the per-pair contact pressure table (from the device)."""
    d = cfg.output.directory
    pts = x.reshape(-1, 3)
    if cfg.output.volume_meshes:
        cells, stress = [], []
        for b in sys_.bodies:
            cells.append(b.vertex_offset + b.mesh.tets.astype(np.int64))
            stress.append(_elem_stress(b.mesh, b.youngs, b.poisson, x, sys_.rest, b.vertex_offset).reshape(-1, 9))
        disp = (x - sys_.rest).reshape(-1, 3)
        save_vtk_tets(os.path.join(d, step_name(step, "volume", "vtk")), pts, np.concatenate(cells),
                      [("displacement", 3, disp)], [("cauchy_stress", 9, np.concatenate(stress))])
    if cfg.output.surface_meshes:
        tris = [b.vertex_offset + b.boundary.vertex_map[b.boundary.triangles] for b in sys_.bodies]
        save_vtk_tris(os.path.join(d, step_name(step, "surface", "vtk")), pts, np.concatenate(tris))
    if cfg.output.pressure_csv and sys_.contacts:
        rows = []
        for ci in range(len(sys_.contacts)):
            for r in sys_.contact_pressure_field(ci).tolist():  # device buffers -> host
                sample, pos, _radius, gap, p = r
                rows.append((float(ci), float(sample), pos[0], pos[1], pos[2], gap, p))
        save_csv(os.path.join(d, step_name(step, "pressure", "csv")),
                 ["pair", "sample", "x", "y", "z", "gap", "pressure"], rows)


def _v3(v):
    return " ".join(format_real(t) for t in v)


def echo_scene(cfg: SC.SceneConfig, sys_, rep: Report):
    """scene.hpp:451-530: every value that influences the run, defaults
    included; resolved contact parameters from the built system."""
    rep.set("scene.path", cfg.path)
    rep.set("scene.bodies", len(cfg.bodies))
    for b in cfg.bodies:
        k = f"body.{b.name}."
        rep.set(k + "generator", b.generator)
        if b.generator == "block":
            rep.set(k + "size", _v3(b.size))
            rep.set(k + "divisions", " ".join(str(int(t)) for t in b.divisions))
            rep.set(k + "origin", _v3(b.origin))
        else:
            rep.set(k + "node", b.node_path)
            rep.set(k + "ele", b.ele_path)
        rep.set(k + "youngs", float(b.youngs))
        rep.set(k + "poisson", float(b.poisson))
        rep.set(k + "translate", _v3(b.translate))
    for i, bc in enumerate(cfg.bcs):
        k = f"bc.{i}."
        rep.set(k + "body", bc.body)
        rep.set(k + "box", _v3(bc.box.lo) + " " + _v3(bc.box.hi))
        rep.set(k + "axes", "".join(a for a, on in zip("xyz", bc.axes) if on))
        rep.set(k + "value", _v3(bc.value))
    for i, ld in enumerate(cfg.loads):
        k = f"load.{i}."
        rep.set(k + "body", ld.body)
        rep.set(k + "box", _v3(ld.box.lo) + " " + _v3(ld.box.hi))
        rep.set(k + "pressure", float(ld.pressure))
        rep.set(k + "direction", _v3(ld.direction) if ld.direction is not None else "inward_normal")
    if cfg.body_force is not None:
        rep.set("body_force", _v3(cfg.body_force))
    for i, c in enumerate(cfg.contacts):
        k = f"contact.{i}."
        rep.set(k + "slave", c.slave)
        rep.set(k + "master", c.master)
        if c.slave_box is not None:
            rep.set(k + "slave_box", _v3(c.slave_box.lo) + " " + _v3(c.slave_box.hi))
        p = sys_.contacts[i][2] if sys_ is not None else c.params
        for key in ("kappa_face", "kappa_edge", "kappa_point", "eps_max", "delta_face", "delta_edge",
                    "detection_radius"):
            rep.set(k + key, float(getattr(p, key)))
        rep.set(k + "quad_order_face", int(p.quad_order_face))
        rep.set(k + "quad_order_edge", int(p.quad_order_edge))
    sv = cfg.solver
    rep.set("solver.load_steps", int(sv.load_steps))
    rep.set("solver.max_newton_iters", int(sv.max_newton_iters))
    rep.set("solver.max_line_search", int(sv.max_line_search))
    rep.set("solver.newton_tol", "derived" if sv.newton_tol < 0 else format_real(sv.newton_tol))
    rep.set("output.directory", cfg.output.directory)
    for key in ("volume_meshes", "surface_meshes", "pressure_csv"):
        rep.set("output." + key, "true" if getattr(cfg.output, key) else "false")


def run_scene(cfg: SC.SceneConfig, out_override: str = "", sequential: bool = False, dry_run: bool = False,
              device: int = 0, **pcg) -> Report:
    """bench.hpp:374-402: build, echo, solve on the device with per-step file
    output; report.txt in the output directory."""
    if out_override:
        cfg.output.directory = out_override
    sys_ = SC.build_scene(cfg, device)
    rep = Report()
    echo_scene(cfg, sys_, rep)
    rep.set("threads", 1 if sequential else int(os.cpu_count() or 1))
    if dry_run:
        rep.set("dry_run", "true")
        return rep
    try:
        os.makedirs(cfg.output.directory, exist_ok=True)
    except OSError as e:
        from .gmcp import ConfigError
        raise ConfigError(f"{cfg.output.directory}: cannot create output directory ({e})")

    def on_step(s, x):
        write_step_outputs(sys_, cfg, x, s.step)
        k = f"step.{s.step}."
        rep.set(k + "newton_iters", int(s.newton_iters))
        rep.set(k + "rebuilds", int(s.rebuilds))
        rep.set(k + "backtracks", int(s.backtracks))
        rep.set(k + "residual", float(s.residual))
        rep.set(k + "energy", float(s.energy))
        rep.set(k + "min_gap", float(s.min_gap))

    stats = sys_.solve(SC.solver_settings(cfg, **pcg), on_step)
    rep.set("total_newton_iters", int(stats.total_newton_iters))
    rep.set("total_rebuilds", int(stats.total_rebuilds))
    rep.set("newton_tol_used", float(stats.newton_tol_used))
    if not sequential:
        rep.set("wall_seconds", float(stats.wall_seconds))
    rep.save(os.path.join(cfg.output.directory, "report.txt"))
    return rep
