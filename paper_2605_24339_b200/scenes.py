"""Host-side scene setup: tet blocks, boundary surfaces, contact surfaces and
the synthetic benchmark scenes.

This is one-time setup on either side of the hot path (out of scope for the
GPU); it is restated in numpy so the oracle and the CUDA path receive
identical arrays. Orderings follow the reference exactly and are pinned by
tests/test_scenes.py against the compiled reference:

* make_block                  <- proj/include/gmcp/tet_mesh.hpp:56-89
* orient_tets_positive        <- tet_mesh.hpp:29-39
* extract_boundary_surface    <- tet_mesh.hpp:127-168 (std::map key order)
* build_surface_edges         <- tet_mesh.hpp:102-116
* make_contact_surface        <- contact_sampling.hpp:226-255
* mean_edge_length            <- contact_sampling.hpp:257-263
* resolve_barrier_params      <- barrier.hpp:25-46
* graded_axis / mirrored_axis <- mesh_gen.hpp:14-64
* make_lattice                <- mesh_gen.hpp:66-106
* make_cylinder_sector        <- mesh_gen.hpp:119-136
* make_sphere_octant          <- mesh_gen.hpp:138-161
* hertz_scene (C1)            <- bench.hpp:134-303 (HertzConfig, meshes, BCs, slave patch)
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


@dataclass
class TetMesh:
    vertices: np.ndarray  # (nv, 3) float64
    tets: np.ndarray  # (nt, 4) int32


@dataclass
class SurfaceMesh:
    triangles: np.ndarray  # (T, 3) surface-local ids
    vertex_map: np.ndarray  # (S,) surface vertex -> volume vertex


@dataclass
class ContactSurface:
    tris: np.ndarray  # (T, 3) int32 global ids
    edges: np.ndarray  # (E, 2) int32, lo < hi, numbered by first appearance
    tri_edges: np.ndarray  # (T, 3) int32
    verts: np.ndarray  # (V,) int32 ascending


@dataclass
class BarrierParams:
    """gmcp::BarrierParams (barrier.hpp:9-19)."""

    kappa_face: float = 1e6
    kappa_edge: float = -1.0
    kappa_point: float = -1.0
    eps_max: float = 1e-3
    delta_face: float = 0.1
    delta_edge: float = 0.1
    detection_radius: float = -1.0
    quad_order_face: int = 2
    quad_order_edge: int = 2


class ConfigError(ValueError):
    """gmcp::ConfigError (core.hpp:40-43)."""


def tet_signed_volume(v: np.ndarray, tets: np.ndarray) -> np.ndarray:
    a, b, c, d = (v[tets[:, k]] for k in range(4))
    ca, da = c - a, d - a
    cr = np.stack(
        [ca[:, 1] * da[:, 2] - ca[:, 2] * da[:, 1],
         ca[:, 2] * da[:, 0] - ca[:, 0] * da[:, 2],
         ca[:, 0] * da[:, 1] - ca[:, 1] * da[:, 0]], axis=1)
    ba = b - a
    return (ba[:, 0] * cr[:, 0] + ba[:, 1] * cr[:, 1] + ba[:, 2] * cr[:, 2]) / 6.0


def orient_tets_positive(v: np.ndarray, tets: np.ndarray) -> np.ndarray:
    tets = tets.copy()
    vol = tet_signed_volume(v, tets)
    neg = vol < 0
    tets[neg, 2], tets[neg, 3] = tets[neg, 3].copy(), tets[neg, 2].copy()
    if not np.all(np.abs(vol) > 0):
        raise ValueError("degenerate tet")
    return tets


def make_block(size, divisions, origin=(0.0, 0.0, 0.0)) -> TetMesh:
    nx, ny, nz = (int(d) for d in divisions)
    if min(nx, ny, nz) < 1:
        raise ConfigError("make_block: divisions must be >= 1")
    sx, sy, sz = (float(s) for s in size)
    ox, oy, oz = (float(o) for o in origin)
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    verts = np.stack([ox + (sx * i) / nx, oy + (sy * j) / ny, oz + (sz * k) / nz], axis=1)

    def vid(a, b, c):
        return (c * (ny + 1) + b) * (nx + 1) + a

    ck, cj, ci = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    tets = np.empty((ci.size, 6, 4), dtype=np.int64)
    for q, p in enumerate(_PERMS):
        at = [ci.copy(), cj.copy(), ck.copy()]
        tets[:, q, 0] = vid(*at)
        for s in range(3):
            at[p[s]] = at[p[s]] + 1
            tets[:, q, s + 1] = vid(*at)
    tets = tets.reshape(-1, 4)
    tets = orient_tets_positive(verts, tets)
    return TetMesh(verts, tets.astype(np.int32))


def _first_appearance_unique(keys: np.ndarray):
    """Unique rows of keys numbered by first appearance; returns (uniq, inverse)."""
    uniq, first, inv = np.unique(keys, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    return uniq[order], rank[inv.ravel()]


def extract_boundary_surface(m: TetMesh) -> SurfaceMesh:
    t = m.tets.astype(np.int64)
    faces = np.stack([t[:, [0, 2, 1]], t[:, [0, 1, 3]], t[:, [0, 3, 2]], t[:, [1, 2, 3]]], axis=1)
    faces = faces.reshape(-1, 3)
    keys = np.sort(faces, axis=1)
    uniq, first, counts = np.unique(keys, axis=0, return_index=True, return_counts=True)
    if np.any(counts > 2):
        raise ValueError("extract_boundary_surface: face shared by more than two tets")
    bnd = faces[first[counts == 1]]  # key order == std::map iteration order
    flat = bnd.ravel()
    uv, firstv = np.unique(flat, return_index=True)
    order = np.argsort(firstv, kind="stable")
    vertex_map = uv[order]
    local = np.empty(int(flat.max()) + 1 if flat.size else 0, dtype=np.int64)
    local[vertex_map] = np.arange(vertex_map.size)
    tris = local[bnd]
    return SurfaceMesh(tris.astype(np.int32), vertex_map.astype(np.int32))


def make_contact_surface(s: SurfaceMesh, vertex_offset: int = 0, tri_subset=None) -> ContactSurface:
    tris_l = s.triangles if tri_subset is None else s.triangles[np.asarray(tri_subset, dtype=np.int64)]
    tris = (vertex_offset + s.vertex_map[tris_l]).astype(np.int64)
    if tris.shape[0] == 0:
        z = np.zeros((0, 3), np.int32)
        return ContactSurface(z, np.zeros((0, 2), np.int32), z, np.zeros(0, np.int32))
    a = tris
    b = np.roll(tris, -1, axis=1)
    e = np.stack([np.minimum(a, b), np.maximum(a, b)], axis=2).reshape(-1, 2)
    edges, inv = _first_appearance_unique(e)
    tri_edges = inv.reshape(-1, 3)
    verts = np.unique(tris)
    return ContactSurface(tris.astype(np.int32), edges.astype(np.int32),
                          tri_edges.astype(np.int32), verts.astype(np.int32))


def mean_edge_length(s: ContactSurface, x: np.ndarray) -> float:
    if s.edges.shape[0] == 0:
        raise ConfigError("contact surface has no edges")
    x3 = x.reshape(-1, 3)
    d = x3[s.edges[:, 0]] - x3[s.edges[:, 1]]
    n = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
    total = 0.0
    for v in n.tolist():  # sequential sum, reference order
        total += v
    return total / float(n.size)


def resolve_barrier_params(p: BarrierParams, mean_slave_edge: float) -> BarrierParams:
    q = BarrierParams(**p.__dict__)
    if not mean_slave_edge > 0:
        raise ConfigError("barrier params: mean slave edge length must be positive")
    if not q.kappa_face > 0:
        raise ConfigError("barrier params: kappa_face must be positive")
    if q.kappa_edge < 0:
        q.kappa_edge = 1e-3 * q.kappa_face * mean_slave_edge
    if q.kappa_point < 0:
        q.kappa_point = 1e-3 * q.kappa_face * mean_slave_edge * mean_slave_edge
    if not (q.kappa_edge > 0 and q.kappa_point > 0):
        raise ConfigError("barrier params: per-type stiffnesses must be positive")
    if not q.eps_max > 0:
        raise ConfigError("barrier params: eps_max must be positive")
    if not (q.delta_face > 0) or q.delta_face > 1.0 / 3.0:
        raise ConfigError("barrier params: delta_face must lie in (0, 1/3]")
    if not (q.delta_edge > 0) or q.delta_edge > 0.5:
        raise ConfigError("barrier params: delta_edge must lie in (0, 1/2]")
    if q.detection_radius < 0:
        q.detection_radius = 10.0 * q.eps_max
    if not q.detection_radius > 0:
        raise ConfigError("barrier params: detection_radius must be positive")
    if not 1 <= q.quad_order_face <= 4:
        raise ConfigError("barrier params: quad_order_face must lie in 1..4")
    if not 1 <= q.quad_order_edge <= 5:
        raise ConfigError("barrier params: quad_order_edge must lie in 1..5")
    return q


@dataclass
class SlabScene:
    """Two stacked slabs: master indenter (body 0) and slave pad (body 1)."""

    rest: np.ndarray  # (3N,) float64
    meshes: list
    offsets: list
    slave: ContactSurface
    master: ContactSurface
    params: BarrierParams
    x_eval: np.ndarray = field(default=None)  # shifted + perturbed evaluation state
    dx: np.ndarray = field(default=None)  # step for the filter
    name: str = ""


def slab_scene(nb: int, nt: int, texture_amp: float = 0.0, texture_freq: float = 20.0,
               seed: int = 12345, shift: float = -1.5e-3, perturb: float = 1e-4,
               kappa_face: float = 1e6, eps_max: float = 1e-3) -> SlabScene:
    """SURVEY.md 8d slab(nb, nt, A, f, seed). C2 = slab(50, 40); C3 = slab(155, 124)."""
    bottom = make_block((1.0, 1.0, 0.1), (nb, nb, 1))
    top = make_block((1.0, 1.0, 0.1), (nt, nt, 1), (0.0, 0.0, 0.102))
    if texture_amp != 0.0:
        v = bottom.vertices.copy()
        topz = np.abs(v[:, 2] - 0.1) < 1e-12
        v[topz, 2] += texture_amp * np.sin(2 * np.pi * texture_freq * v[topz, 0]) * \
            np.sin(2 * np.pi * texture_freq * v[topz, 1])
        bottom = TetMesh(v, bottom.tets)
    off_top = bottom.vertices.shape[0]
    rest = np.concatenate([bottom.vertices.ravel(), top.vertices.ravel()]).astype(np.float64)
    sb = extract_boundary_surface(bottom)
    stp = extract_boundary_surface(top)
    zt = top.vertices[stp.vertex_map[stp.triangles], 2]
    down = np.nonzero(np.all(np.abs(zt - 0.102) < 1e-9, axis=1))[0]
    slave = make_contact_surface(stp, off_top, down)
    master = make_contact_surface(sb, 0)
    params = resolve_barrier_params(BarrierParams(kappa_face=kappa_face, eps_max=eps_max),
                                    mean_edge_length(slave, rest))
    rng = np.random.default_rng(seed)
    x = rest.copy().reshape(-1, 3)
    x[off_top:, 2] += shift
    x = x.ravel() + rng.uniform(-perturb, perturb, size=rest.size)
    dx = np.zeros_like(rest).reshape(-1, 3)
    dx[off_top:, 2] = -1e-3
    dx = dx.ravel() + rng.uniform(-perturb, perturb, size=rest.size)
    return SlabScene(rest, [bottom, top], [0, off_top], slave, master, params, x, dx,
                     name=f"slab({nb},{nt})" + (f"+tex({texture_amp},{texture_freq})" if texture_amp else ""))


# ---------------------------------------------------------------------------
# graded lattices (mesh_gen.hpp) and the Hertz indentation scene (C1)

def graded_axis(length: float, h_fine: float, n_fine: int, n_coarse: int) -> list:
    """mesh_gen.hpp:14-53: n_fine cells of width h_fine, then n_coarse cells
    growing geometrically (ratio by 200 bisection steps) so the last node is length."""
    if not (length > 0) or not (h_fine > 0) or n_fine < 1 or n_coarse < 0:
        raise ConfigError("graded_axis: non-positive length, width or cell count")
    fine_len = n_fine * h_fine
    rest = length - fine_len
    if n_coarse == 0:
        if abs(rest) > 1e-9 * length:
            raise ConfigError("graded_axis: fine cells do not fill the axis")
    elif rest < n_coarse * h_fine * (1.0 - 1e-12):
        raise ConfigError("graded_axis: remaining length too short for coarse cells")
    nodes = [i * h_fine for i in range(n_fine + 1)]
    if n_coarse > 0:
        def coarse_len(g):
            tot, h = 0.0, h_fine
            for _ in range(n_coarse):
                h *= g
                tot += h
            return tot
        lo, hi = 1.0, 2.0
        while coarse_len(hi) < rest:
            hi *= 2
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if coarse_len(mid) < rest:
                lo = mid
            else:
                hi = mid
        g = 0.5 * (lo + hi)
        h = h_fine
        for _ in range(n_coarse):
            h *= g
            nodes.append(nodes[-1] + h)
    nodes[-1] = length
    return nodes


def mirrored_axis(nodes: list) -> list:
    """mesh_gen.hpp:55-64."""
    length = nodes[-1]
    out = [length - nodes[len(nodes) - 1 - i] for i in range(len(nodes))]
    out[0] = 0.0
    out[-1] = length
    return out


_ODD = (False, True, True, False, False, True)


def make_lattice(n0: int, n1: int, n2: int, pos: np.ndarray) -> TetMesh:
    """mesh_gen.hpp:66-106. pos: (n2+1, n1+1, n0+1, 3) node positions [k, j, i]."""
    verts = np.ascontiguousarray(pos.reshape(-1, 3), np.float64)

    def vid(a, b, c):
        return (c * (n1 + 1) + b) * (n0 + 1) + a

    ck, cj, ci = np.meshgrid(np.arange(n2), np.arange(n1), np.arange(n0), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    tets = np.empty((ci.size, 6, 4), dtype=np.int64)
    for q, p in enumerate(_PERMS):
        at = [ci.copy(), cj.copy(), ck.copy()]
        tets[:, q, 0] = vid(*at)
        for s_ in range(3):
            at[p[s_]] = at[p[s_]] + 1
            tets[:, q, s_ + 1] = vid(*at)
        if _ODD[q]:
            tets[:, q, 2], tets[:, q, 3] = tets[:, q, 3].copy(), tets[:, q, 2].copy()
    tets = tets.reshape(-1, 4)
    vol = tet_signed_volume(verts, tets)
    bad = np.nonzero(~(vol > 0))[0]
    if bad.size:
        raise ValueError(f"make_lattice: mapped cell produced a non-positive tet (index {int(bad[0])})")
    return TetMesh(verts, tets.astype(np.int32))


def _square_to_disk(a: np.ndarray, b: np.ndarray):
    """mesh_gen.hpp:108-117 (elementwise)."""
    mx = np.maximum(a, b)
    with np.errstate(invalid="ignore", divide="ignore"):
        n = np.sqrt(a * a + b * b)
        f = mx / n
    x, y = a * f, b * f
    zero = mx <= 0
    return np.where(zero, 0.0, x), np.where(zero, 0.0, y)


def make_cylinder_sector(radius: float, height: float, radial_nodes, z_nodes) -> TetMesh:
    """mesh_gen.hpp:119-136: quarter cylinder x, y >= 0, z in [-height, 0]."""
    if len(radial_nodes) < 2 or len(z_nodes) < 2:
        raise ConfigError("make_cylinder_sector: node sequences need at least two entries")
    if not (radius > 0) or not (height > 0):
        raise ConfigError("make_cylinder_sector: radius and height must be positive")
    rn, zn = np.asarray(radial_nodes, np.float64), np.asarray(z_nodes, np.float64)
    nr, nz = rn.size - 1, zn.size - 1
    K, J, I = np.meshgrid(np.arange(nz + 1), np.arange(nr + 1), np.arange(nr + 1), indexing="ij")
    x, y = _square_to_disk(rn[I], rn[J])
    pos = np.stack([x, y, zn[K] - height], axis=-1)
    return make_lattice(nr, nr, nz, pos)


def make_sphere_octant(radius: float, tangential_nodes, radial_nodes) -> TetMesh:
    """mesh_gen.hpp:138-161: cube-to-ball map, pole at (0, 0, radius)."""
    if len(tangential_nodes) < 2 or len(radial_nodes) < 2:
        raise ConfigError("make_sphere_octant: node sequences need at least two entries")
    if not (radius > 0):
        raise ConfigError("make_sphere_octant: radius must be positive")
    if abs(tangential_nodes[-1] - 1.0) > 1e-12 or abs(radial_nodes[-1] - 1.0) > 1e-12:
        raise ConfigError("make_sphere_octant: node sequences must end at 1")
    tn, wn = np.asarray(tangential_nodes, np.float64), np.asarray(radial_nodes, np.float64)
    nt, nw = tn.size - 1, wn.size - 1
    K, J, I = np.meshgrid(np.arange(nw + 1), np.arange(nt + 1), np.arange(nt + 1), indexing="ij")
    px, py, pz = tn[I], tn[J], wn[K]
    mx = np.maximum(np.maximum(np.abs(px), np.abs(py)), np.abs(pz))
    with np.errstate(invalid="ignore", divide="ignore"):
        nrm = np.sqrt((px * px + py * py) + pz * pz)
        f = mx / nrm
    pos = np.stack([(px * f) * radius, (py * f) * radius, (pz * f) * radius], axis=-1)
    pos[mx <= 0] = 0.0
    return make_lattice(nt, nt, nw, pos)


@dataclass
class HertzConfig:
    """bench.hpp:157-176."""
    refine: float = 1.0
    load_steps: int = 10
    Q: float = 1e7
    R: float = 0.05
    E: float = 2.1e11
    nu: float = 0.3
    block_radius: float = 0.12
    block_height: float = 0.06
    initial_gap: float = 5e-5
    eps_max: float = 1e-5
    detection_radius: float = 6e-4
    slave_patch_radius: float = 0.02
    kappa_face: float = -1.0


@dataclass
class HertzOracle:
    """bench.hpp:134-155: Hertz contact of a sphere on a half space."""
    Q: float
    R: float
    E_star: float
    alpha_H: float
    p0: float

    def pressure(self, r):
        r = np.asarray(r, np.float64)
        return np.where(r >= self.alpha_H, 0.0,
                        self.p0 * np.sqrt(np.maximum(1 - r * r / (self.alpha_H * self.alpha_H), 0.0)))


def make_hertz_oracle(Q: float, R: float, E: float, nu: float) -> HertzOracle:
    E_star = E / (2 * (1 - nu * nu))
    alpha_H = math.cbrt(3.0 * Q * math.pi * R * R * R / (4.0 * E_star))  # glibc cbrt, as std::cbrt
    p0 = 3.0 * Q * R * R / (2.0 * alpha_H * alpha_H)
    return HertzOracle(Q, R, E_star, alpha_H, p0)


def _n_scaled(base: int, refine: float) -> int:
    v = base * refine  # std::lround: half away from zero
    return max(1, int(np.floor(v + 0.5)) if v >= 0 else -int(np.floor(-v + 0.5)))


def make_hertz_block(c: HertzConfig) -> TetMesh:
    """bench.hpp:178-183."""
    n = lambda b: _n_scaled(b, c.refine)  # noqa: E731
    return make_cylinder_sector(c.block_radius, c.block_height,
                                graded_axis(c.block_radius, 0.0006 / c.refine, n(6), n(6)),
                                mirrored_axis(graded_axis(c.block_height, 0.0007 / c.refine, n(4), n(5))))


def make_hertz_ball(c: HertzConfig) -> TetMesh:
    """bench.hpp:185-193: sphere octant, pole rotated downward, flat top seated above the block."""
    n = lambda b: _n_scaled(b, c.refine)  # noqa: E731
    ball = make_sphere_octant(c.R, graded_axis(1.0, 0.0055 / c.refine, n(12), n(3)),
                              mirrored_axis(graded_axis(1.0, 0.02 / c.refine, n(3), n(3))))
    lift = c.R + c.initial_gap
    v = ball.vertices
    nv = np.stack([v[:, 1], v[:, 0], -v[:, 2] + lift], axis=1)
    return TetMesh(nv, orient_tets_positive(nv, ball.tets).astype(np.int32))


def add_pressure_forces(faces: np.ndarray, rest: np.ndarray, magnitude: float, direction, f: np.ndarray):
    """elasticity.hpp:147-160: magnitude * area / 3 per face vertex along
    direction (default: inward normal -cr.normalized()), faces in order, in the
    reference's scalar op order (bitwise the reference's f_ext)."""
    x3 = rest.reshape(-1, 3)
    for tri in np.asarray(faces).tolist():
        a, b, c = x3[tri[0]].tolist(), x3[tri[1]].tolist(), x3[tri[2]].tolist()
        u = (b[0] - a[0], b[1] - a[1], b[2] - a[2])
        v = (c[0] - a[0], c[1] - a[1], c[2] - a[2])
        cr = (u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0])
        sq = (cr[0] * cr[0] + cr[1] * cr[1]) + cr[2] * cr[2]
        area = 0.5 * math.sqrt(sq)
        if direction is not None:
            d = tuple(float(t) for t in direction)
        else:
            nrm = math.sqrt(sq)
            d = (-(cr[0] / nrm), -(cr[1] / nrm), -(cr[2] / nrm)) if sq > 0 else (-cr[0], -cr[1], -cr[2])
        s_ = magnitude * area / 3.0
        for i in range(3):
            g = 3 * tri[i]
            f[g] += s_ * d[0]
            f[g + 1] += s_ * d[1]
            f[g + 2] += s_ * d[2]


@dataclass
class HertzScene:
    """C1: everything run_hertz sets up before System::solve (bench.hpp:210-272)."""
    cfg: HertzConfig
    oracle: HertzOracle
    block: TetMesh
    ball: TetMesh
    rest: np.ndarray           # (3N,) block then ball
    ball_offset: int
    fixed: np.ndarray          # (F, 2) int64: vertex, axis
    fixed_target: np.ndarray   # (F,)
    f_ext: np.ndarray          # (3N,)
    applied_force: float
    slave_tris: np.ndarray     # block boundary triangle indices (slave patch)
    slave: ContactSurface
    master: ContactSurface
    params: BarrierParams      # resolved


def hertz_scene(cfg: HertzConfig | None = None, ball_shift=(0.0, 0.0)) -> HertzScene:
    """Hertz indentation scene (C1 at refine 0.7). ball_shift moves the ball in
    x/y (C5's per-scene indenter offset; (0, 0) is the reference scene)."""
    cfg = cfg or HertzConfig()
    oracle = make_hertz_oracle(cfg.Q, cfg.R, cfg.E, cfg.nu)
    block, ball = make_hertz_block(cfg), make_hertz_ball(cfg)
    for name, cnt in (("block", block.tets.shape[0]), ("ball", ball.tets.shape[0])):
        if cnt < 1000:
            raise ConfigError(f"refine {cfg.refine} produces only {cnt} tets for the {name}; need >= 1000")
    ball0 = ball  # symmetry-plane selection uses the unshifted ball
    if ball_shift[0] != 0.0 or ball_shift[1] != 0.0:
        v = ball.vertices.copy()
        v[:, 0] += ball_shift[0]
        v[:, 1] += ball_shift[1]
        ball = TetMesh(v, ball.tets)
    nb = block.vertices.shape[0]
    rest = np.concatenate([block.vertices.ravel(), ball.vertices.ravel()]).astype(np.float64)
    fixed, target = [], []
    for v, p in enumerate(block.vertices):
        if abs(p[2] + cfg.block_height) < 1e-9:
            fixed.append((v, 2)); target.append(p[2])
        if abs(p[0]) < 1e-12:
            fixed.append((v, 0)); target.append(0.0)
        if abs(p[1]) < 1e-12:
            fixed.append((v, 1)); target.append(0.0)
    for v, p in enumerate(ball0.vertices):
        if abs(p[0]) < 1e-12:
            fixed.append((nb + v, 0)); target.append(ball.vertices[v, 0])
        if abs(p[1]) < 1e-12:
            fixed.append((nb + v, 1)); target.append(ball.vertices[v, 1])
    sb, sh = extract_boundary_surface(block), extract_boundary_surface(ball)
    lift = cfg.R + cfg.initial_gap
    lz = ball.vertices[sh.vertex_map[sh.triangles], 2]
    top = nb + sh.vertex_map[sh.triangles[np.all(np.abs(lz - lift) <= 1e-9, axis=1)]]
    f_ext = np.zeros_like(rest)
    add_pressure_forces(top, rest, cfg.Q, (0, 0, -1), f_ext)
    applied = 0.0
    for v in range(rest.size // 3):
        applied -= f_ext[3 * v + 2]
    bp = block.vertices[sb.vertex_map[sb.triangles]]
    inside = np.all((np.abs(bp[:, :, 2]) <= 1e-9) & (np.hypot(bp[:, :, 0], bp[:, :, 1]) <= cfg.slave_patch_radius),
                    axis=1)
    slave_tris = np.nonzero(inside)[0]
    slave = make_contact_surface(sb, 0, slave_tris)
    master = make_contact_surface(sh, nb)
    kf = cfg.kappa_face if cfg.kappa_face > 0 else oracle.p0 / (cfg.eps_max * (math.log(2.0) + 0.5))
    params = resolve_barrier_params(BarrierParams(kappa_face=kf, eps_max=cfg.eps_max,
                                                  detection_radius=cfg.detection_radius),
                                    mean_edge_length(slave, rest))
    return HertzScene(cfg, oracle, block, ball, rest, nb, np.asarray(fixed, np.int64).reshape(-1, 2),
                      np.asarray(target, np.float64), f_ext, applied, slave_tris, slave, master, params)


# ---------------------------------------------------------------------------
# C5: batched independent scenes packed into one SoA

def concat_surfaces(surfs, vertex_offsets) -> ContactSurface:
    """Packs contact surfaces of disjoint scenes: vertex ids shift by the
    scene's vertex offset, edge ids by the edges before it. Equals
    make_contact_surface over the concatenated triangle list (edges are
    numbered by first appearance, verts ascending)."""
    tris, edges, tedges, verts = [], [], [], []
    e_off = 0
    for s_, off in zip(surfs, vertex_offsets):
        tris.append(s_.tris.astype(np.int64) + off)
        edges.append(s_.edges.astype(np.int64) + off)
        tedges.append(s_.tri_edges.astype(np.int64) + e_off)
        verts.append(s_.verts.astype(np.int64) + off)
        e_off += s_.edges.shape[0]
    cat = lambda a, w: np.concatenate(a).astype(np.int32) if a else np.zeros((0, w), np.int32)  # noqa: E731
    return ContactSurface(cat(tris, 3), cat(edges, 2), cat(tedges, 3),
                          np.concatenate(verts).astype(np.int32) if verts else np.zeros(0, np.int32))


@dataclass
class SceneBatch:
    """n_scenes Hertz scenes packed into one system (C5 = 1024 x C1)."""
    scenes: np.ndarray        # global scene ids held by this batch
    rest: np.ndarray          # (3N,)
    x_eval: np.ndarray        # shifted + perturbed evaluation state (active contact)
    dx: np.ndarray
    vscene: np.ndarray        # (N,) int32 local scene index per vertex
    v_off: np.ndarray         # (S+1,) vertex offsets
    slave: ContactSurface
    master: ContactSurface
    params: BarrierParams
    shifts: np.ndarray        # (S, 2) indenter x/y offsets
    q_scale: np.ndarray       # (S,) load scale (Newton workload; not used by assembly)
    base: HertzScene


def c5_batch(n_scenes: int = 1024, first: int = 0, count: int | None = None, refine: float = 0.7,
             seed: int = 20260518, perturb: float = 1e-7) -> SceneBatch:
    """Scenes first .. first+count-1 of the C5 job (1024 x C1 at refine 0.7).
    Scene s: the C1 geometry with the indenter offset by |U(-2e-3, 2e-3)| in x/y and
    its load scaled by U(0.5, 1.5), both from default_rng(seed + s). Sampling
    happens at rest; the evaluation state lowers each indenter so its pole gap
    is eps_max / 2 and adds a seeded +-perturb to every coordinate."""
    count = n_scenes - first if count is None else count
    base = hertz_scene(HertzConfig(refine=refine))
    nb = base.ball_offset
    N = base.rest.size // 3
    ids = np.arange(first, first + count)
    shifts = np.zeros((count, 2))
    qs = np.zeros(count)
    for k, s_ in enumerate(ids):
        rng = np.random.default_rng(seed + int(s_))
        # the quarter models' symmetry planes sit at x = 0 / y = 0: the offset is
        # kept inside the quadrant (|U(-2e-3, 2e-3)|) so the pole stays on the block
        shifts[k] = np.abs(rng.uniform(-2e-3, 2e-3, size=2))
        qs[k] = rng.uniform(0.5, 1.5)
    r3 = np.tile(base.rest.reshape(1, N, 3), (count, 1, 1))
    r3[:, nb:, 0] += shifts[:, 0:1]
    r3[:, nb:, 1] += shifts[:, 1:2]
    rest = r3.reshape(-1)
    v_off = np.arange(count + 1, dtype=np.int64) * N
    slave = concat_surfaces([base.slave] * count, v_off[:-1])
    master = concat_surfaces([base.master] * count, v_off[:-1])
    drop = base.cfg.initial_gap - 0.5 * base.cfg.eps_max
    x = r3.copy()
    x[:, nb:, 2] -= drop
    rng = np.random.default_rng(seed - 1)
    x = x.reshape(-1) + rng.uniform(-perturb, perturb, size=rest.size)
    dx = np.zeros_like(r3)
    dx[:, nb:, 2] = -0.5 * base.cfg.eps_max
    dx = dx.reshape(-1) + rng.uniform(-perturb, perturb, size=rest.size)
    vscene = np.repeat(np.arange(count, dtype=np.int32), N)
    return SceneBatch(ids, rest, x, dx, vscene, v_off, slave, master, base.params, shifts, qs, base)
