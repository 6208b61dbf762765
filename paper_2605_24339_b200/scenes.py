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
"""
from __future__ import annotations

from dataclasses import dataclass, field

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
