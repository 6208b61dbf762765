"""Dual-mesh embedding on the device -- embedding.hpp:14-106:
a detailed visual surface bound to the simulated host surface once
(embed_in_surface: nearest host triangle by LBVH branch and bound, lowest
index on ties, unclamped plane barycentrics and a signed normal offset), then
reconstructed every frame from the deformed host (apply_embedding). Same
names, arguments and errors (MeshError naming the triangle) as the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import gmcp as _g


@dataclass
class SurfaceEmbedding:
    """VertexEmbedding per point (embedding.hpp:14-20), as arrays."""
    tri: np.ndarray     # (n,) int32 host triangle
    bary: np.ndarray    # (n, 3) plane barycentrics, unclamped
    offset: np.ndarray  # (n,) signed distance along the host triangle normal

    def __len__(self):
        return int(self.tri.size)


def _ctx(ctx):
    return ctx if ctx is not None else _g.Context(0)


def embed_in_surface(points, host_vertices, host_triangles, use_tree: bool = True, ctx=None) -> SurfaceEmbedding:
    """embedding.hpp:26-84. use_tree is accepted for API parity: the device
    search returns the same binding as both of the reference's paths."""
    c = _ctx(ctx)
    P = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    V = np.ascontiguousarray(host_vertices, np.float64).reshape(-1, 3)
    T = np.ascontiguousarray(host_triangles, np.int32).reshape(-1, 3)
    n = P.shape[0]
    tri, bary, off = np.zeros(n, np.int32), np.zeros((n, 3)), np.zeros(n)
    bad = C.c_int64(-1)
    rc = c.L.gmcp_embed_in_surface(c.h, _g._p(P), C.c_int64(n), _g._p(V), C.c_int64(V.shape[0]), _g._p(T),
                                   C.c_int64(T.shape[0]), _g._p(tri), _g._p(bary), _g._p(off), C.byref(bad))
    _g._check(rc, bad.value)
    return SurfaceEmbedding(tri, bary, off)


def apply_embedding(emb: SurfaceEmbedding, host_triangles, host_positions, ctx=None) -> np.ndarray:
    """embedding.hpp:87-106 -> (n, 3) reconstructed positions."""
    c = _ctx(ctx)
    T = np.ascontiguousarray(host_triangles, np.int32).reshape(-1, 3)
    X = np.ascontiguousarray(host_positions, np.float64).reshape(-1, 3)
    tri = np.ascontiguousarray(emb.tri, np.int32)
    bary = np.ascontiguousarray(emb.bary, np.float64)
    off = np.ascontiguousarray(emb.offset, np.float64)
    out = np.zeros((tri.size, 3))
    bad = C.c_int64(-1)
    rc = c.L.gmcp_apply_embedding(c.h, _g._p(tri), _g._p(bary), _g._p(off), C.c_int64(tri.size), _g._p(T),
                                  C.c_int64(T.shape[0]), _g._p(X), C.c_int64(X.shape[0]), _g._p(out), C.byref(bad))
    _g._check(rc, bad.value)
    return out
