"""Host-side mirror of the reference's contact API over the B200 C-ABI.

The reference (proj/include/gmcp/, header-only C++) exposes free functions
over ContactSurface / ContactState / BarrierParams / VecX. This module keeps
those names, argument meanings and error behaviour, and routes every call
through libgmcp_b200.so (include/gmcp_b200.h) -- hand-written sm_100a CUDA.
There is no CPU fallback: if the library or a CUDA device is missing, calls
raise GmcpCudaError.

    reference (file:line)                              here
    build_candidate_pairs  contact_sampling.hpp:281    build_candidate_pairs
    build_contact_state    contact_sampling.hpp:382    build_contact_state
    try_contact_energy     contact_energy.hpp:95       try_contact_energy
    contact_energy         contact_energy.hpp:110      contact_energy
    add_contact_gradient   contact_energy.hpp:126      add_contact_gradient
    add_contact_gradient_hessian  contact_energy.hpp:146  add_contact_gradient_hessian
    step_filter            contact_energy.hpp:184      step_filter
    displacement_cap       contact_energy.hpp:198      displacement_cap
    contact_pressure_field contact_energy.hpp:225      contact_pressure_field
    contact_force_summary  contact_energy.hpp:253      contact_force_summary
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import scenes as _scenes

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GMCP_B200_LIB") or os.path.join(HERE, "libgmcp_b200.so")  # env: dev variants

GMCP_OK, GMCP_ERR_INFEASIBLE, GMCP_ERR_DEGENERATE, GMCP_ERR_CONFIG, GMCP_ERR_SOLVER, GMCP_ERR_CUDA, \
    GMCP_ERR_ARG, GMCP_ERR_PARSE = range(8)
POINT, EDGE, FACE = 0, 1, 2


# ---- reference exception hierarchy (core.hpp:25-56) -------------------------
class Error(RuntimeError):
    pass


class MeshError(Error):
    pass


class ConfigError(Error):
    pass


class ParseError(Error):
    pass


class SolverError(Error):
    def __init__(self, msg, residual=float("nan")):
        super().__init__(msg)
        self.residual = residual


class InfeasibleGapError(Error):
    def __init__(self, msg, sample_id):
        super().__init__(msg)
        self.sample_id = sample_id


class GmcpCudaError(Error):
    pass


_EXC = {GMCP_ERR_INFEASIBLE: InfeasibleGapError, GMCP_ERR_DEGENERATE: MeshError, GMCP_ERR_CONFIG: ConfigError,
        GMCP_ERR_SOLVER: SolverError, GMCP_ERR_CUDA: GmcpCudaError, GMCP_ERR_ARG: Error, GMCP_ERR_PARSE: ParseError}


# ---- ABI structs ---------------------------------------------------------------
class _Surface(C.Structure):
    _fields_ = [("n_tris", C.c_int32), ("tris", C.c_void_p), ("n_edges", C.c_int32), ("edges", C.c_void_p),
                ("tri_edges", C.c_void_p), ("n_verts", C.c_int32), ("verts", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("kappa_face", C.c_double), ("kappa_edge", C.c_double), ("kappa_point", C.c_double),
                ("eps_max", C.c_double), ("delta_face", C.c_double), ("delta_edge", C.c_double),
                ("detection_radius", C.c_double), ("quad_order_face", C.c_int32), ("quad_order_edge", C.c_int32)]


class _Samples(C.Structure):
    _fields_ = [("n", C.c_int64)] + [(k, C.c_void_p) for k in
                                      ("type", "slave", "master", "beta_s", "beta_m", "eta", "weight", "gamma",
                                       "eps", "g_ref")]


SAMPLE_FIELDS = (("type", np.int8, 1), ("slave", np.int32, 3), ("master", np.int32, 3), ("beta_s", np.float64, 3),
                 ("beta_m", np.float64, 3), ("eta", np.float64, 1), ("weight", np.float64, 1),
                 ("gamma", np.float64, 1), ("eps", np.float64, 1), ("g_ref", np.float64, 1))
PRESSURE_DTYPE = np.dtype([("sample", np.int64), ("position", np.float64, 3), ("radius", np.float64),
                           ("gap", np.float64), ("pressure", np.float64)])

_lib = None


def library() -> C.CDLL:
    """Loads libgmcp_b200.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GmcpCudaError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; "
                                f"g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.gmcp_last_error.restype = C.c_char_p
        L.gmcp_num_samples.restype = C.c_int64
        L.gmcp_launch_count.restype = C.c_int64
        L.gmcp_positions_device.restype = C.c_void_p
        L.gmcp_step_device.restype = C.c_void_p
        L.gmcp_ctx_destroy.restype = None
        L.gmcp_ctx_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _check(rc, bad=-1):
    if rc != GMCP_OK:
        msg = library().gmcp_last_error().decode()
        exc = _EXC.get(rc, Error)
        if exc is InfeasibleGapError:
            raise InfeasibleGapError(msg, bad)
        raise exc(msg)


def _params(p) -> _Params:
    return _Params(p.kappa_face, p.kappa_edge, p.kappa_point, p.eps_max, p.delta_face, p.delta_edge,
                   p.detection_radius, p.quad_order_face, p.quad_order_edge)


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


class Context:
    """One gmcp_ctx: device copies of surfaces, x, dx, samples and the BCSR."""

    def __init__(self, device: int = 0):
        self.L = library()
        h = C.c_void_p()
        _check(self.L.gmcp_ctx_create(C.c_int(device), C.byref(h)))
        self.h = h
        self.n_dof = 0
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            self.L.gmcp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self.L.gmcp_launch_count(self.h))

    # -- inputs --------------------------------------------------------------
    def set_params(self, p):
        cp = _params(p)
        _check(self.L.gmcp_set_params(self.h, C.byref(cp)))
        self.params = p

    def set_surfaces(self, slave, master):
        arrs, structs = [], []
        for s in (slave, master):
            a = [np.ascontiguousarray(v, dtype=np.int32) for v in (s.tris, s.edges, s.tri_edges, s.verts)]
            arrs += a
            structs.append(_Surface(a[0].shape[0], a[0].ctypes.data, a[1].shape[0], a[1].ctypes.data,
                                    a[2].ctypes.data, a[3].shape[0], a[3].ctypes.data))
        _check(self.L.gmcp_set_surfaces(self.h, C.byref(structs[0]), C.byref(structs[1])))
        self.slave, self.master = slave, master

    def set_positions(self, x):
        x = _f64(x)
        _check(self.L.gmcp_set_positions(self.h, _p(x), C.c_int64(x.size)))
        self.n_dof = x.size

    def set_vertex_scenes(self, scene):
        """Batched independent scenes (C5): scene id per vertex, or None."""
        if scene is None:
            _check(self.L.gmcp_set_vertex_scenes(self.h, None, C.c_int64(0)))
            return
        sc = np.ascontiguousarray(scene, np.int32)
        _check(self.L.gmcp_set_vertex_scenes(self.h, _p(sc), C.c_int64(sc.size)))

    def set_step(self, dx):
        dx = _f64(dx)
        _check(self.L.gmcp_set_step(self.h, _p(dx), C.c_int64(dx.size)))

    def upload_samples(self, s: dict):
        arrs = {k: np.ascontiguousarray(s[k], dtype=dt) for k, dt, _ in SAMPLE_FIELDS}
        cs = _Samples(arrs["type"].shape[0], *[arrs[k].ctypes.data for k, _, _ in SAMPLE_FIELDS])
        _check(self.L.gmcp_upload_samples(self.h, C.byref(cs)))

    def num_samples(self) -> int:
        return int(self.L.gmcp_num_samples(self.h))

    def download_samples(self) -> dict:
        n = self.num_samples()
        out = {k: np.zeros((n, w) if w > 1 else n, dtype=dt) for k, dt, w in SAMPLE_FIELDS}
        cs = _Samples(n, *[out[k].ctypes.data for k, _, _ in SAMPLE_FIELDS])
        _check(self.L.gmcp_download_samples(self.h, C.byref(cs)))
        return out

    # -- broadphase / sampler --------------------------------------------------
    def broadphase(self, r: float):
        counts = np.zeros(3, np.int64)
        _check(self.L.gmcp_broadphase(self.h, C.c_double(r), _p(counts)))
        return counts

    def download_pairs(self) -> dict:
        nst = self.slave.tris.shape[0]
        out = {}
        for which, name in enumerate(("tris", "edges", "verts")):
            off = np.zeros(nst + 1, np.int64)
            _check(self.L.gmcp_download_pairs(self.h, C.c_int(which), _p(off), None))
            ids = np.zeros(max(int(off[-1]), 1), np.int32)
            _check(self.L.gmcp_download_pairs(self.h, C.c_int(which), _p(off), _p(ids)))
            out[name] = (off, ids[:int(off[-1])])
        return out

    def upload_pairs(self, pairs: dict):
        a = []
        for name in ("tris", "edges", "verts"):
            a += [np.ascontiguousarray(pairs[name][0], np.int64), np.ascontiguousarray(pairs[name][1], np.int32)]
        _check(self.L.gmcp_upload_pairs(self.h, *[_p(v) for v in a]))

    def build_samples(self, eps_reference=None) -> int:
        n = C.c_int64()
        er = None if eps_reference is None else _f64(eps_reference)
        _check(self.L.gmcp_build_samples(self.h, _p(er), C.byref(n)))
        return n.value

    # -- per iteration ------------------------------------------------------------
    def try_energy(self):
        e, mg, f = C.c_double(), C.c_double(), C.c_int32()
        _check(self.L.gmcp_try_energy(self.h, C.byref(e), C.byref(mg), C.byref(f)))
        return e.value, mg.value, bool(f.value)

    def energy(self):
        e, bad = C.c_double(), C.c_int64(-1)
        rc = self.L.gmcp_energy(self.h, C.byref(e), C.byref(bad))
        _check(rc, bad.value)
        return e.value

    def gradient(self, grad=None, hessian=False):
        e, bad = C.c_double(), C.c_int64(-1)
        g = None if grad is None else grad
        fn = self.L.gmcp_gradient_hessian if hessian else self.L.gmcp_gradient
        rc = fn(self.h, _p(g), C.byref(e), C.byref(bad))
        _check(rc, bad.value)
        return e.value

    def add_gradient(self, x, grad=None, hessian=False):
        """One C-ABI call: positions x, accumulate into grad (host), energy back
        (gmcp_add_gradient[_hessian]; transfers overlap the assembly)."""
        x = _f64(x)
        e, bad = C.c_double(), C.c_int64(-1)
        fn = self.L.gmcp_add_gradient_hessian if hessian else self.L.gmcp_add_gradient
        rc = fn(self.h, _p(x), C.c_int64(x.size), _p(grad), C.byref(e), C.byref(bad))
        _check(rc, bad.value)
        self.n_dof = x.size
        return e.value

    def download_hessian(self, out=None):
        """The assembled Gauss-Newton Hessian as BCSR (rowptr, cols, vals[nnzb,3,3]).
        out: optional caller arrays (e.g. pinned host memory) of sufficient size."""
        nnzb = C.c_int64()
        _check(self.L.gmcp_download_hessian(self.h, C.byref(nnzb), None, None, None))
        if out is not None:
            rowptr, cols, vals = out
            assert rowptr.size >= self.n_dof // 3 + 1 and cols.size >= nnzb.value and vals.shape[0] >= nnzb.value
        else:
            rowptr = np.zeros(self.n_dof // 3 + 1, np.int32)
            cols = np.zeros(max(nnzb.value, 1), np.int32)
            vals = np.zeros((max(nnzb.value, 1), 3, 3))
        _check(self.L.gmcp_download_hessian(self.h, C.byref(nnzb), _p(rowptr), _p(cols), _p(vals)))
        return rowptr, cols[:nnzb.value], vals[:nnzb.value]

    def step_filter(self) -> float:
        a = C.c_double()
        _check(self.L.gmcp_step_filter(self.h, C.byref(a)))
        return a.value

    def displacement_cap(self) -> float:
        a = C.c_double()
        _check(self.L.gmcp_displacement_cap(self.h, C.byref(a)))
        return a.value

    def pressure_field(self):
        n = C.c_int64()
        _check(self.L.gmcp_pressure_field(self.h, C.byref(n), None))
        out = np.zeros(n.value, PRESSURE_DTYPE)
        if n.value:
            _check(self.L.gmcp_pressure_field(self.h, C.byref(n), _p(out)))
        return out

    def force_summary(self):
        out = np.zeros(12)
        _check(self.L.gmcp_force_summary(self.h, _p(out)))
        return out.reshape(4, 3)

    def kinematics(self):
        n = self.num_samples()
        g, nv = np.zeros(n), np.zeros(n, np.int32)
        ids, dg = np.zeros((n, 6), np.int32), np.zeros((n, 6, 3))
        _check(self.L.gmcp_kinematics(self.h, _p(g), _p(nv), _p(ids), _p(dg)))
        return g, nv, ids, dg

    def time_assembly(self, reps=10, flush_l2=True):
        a, b = C.c_double(), C.c_double()
        _check(self.L.gmcp_time_assembly(self.h, C.c_int(reps), C.c_int(int(flush_l2)), C.byref(a), C.byref(b)))
        return a.value, b.value


# ---------------------------------------------------------------------------
# reference-shaped free functions (drop-in for the contact path)

@dataclass
class ContactPairSet:
    """contact_sampling.hpp:267-279, CSR per slave triangle."""

    tris: tuple
    edges: tuple
    verts: tuple

    def total_candidates(self) -> int:
        return int(self.tris[0][-1] + self.edges[0][-1] + self.verts[0][-1])

    def as_dict(self):
        return {"tris": self.tris, "edges": self.edges, "verts": self.verts}


class ContactState:
    """Device-resident frozen sample set (contact_sampling.hpp:343-346)."""

    def __init__(self, ctx: Context, params, reference_positions):
        self.ctx = ctx
        self.params = params
        self.reference_positions = np.array(reference_positions, dtype=np.float64)

    @property
    def samples(self) -> dict:
        return self.ctx.download_samples()

    def __len__(self):
        return self.ctx.num_samples()


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def build_candidate_pairs(slave, master, x, detection_radius, ctx: Context | None = None) -> ContactPairSet:
    ctx = ctx or default_context()
    ctx.set_surfaces(slave, master)
    ctx.set_positions(x)
    ctx.broadphase(detection_radius)
    d = ctx.download_pairs()
    return ContactPairSet(d["tris"], d["edges"], d["verts"])


def build_contact_state(slave, master, pairs: ContactPairSet, x, params, eps_reference=None,
                        ctx: Context | None = None) -> ContactState:
    ctx = ctx or Context(0)
    ctx.set_surfaces(slave, master)
    ctx.set_params(params)
    ctx.set_positions(x)
    ctx.upload_pairs(pairs.as_dict())
    ctx.build_samples(eps_reference)
    return ContactState(ctx, params, x)


def state_from_samples(samples: dict, params, reference_positions, ctx: Context | None = None) -> ContactState:
    ctx = ctx or Context(0)
    ctx.set_params(params)
    ctx.set_positions(reference_positions)
    ctx.upload_samples(samples)
    return ContactState(ctx, params, reference_positions)


def try_contact_energy(state: ContactState, params, x):
    """Returns (feasible, energy, min_gap) like ContactEnergyResult."""
    state.ctx.set_positions(x)
    e, mg, feas = state.ctx.try_energy()
    return feas, e, mg


def contact_energy(state: ContactState, params, x) -> float:
    state.ctx.set_positions(x)
    return state.ctx.energy()


def add_contact_gradient(state: ContactState, params, x, grad: np.ndarray) -> float:
    return state.ctx.add_gradient(x, grad, hessian=False)


def add_contact_gradient_hessian(state: ContactState, params, x, grad: np.ndarray):
    """Returns (energy, (rowptr, cols, vals)) -- the Gauss-Newton Hessian as BCSR."""
    e = state.ctx.add_gradient(x, grad, hessian=True)
    return e, state.ctx.download_hessian()


def step_filter(state: ContactState, x, dx) -> float:
    state.ctx.set_positions(x)
    state.ctx.set_step(dx)
    return state.ctx.step_filter()


def displacement_cap(state: ContactState, params, x, dx) -> float:
    state.ctx.set_positions(x)
    state.ctx.set_step(dx)
    return state.ctx.displacement_cap()


def contact_pressure_field(state: ContactState, params, x):
    state.ctx.set_positions(x)
    return state.ctx.pressure_field()


def contact_force_summary(state: ContactState, params, x):
    state.ctx.set_positions(x)
    return state.ctx.force_summary()


resolve_barrier_params = _scenes.resolve_barrier_params
mean_edge_length = _scenes.mean_edge_length
