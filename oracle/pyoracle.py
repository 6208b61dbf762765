"""ctypes binding of the CPU oracle API (oracle/gmcp_oracle_api.h).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product.

    Oracle("restated")   -> oracle/libgmcp_oracle.so  (C restatement)
    Oracle("reference")  -> oracle/_ref/libgmcp_ref.so (reference headers + shim)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restated": os.path.join(HERE, "libgmcp_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "libgmcp_ref.so"),
}

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class CSurface(C.Structure):
    _fields_ = [("n_tris", C.c_int32), ("tris", C.c_void_p), ("n_edges", C.c_int32),
                ("edges", C.c_void_p), ("tri_edges", C.c_void_p), ("n_verts", C.c_int32),
                ("verts", C.c_void_p)]


class CParams(C.Structure):
    _fields_ = [("kappa_face", C.c_double), ("kappa_edge", C.c_double),
                ("kappa_point", C.c_double), ("eps_max", C.c_double),
                ("delta_face", C.c_double), ("delta_edge", C.c_double),
                ("detection_radius", C.c_double), ("quad_order_face", C.c_int32),
                ("quad_order_edge", C.c_int32)]


class CSamples(C.Structure):
    _fields_ = [("n", C.c_int64), ("type", C.c_void_p), ("slave", C.c_void_p),
                ("master", C.c_void_p), ("beta_s", C.c_void_p), ("beta_m", C.c_void_p),
                ("eta", C.c_void_p), ("weight", C.c_void_p), ("gamma", C.c_void_p),
                ("eps", C.c_void_p), ("g_ref", C.c_void_p)]


class CPressure(C.Structure):
    _fields_ = [("sample", C.c_int64), ("position", C.c_double * 3), ("radius", C.c_double),
                ("gap", C.c_double), ("pressure", C.c_double)]


PRESSURE_DTYPE = np.dtype([("sample", np.int64), ("position", np.float64, 3),
                           ("radius", np.float64), ("gap", np.float64),
                           ("pressure", np.float64)])

SAMPLE_FIELDS = (("type", np.int8, 1), ("slave", np.int32, 3), ("master", np.int32, 3),
                 ("beta_s", np.float64, 3), ("beta_m", np.float64, 3), ("eta", np.float64, 1),
                 ("weight", np.float64, 1), ("gamma", np.float64, 1), ("eps", np.float64, 1),
                 ("g_ref", np.float64, 1))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str, bad: int = -1):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.bad = bad


def empty_samples(n: int) -> dict:
    return {name: np.zeros((n, k) if k > 1 else n, dtype=dt) for name, dt, k in SAMPLE_FIELDS}


def samples_struct(s: dict):
    """Returns (CSamples, keepalive) over a dict of contiguous numpy arrays."""
    arrs = {k: np.ascontiguousarray(v) for k, v in s.items()}
    n = arrs["type"].shape[0]
    cs = CSamples(n, *[arrs[name].ctypes.data for name, _, _ in SAMPLE_FIELDS])
    return cs, arrs


def surface_struct(surf):
    arrs = [np.ascontiguousarray(a, dtype=np.int32) for a in (surf.tris, surf.edges, surf.tri_edges, surf.verts)]
    cs = CSurface(arrs[0].shape[0], arrs[0].ctypes.data, arrs[1].shape[0], arrs[1].ctypes.data,
                  arrs[2].ctypes.data, arrs[3].shape[0], arrs[3].ctypes.data)
    return cs, arrs


def params_struct(p) -> CParams:
    return CParams(p.kappa_face, p.kappa_edge, p.kappa_point, p.eps_max, p.delta_face,
                   p.delta_edge, p.detection_radius, p.quad_order_face, p.quad_order_edge)


class Oracle:
    def __init__(self, kind: str = "restated"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run `make -C oracle`)")
        self.kind = kind
        self.lib = L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_pairs_size.restype = C.c_int64
        L.orc_pairs_slave_tris.restype = C.c_int32
        L.orc_state_size.restype = C.c_int64
        for name in ("orc_pairs_free", "orc_state_free", "orc_pairs_copy", "orc_state_copy"):
            getattr(L, name).restype = None

    # -- helpers ---------------------------------------------------------
    def _check(self, rc: int, bad: int = -1):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode(), bad)

    def is_reference(self) -> bool:
        return bool(self.lib.orc_is_reference())

    def resolve_params(self, p, mean_edge: float):
        cp = params_struct(p)
        self._check(self.lib.orc_resolve_barrier_params(C.byref(cp), C.c_double(mean_edge)))
        return cp

    def barrier(self, g: float, eps: float):
        out = np.zeros(3)
        self._check(self.lib.orc_barrier(C.c_double(g), C.c_double(eps), out.ctypes.data_as(C.c_void_p)))
        return out

    # -- dual-mesh embedding (embedding.hpp) -----------------------------
    def embed_in_surface(self, points, host_v, host_t, use_tree=True):
        P = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        V = np.ascontiguousarray(host_v, np.float64).reshape(-1, 3)
        T = np.ascontiguousarray(host_t, np.int32).reshape(-1, 3)
        n = P.shape[0]
        tri, bary, off = np.zeros(n, np.int32), np.zeros((n, 3)), np.zeros(n)
        bad = C.c_int64(-1)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        rc = self.lib.orc_embed_in_surface(p(P), C.c_int64(n), p(V), C.c_int64(V.shape[0]), p(T),
                                           C.c_int64(T.shape[0]), C.c_int32(int(use_tree)), p(tri), p(bary),
                                           p(off), C.byref(bad))
        self._check(rc, bad.value)
        return tri, bary, off

    def apply_embedding(self, tri, bary, off, host_t, host_x):
        tri = np.ascontiguousarray(tri, np.int32)
        bary = np.ascontiguousarray(bary, np.float64).reshape(-1, 3)
        off = np.ascontiguousarray(off, np.float64)
        T = np.ascontiguousarray(host_t, np.int32).reshape(-1, 3)
        X = np.ascontiguousarray(host_x, np.float64).reshape(-1, 3)
        out = np.zeros((tri.size, 3))
        bad = C.c_int64(-1)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        rc = self.lib.orc_apply_embedding(p(tri), p(bary), p(off), C.c_int64(tri.size), p(T), C.c_int64(T.shape[0]),
                                          p(X), C.c_int64(X.shape[0]), p(out), C.byref(bad))
        self._check(rc, bad.value)
        return out

    # -- broadphase ------------------------------------------------------
    def candidate_pairs(self, slave, master, x, r: float, use_tree: bool = True):
        s, ka = surface_struct(slave)
        m, kb = surface_struct(master)
        x = np.ascontiguousarray(x, dtype=np.float64)
        h = C.c_void_p()
        self._check(self.lib.orc_build_candidate_pairs(C.byref(s), C.byref(m), x.ctypes.data_as(C.c_void_p),
                                                       C.c_double(r), C.c_int(int(use_tree)), C.byref(h)))
        try:
            return self._pairs_to_csr(h)
        finally:
            self.lib.orc_pairs_free(h)

    def _pairs_to_csr(self, h):
        nst = self.lib.orc_pairs_slave_tris(h)
        out = {}
        for which, name in enumerate(("tris", "edges", "verts")):
            n = self.lib.orc_pairs_size(h, which)
            off = np.zeros(nst + 1, np.int64)
            ids = np.zeros(max(n, 1), np.int32)
            self.lib.orc_pairs_copy(h, which, off.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p))
            out[name] = (off, ids[:n])
        return out

    def _pairs_handle(self, pairs):
        h = C.c_void_p()
        (to, ti), (eo, ei), (vo, vi) = pairs["tris"], pairs["edges"], pairs["verts"]
        arrs = [np.ascontiguousarray(a, dtype=dt) for a, dt in
                ((to, np.int64), (ti, np.int32), (eo, np.int64), (ei, np.int32), (vo, np.int64), (vi, np.int32))]
        self._check(self.lib.orc_pairs_from_csr(C.c_int32(to.size - 1), *[a.ctypes.data_as(C.c_void_p) for a in arrs],
                                                C.byref(h)))
        return h, arrs

    # -- sampler ---------------------------------------------------------
    def contact_state(self, slave, master, pairs, x, params, eps_reference=None):
        """Returns an OracleState (samples + reference positions)."""
        s, ka = surface_struct(slave)
        m, kb = surface_struct(master)
        ph, kc = self._pairs_handle(pairs)
        x = np.ascontiguousarray(x, dtype=np.float64)
        cp = params_struct(params)
        er = None if eps_reference is None else np.ascontiguousarray(eps_reference, dtype=np.float64)
        h = C.c_void_p()
        try:
            self._check(self.lib.orc_build_contact_state(
                C.byref(s), C.byref(m), ph, x.ctypes.data_as(C.c_void_p), C.c_int64(x.size), C.byref(cp),
                None if er is None else er.ctypes.data_as(C.c_void_p), C.byref(h)))
        finally:
            self.lib.orc_pairs_free(ph)
        return OracleState(self, h, x.size)

    def state_from_samples(self, samples: dict, ref_x):
        cs, keep = samples_struct(samples)
        ref_x = np.ascontiguousarray(ref_x, dtype=np.float64)
        h = C.c_void_p()
        self._check(self.lib.orc_state_from_samples(C.byref(cs), ref_x.ctypes.data_as(C.c_void_p),
                                                    C.c_int64(ref_x.size), C.byref(h)))
        return OracleState(self, h, ref_x.size)


class OracleState:
    def __init__(self, orc: Oracle, h, n_dof: int):
        self.orc, self.h, self.n_dof = orc, h, n_dof
        self.L = orc.lib

    def __del__(self):
        try:
            if self.h:
                self.L.orc_state_free(self.h)
                self.h = None
        except Exception:
            pass

    def __len__(self):
        return int(self.L.orc_state_size(self.h))

    def samples(self) -> dict:
        s = empty_samples(len(self))
        cs, keep = samples_struct(s)
        self.L.orc_state_copy(self.h, C.byref(cs))
        return keep

    @staticmethod
    def _p(a):
        return a.ctypes.data_as(C.c_void_p)

    def _x(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        assert x.size == self.n_dof
        return x

    def kinematics(self, x):
        n = len(self)
        g, nv = np.zeros(n), np.zeros(n, np.int32)
        ids, dg = np.zeros((n, 6), np.int32), np.zeros((n, 6, 3))
        x = self._x(x)
        self.orc._check(self.L.orc_kinematics(self.h, self._p(x), self._p(g), self._p(nv), self._p(ids), self._p(dg)))
        return g, nv, ids, dg

    def try_energy(self, params, x):
        e, mg, f = C.c_double(), C.c_double(), C.c_int32()
        cp = params_struct(params)
        x = self._x(x)
        self.orc._check(self.L.orc_try_contact_energy(self.h, C.byref(cp), self._p(x), C.byref(e), C.byref(mg), C.byref(f)))
        return e.value, mg.value, bool(f.value)

    def energy(self, params, x):
        e, bad = C.c_double(), C.c_int64(-1)
        cp = params_struct(params)
        x = self._x(x)
        rc = self.L.orc_contact_energy(self.h, C.byref(cp), self._p(x), C.byref(e), C.byref(bad))
        self.orc._check(rc, bad.value)
        return e.value

    def gradient(self, params, x, grad=None):
        x = self._x(x)
        grad = np.zeros(self.n_dof) if grad is None else np.ascontiguousarray(grad, dtype=np.float64).copy()
        e, bad = C.c_double(), C.c_int64(-1)
        cp = params_struct(params)
        rc = self.L.orc_add_contact_gradient(self.h, C.byref(cp), self._p(x), self._p(grad), C.byref(e), C.byref(bad))
        self.orc._check(rc, bad.value)
        return e.value, grad

    def gradient_hessian(self, params, x):
        """Returns (energy, grad, brow, bcol, bval(nb,3,3), n_triplets)."""
        x = self._x(x)
        cp = params_struct(params)
        g0 = np.zeros(self.n_dof)
        e, bad, nb, nt = C.c_double(), C.c_int64(-1), C.c_int64(), C.c_int64()
        rc = self.L.orc_add_contact_gradient_hessian(self.h, C.byref(cp), self._p(x), self._p(g0), C.byref(e),
                                                     C.byref(bad), C.byref(nb), None, None, None, C.byref(nt))
        self.orc._check(rc, bad.value)
        grad = np.zeros(self.n_dof)
        brow, bcol = np.zeros(nb.value, np.int32), np.zeros(nb.value, np.int32)
        bval = np.zeros((nb.value, 3, 3))
        rc = self.L.orc_add_contact_gradient_hessian(self.h, C.byref(cp), self._p(x), self._p(grad), C.byref(e),
                                                     C.byref(bad), C.byref(nb), self._p(brow), self._p(bcol),
                                                     self._p(bval), C.byref(nt))
        self.orc._check(rc, bad.value)
        return e.value, grad, brow, bcol, bval, nt.value

    def step_filter(self, x, dx):
        a = C.c_double()
        x, dx = self._x(x), self._x(dx)
        self.orc._check(self.L.orc_step_filter(self.h, self._p(x), self._p(dx), C.byref(a)))
        return a.value

    def displacement_cap(self, params, x, dx):
        a = C.c_double()
        cp = params_struct(params)
        x = self._x(x)
        dx = np.ascontiguousarray(dx, dtype=np.float64)
        self.orc._check(self.L.orc_displacement_cap(self.h, C.byref(cp), self._p(x), self._p(dx),
                                                    C.c_int64(dx.size), C.byref(a)))
        return a.value

    def pressure(self, params, x):
        x = self._x(x)
        cp = params_struct(params)
        n = C.c_int64()
        self.orc._check(self.L.orc_pressure_field(self.h, C.byref(cp), self._p(x), C.byref(n), None))
        out = np.zeros(n.value, PRESSURE_DTYPE)
        self.orc._check(self.L.orc_pressure_field(self.h, C.byref(cp), self._p(x), C.byref(n), self._p(out)))
        return out

    def time_assembly(self, params, x, reps=1):
        """Best-of-reps seconds of one add_contact_gradient_hessian call."""
        x = self._x(x)
        cp = params_struct(params)
        sec, nt = C.c_double(), C.c_int64()
        self.orc._check(self.L.orc_time_assembly(self.h, C.byref(cp), self._p(x), C.c_int32(reps), C.byref(sec),
                                                 C.byref(nt)))
        return sec.value, nt.value

    def force_summary(self, params, x):
        x = self._x(x)
        cp = params_struct(params)
        out = np.zeros(12)
        self.orc._check(self.L.orc_force_summary(self.h, C.byref(cp), self._p(x), self._p(out)))
        return out.reshape(4, 3)
