"""Host mirror of gmcp::System (proj/include/gmcp/solver.hpp:63-376) over the
device-resident solver C-ABI (include/gmcp_solver.h), plus the patch-test
scene of bench.hpp:44-124 / scene.hpp:381-449.

Same names and argument meaning as the reference: add_body, fix_dof,
fix_vertex, add_contact_pair, solve(settings, on_step) -> RunStats, with the
reference exceptions (ConfigError, SolverError{residual}). The linear solve
is a block-Jacobi PCG on the GPU instead of SimplicialLDLT.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import gmcp as _g
from . import scenes as S


@dataclass
class SolverSettings:
    """solver.hpp:35-42 + PCG controls."""

    load_steps: int = 10
    max_newton_iters: int = 200
    newton_tol: float = -1.0
    max_line_search: int = 40
    pcg_tol: float = 1e-10
    pcg_max_iters: int = 20000


class _Settings(C.Structure):
    _fields_ = [("load_steps", C.c_int32), ("max_newton_iters", C.c_int32), ("newton_tol", C.c_double),
                ("max_line_search", C.c_int32), ("pcg_tol", C.c_double), ("pcg_max_iters", C.c_int32)]


class _StepStats(C.Structure):
    _fields_ = [("step", C.c_int32), ("newton_iters", C.c_int32), ("rebuilds", C.c_int32),
                ("backtracks", C.c_int32), ("pcg_iters", C.c_int64), ("residual", C.c_double),
                ("energy", C.c_double), ("min_gap", C.c_double), ("energy_monotone", C.c_int32)]


# gmcp_step_stats as a numpy record (include/gmcp_solver.h; natural C alignment)
SCENE_STEP_DTYPE = np.dtype([("step", np.int32), ("newton_iters", np.int32), ("rebuilds", np.int32),
                             ("backtracks", np.int32), ("pcg_iters", np.int64), ("residual", np.float64),
                             ("energy", np.float64), ("min_gap", np.float64), ("energy_monotone", np.int32),
                             ("_pad", np.int32)])


class _RunStats(C.Structure):
    _fields_ = [("total_newton_iters", C.c_int64), ("total_rebuilds", C.c_int64), ("total_pcg_iters", C.c_int64),
                ("newton_tol_used", C.c_double), ("wall_seconds", C.c_double), ("residual", C.c_double)]


_CB = C.CFUNCTYPE(None, C.POINTER(_StepStats), C.POINTER(C.c_double), C.c_int64, C.c_void_p)


@dataclass
class StepStats:
    step: int
    newton_iters: int
    rebuilds: int
    backtracks: int
    pcg_iters: int
    residual: float
    energy: float
    min_gap: float
    energy_monotone: bool


@dataclass
class RunStats:
    steps: list = field(default_factory=list)
    newton_tol_used: float = 0.0
    wall_seconds: float = 0.0
    total_newton_iters: int = 0
    total_rebuilds: int = 0
    total_pcg_iters: int = 0


@dataclass
class Body:
    mesh: S.TetMesh
    youngs: float
    poisson: float
    name: str
    vertex_offset: int
    boundary: S.SurfaceMesh


def _lib():
    L = _g.library()
    L.gmcp_system_last_error.restype = C.c_char_p
    L.gmcp_system_launch_count.restype = C.c_int64
    L.gmcp_system_num_samples.restype = C.c_int64
    L.gmcp_system_destroy.restype = None
    L.gmcp_system_destroy.argtypes = [C.c_void_p]
    return L


def _check(L, rc, residual=float("nan")):
    if rc != 0:
        msg = L.gmcp_system_last_error().decode()
        if rc == _g.GMCP_ERR_SOLVER:
            raise _g.SolverError(msg, residual)
        raise _g._EXC.get(rc, _g.Error)(msg)


class System:
    def __init__(self, device: int = 0):
        self.L = _lib()
        h = C.c_void_p()
        _check(self.L, self.L.gmcp_system_create(C.c_int(device), C.byref(h)))
        self.h = h
        self.bodies: list[Body] = []
        self.rest = np.zeros(0)
        self.x = np.zeros(0)
        self.f_ext = np.zeros(0)
        self.fixed = np.zeros(0, np.uint8)
        self.dirichlet = np.zeros(0)
        self.contacts = []  # (slave ContactSurface, master ContactSurface, resolved params)

    def __del__(self):
        try:
            if self.h:
                self.L.gmcp_system_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def num_vertices(self) -> int:
        return self.rest.size // 3

    def add_body(self, mesh: S.TetMesh, youngs: float, poisson: float, name: str = "", boundary=None) -> int:
        return self.add_bodies([(mesh, youngs, poisson, name, boundary)])

    def add_bodies(self, specs) -> int:
        """Adds (mesh, youngs, poisson, name, boundary or None) bodies in order;
        returns the index of the last one. Loads and BCs are set afterwards."""
        parts = [self.rest]
        for mesh, youngs, poisson, name, boundary in specs:
            v = np.ascontiguousarray(mesh.vertices, np.float64)
            t = np.ascontiguousarray(mesh.tets, np.int32)
            off = C.c_int32()
            _check(self.L, self.L.gmcp_system_add_body(self.h, _g._p(v), C.c_int64(v.shape[0]), _g._p(t),
                                                       C.c_int64(t.shape[0]), C.c_double(youngs),
                                                       C.c_double(poisson), C.byref(off)))
            self.bodies.append(Body(mesh, youngs, poisson, name, off.value,
                                    boundary if boundary is not None else S.extract_boundary_surface(mesh)))
            parts.append(v.ravel())
        self.rest = np.concatenate(parts)
        self.x = self.rest.copy()
        self.f_ext = np.zeros_like(self.rest)
        self.fixed = np.zeros(self.rest.size, np.uint8)
        self.dirichlet = self.rest.copy()
        return len(self.bodies) - 1

    def set_vertex_scenes(self, scene):
        """Batched independent scenes (C5): scene id per vertex, 0, 1, ... in
        contiguous vertex ranges; solve() then converges each scene on its own."""
        self._scenes = None if scene is None else np.ascontiguousarray(scene, np.int32)

    _scenes = None

    def timed_active_scenes(self, n: int) -> np.ndarray:
        """After time_newton on a batched system: scenes iterated per timed pass."""
        out = np.zeros(n, np.int64)
        self.L.gmcp_system_timed_active_scenes(self.h, _g._p(out), C.c_int32(n))
        return out

    def scene_newton_iters(self) -> np.ndarray:
        n = 0 if self._scenes is None else int(self._scenes.max()) + 1
        out = np.zeros(n, np.int64)
        if n:
            self.L.gmcp_system_scene_newton_iters(self.h, _g._p(out))
        return out

    def scene_step_stats(self) -> np.ndarray:
        """Per-scene StepStats of the last batched solve: (load_steps, n_scenes)
        structured array (step, newton_iters, rebuilds, backtracks, pcg_iters,
        residual, energy, min_gap, energy_monotone)."""
        n_steps = C.c_int32()
        _check(self.L, self.L.gmcp_system_scene_step_stats(self.h, C.byref(n_steps), None))
        ns = 0 if self._scenes is None else int(self._scenes.max()) + 1
        out = np.zeros((n_steps.value, ns), dtype=SCENE_STEP_DTYPE)
        if out.size:
            _check(self.L, self.L.gmcp_system_scene_step_stats(self.h, C.byref(n_steps), _g._p(out)))
        return out

    def pair_scene_offsets(self, pair: int = 0) -> np.ndarray:
        """Sample offsets of each scene in a pair's packed sample set (after a batched solve)."""
        ns = 0 if self._scenes is None else int(self._scenes.max()) + 1
        out = np.zeros(ns + 1, np.int64)
        _check(self.L, self.L.gmcp_system_pair_scene_offsets(self.h, C.c_int32(pair), _g._p(out)))
        return out

    def fix_dof(self, gv: int, axis: int, target: float):
        self.fixed[3 * gv + axis] = 1
        self.dirichlet[3 * gv + axis] = target

    def fix_vertex(self, gv: int, target):
        for c in range(3):
            self.fix_dof(gv, c, target[c])

    def add_contact_pair(self, slave_body: int, master_body: int, params: S.BarrierParams, slave_tris=None,
                         master_tris=None) -> int:
        sb, mb = self.bodies[slave_body], self.bodies[master_body]
        slave = S.make_contact_surface(sb.boundary, sb.vertex_offset, slave_tris)
        master = S.make_contact_surface(mb.boundary, mb.vertex_offset, master_tris)
        p = S.resolve_barrier_params(params, S.mean_edge_length(slave, self.rest))
        self.contacts.append((slave, master, p))
        return len(self.contacts) - 1

    def add_contact_surfaces(self, slave: S.ContactSurface, master: S.ContactSurface,
                             resolved_params: S.BarrierParams) -> int:
        """A contact pair over prebuilt (global-id) surfaces, e.g. packed scene
        batches spanning several bodies; params already resolved."""
        self.contacts.append((slave, master, resolved_params))
        return len(self.contacts) - 1

    def _push(self):
        idx = np.nonzero(self.fixed)[0].astype(np.int64)
        tg = np.ascontiguousarray(self.dirichlet[idx])
        _check(self.L, self.L.gmcp_system_fix_dofs(self.h, C.c_int64(idx.size), _g._p(idx), _g._p(tg)))
        f = np.ascontiguousarray(self.f_ext, np.float64)
        _check(self.L, self.L.gmcp_system_set_external_force(self.h, _g._p(f), C.c_int64(f.size)))
        x = np.ascontiguousarray(self.x, np.float64)
        _check(self.L, self.L.gmcp_system_set_positions(self.h, _g._p(x), C.c_int64(x.size)))
        if self._scenes is not None:
            _check(self.L, self.L.gmcp_system_set_vertex_scenes(self.h, _g._p(self._scenes),
                                                                C.c_int64(self._scenes.size)))
        for (slave, master, p) in self.contacts[self._pushed_pairs:]:
            arrs, st = [], []
            for s in (slave, master):
                a = [np.ascontiguousarray(v, dtype=np.int32) for v in (s.tris, s.edges, s.tri_edges, s.verts)]
                arrs += a
                st.append(_g._Surface(a[0].shape[0], a[0].ctypes.data, a[1].shape[0], a[1].ctypes.data,
                                      a[2].ctypes.data, a[3].shape[0], a[3].ctypes.data))
            cp = _g._params(p)
            pid = C.c_int32()
            _check(self.L, self.L.gmcp_system_add_contact_pair(self.h, C.byref(st[0]), C.byref(st[1]), C.byref(cp),
                                                               C.byref(pid)))
        self._pushed_pairs = len(self.contacts)

    _pushed_pairs = 0

    def solve(self, settings: SolverSettings | None = None, on_step=None) -> RunStats:
        settings = settings or SolverSettings()
        self._push()
        stats = RunStats()

        def cb(ss_p, x_p, n, user):
            ss = ss_p.contents
            s = StepStats(ss.step, ss.newton_iters, ss.rebuilds, ss.backtracks, ss.pcg_iters, ss.residual, ss.energy,
                          ss.min_gap, bool(ss.energy_monotone))
            stats.steps.append(s)
            if on_step is not None:
                on_step(s, np.ctypeslib.as_array(x_p, shape=(n,)).copy())

        cbf = _CB(cb)
        st = _Settings(settings.load_steps, settings.max_newton_iters, settings.newton_tol, settings.max_line_search,
                       settings.pcg_tol, settings.pcg_max_iters)
        out = _RunStats()
        rc = self.L.gmcp_system_solve(self.h, C.byref(st), cbf, None, C.byref(out))
        _check(self.L, rc, out.residual)
        x = np.zeros_like(self.rest)
        _check(self.L, self.L.gmcp_system_positions(self.h, _g._p(x), C.c_int64(x.size)))
        self.x = x
        stats.newton_tol_used = out.newton_tol_used
        stats.wall_seconds = out.wall_seconds
        stats.total_newton_iters = out.total_newton_iters
        stats.total_rebuilds = out.total_rebuilds
        stats.total_pcg_iters = out.total_pcg_iters
        return stats

    def time_newton(self, settings: SolverSettings | None = None, n_iters: int = 3):
        """Wall ms and PCG iterations of the first n_iters full Newton iterations."""
        settings = settings or SolverSettings()
        self._push()
        st = _Settings(settings.load_steps, settings.max_newton_iters, settings.newton_tol, settings.max_line_search,
                       settings.pcg_tol, settings.pcg_max_iters)
        ms = np.zeros(n_iters)
        pcg = np.zeros(n_iters, np.int64)
        done = C.c_int32()
        _check(self.L, self.L.gmcp_system_time_newton(self.h, C.byref(st), C.c_int32(n_iters), _g._p(ms), _g._p(pcg),
                                                      C.byref(done)))
        return ms[:done.value], pcg[:done.value]

    def pcg_stats(self) -> dict:
        """PCG chunk-graph device time (CUDA events) and iterations since the
        last time_newton started, and the merged operand's shape."""
        ms = C.c_double()
        it, rows, nnzb = C.c_int64(), C.c_int64(), C.c_int64()
        _check(self.L, self.L.gmcp_system_pcg_stats(self.h, C.byref(ms), C.byref(it), C.byref(rows), C.byref(nnzb)))
        return {"ms": ms.value, "iters": it.value, "rows": rows.value, "nnzb": nnzb.value}

    def precond_info(self) -> dict:
        a, b, c, d = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(self.L, self.L.gmcp_system_precond_info(self.h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return {"pair_jacobi": bool(a.value), "coarse": bool(b.value), "aggregates": c.value, "coarse_padded": d.value}

    def operand_info(self) -> dict:
        """Blocks the PCG SpMV streams from the symmetric-half operand copy
        (0: it reads the full merged BCSR)."""
        n = C.c_int64()
        _check(self.L, self.L.gmcp_system_operand_info(self.h, C.byref(n)))
        return {"half": n.value > 0, "stored_blocks": n.value}

    def linear_stats(self, reset: bool = False) -> dict:
        """Recomputed true residuals of the linear solves since the last reset:
        max ||H dx - rhs||_2/||rhs||_2, max inf-norm ratio (the reference's
        acceptance test, solver.hpp:349-356), number of solves."""
        r2, ri, n = C.c_double(), C.c_double(), C.c_int64()
        _check(self.L, self.L.gmcp_system_linear_stats(self.h, C.c_int32(1 if reset else 0), C.byref(r2), C.byref(ri),
                                                       C.byref(n)))
        return {"max_rel2": r2.value, "max_relinf": ri.value, "solves": n.value}

    def capture_linear_system(self, on: bool = True):
        _check(self.L, self.L.gmcp_system_capture_linear_system(self.h, C.c_int32(1 if on else 0)))

    def captured_linear_system(self) -> dict:
        """The last captured solve: BCSR operand (all sources summed), mask,
        gradient (rhs = -mask * grad), dx and the diagonal shift."""
        nnzb, shift = C.c_int64(), C.c_double()
        _check(self.L, self.L.gmcp_system_captured_linear_system(self.h, C.byref(nnzb), None, None, None, None, None,
                                                                 None, C.byref(shift)))
        nv, n = self.rest.size // 3, self.rest.size
        rowptr, cols = np.zeros(nv + 1, np.int32), np.zeros(nnzb.value, np.int32)
        vals = np.zeros((nnzb.value, 3, 3))
        mask, grad, dx = np.zeros(n), np.zeros(n), np.zeros(n)
        _check(self.L, self.L.gmcp_system_captured_linear_system(self.h, C.byref(nnzb), _g._p(rowptr), _g._p(cols),
                                                                 _g._p(vals), _g._p(mask), _g._p(grad), _g._p(dx),
                                                                 C.byref(shift)))
        return {"rowptr": rowptr, "cols": cols, "vals": vals, "mask": mask, "grad": grad, "dx": dx,
                "shift": shift.value}

    @property
    def launches(self) -> int:
        return int(self.L.gmcp_system_launch_count(self.h))

    def num_samples(self, pair: int = 0) -> int:
        return int(self.L.gmcp_system_num_samples(self.h, C.c_int32(pair)))

    def contact_force_summary(self, pair: int = 0):
        out = np.zeros(12)
        _check(self.L, self.L.gmcp_system_pair_force_summary(self.h, C.c_int32(pair), _g._p(out)))
        return out.reshape(4, 3)

    def contact_pressure_field(self, pair: int = 0):
        n = C.c_int64()
        _check(self.L, self.L.gmcp_system_pair_pressure(self.h, C.c_int32(pair), C.byref(n), None))
        out = np.zeros(n.value, _g.PRESSURE_DTYPE)
        if n.value:
            _check(self.L, self.L.gmcp_system_pair_pressure(self.h, C.c_int32(pair), C.byref(n), _g._p(out)))
        return out


# ---------------------------------------------------------------------------
# elasticity helpers (elasticity.hpp:20-61, 147-160; bench.hpp:18-25)

@dataclass
class LinearSolveResult:
    dx: np.ndarray
    iterations: int
    residual_inf_rel: float  # ||H dx - rhs||_inf / ||rhs||_inf (the reference's acceptance test)
    regularized: bool        # accepted only after the 1e-8 diagonal shift (solver.hpp:352-361)


def solve_descent(rowptr: np.ndarray, cols: np.ndarray, vals: np.ndarray, rhs: np.ndarray,
                  fixed: np.ndarray | None = None, positions: np.ndarray | None = None, pcg_tol: float = 1e-10,
                  max_iters: int = 20000, device: int = 0) -> LinearSolveResult:
    """The reference's System::solve_descent (solver.hpp:325-375) on the GPU for
    a caller-assembled Newton matrix: H as an AoS BCSR of 3x3 blocks (rowptr
    [n+1], ascending cols, vals [nnzb, 3, 3] or [9 nnzb]), Dirichlet dofs
    `fixed` (eliminated as P H P + I - P), optional rest `positions` for the
    two-level preconditioner's aggregates. Same acceptance, regularized retry
    and SolverError as the reference (gmcp_system_linear_solve)."""
    L = _lib()
    h = C.c_void_p()
    _check(L, L.gmcp_system_create(C.c_int(device), C.byref(h)))
    try:
        rp = np.ascontiguousarray(rowptr, np.int32)
        cl = np.ascontiguousarray(cols, np.int32)
        vl = np.ascontiguousarray(vals, np.float64).reshape(-1)
        n = rp.size - 1
        b = np.ascontiguousarray(rhs, np.float64)
        if b.size != 3 * n or vl.size != 9 * cl.size:
            raise _g.ConfigError("solve_descent: rhs must have 3 n entries and vals 9 per block")
        fx = None if fixed is None else np.ascontiguousarray(fixed, np.uint8)
        ps = None if positions is None else np.ascontiguousarray(positions, np.float64)
        dx = np.zeros(3 * n)
        it, rel, reg = C.c_int32(), C.c_double(), C.c_int32()
        rc = L.gmcp_system_linear_solve(h, C.c_int64(n), _g._p(rp), _g._p(cl), _g._p(vl),
                                        None if fx is None else _g._p(fx), None if ps is None else _g._p(ps),
                                        _g._p(b), C.c_double(pcg_tol), C.c_int32(max_iters), _g._p(dx),
                                        C.byref(it), C.byref(rel), C.byref(reg))
        _check(L, rc)
        return LinearSolveResult(dx, it.value, rel.value, bool(reg.value))
    finally:
        L.gmcp_system_destroy(h)


def material(E: float, nu: float):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    return lam, mu


def shape_gradients(verts: np.ndarray, tets: np.ndarray):
    D = np.stack([verts[tets[:, i + 1]] - verts[tets[:, 0]] for i in range(3)], axis=2)  # columns
    G = np.linalg.inv(D)  # rows = grads of shape functions 1..3
    g0 = -G.sum(axis=1)
    return np.concatenate([g0[:, None, :], G], axis=1), np.linalg.det(D) / 6.0  # (nt,4,3), vol


def body_stresses(body: Body, x: np.ndarray, rest: np.ndarray) -> np.ndarray:
    g, _ = shape_gradients(body.mesh.vertices, body.mesh.tets)
    off = body.vertex_offset
    u = (x.reshape(-1, 3) - rest.reshape(-1, 3))[off + body.mesh.tets]  # (nt,4,3)
    grad_u = np.einsum("tia,tib->tab", u, g)
    eps = 0.5 * (grad_u + np.swapaxes(grad_u, 1, 2))
    lam, mu = material(body.youngs, body.poisson)
    tr = np.trace(eps, axis1=1, axis2=2)
    return lam * tr[:, None, None] * np.eye(3) + 2 * mu * eps


add_pressure_forces = S.add_pressure_forces


def build_patch_scene(kappa: float = 1e6, div_bottom=(5, 5, 2), div_top=(4, 4, 2), device: int = 0) -> System:
    """make_patch_scene + build_scene (bench.hpp:44-99, scene.hpp:381-449)."""
    sys_ = System(device)
    bottom = S.make_block((1, 1, 0.5), div_bottom)
    top = S.make_block((1, 1, 0.5), div_top, (0, 0, 0.502))
    ib = sys_.add_body(bottom, 1000.0, 0.0, "bottom")
    it = sys_.add_body(top, 1000.0, 0.0, "top")

    def inside(p, lo, hi):
        return np.all((p >= lo) & (p <= hi), axis=-1)

    r3 = sys_.rest.reshape(-1, 3)
    for bi, lo, hi, axes in ((ib, (-1, -1, -1), (2, 2, 1e-9), (0, 1, 2)), (it, (-1, -1, 0.5), (2, 2, 2), (0, 1))):
        b = sys_.bodies[bi]
        gv = b.vertex_offset + np.arange(b.mesh.vertices.shape[0])
        sel = gv[inside(r3[gv], np.array(lo), np.array(hi))]
        for v in sel:
            for k in axes:
                sys_.fix_dof(int(v), k, r3[v, k])
    tb = sys_.bodies[it]
    gtris = tb.vertex_offset + tb.boundary.vertex_map[tb.boundary.triangles]
    load = gtris[np.all(inside(r3[gtris], np.array((-1, -1, 1.0019)), np.array((2, 2, 2))), axis=1)]
    add_pressure_forces(load, sys_.rest, 10.0, (0, 0, -1), sys_.f_ext)
    slave_sel = np.nonzero(np.all(inside(r3[gtris], np.array((-1, -1, 0.5019)), np.array((2, 2, 0.5021))),
                                  axis=1))[0]
    sys_.add_contact_pair(it, ib, S.BarrierParams(kappa_face=kappa, eps_max=0.001), slave_sel, None)
    return sys_


def patch_stress_metrics(sys_: System, pressure: float = 10.0):
    """bench.hpp:101-111 -> (sigma_zz_max_rel_err, sigma_spur)."""
    zz, spur = 0.0, 0.0
    for b in sys_.bodies:
        s = body_stresses(b, sys_.x, sys_.rest)
        zz = max(zz, float(np.max(np.abs(s[:, 2, 2] + pressure) / pressure)))
        spur = max(spur, float(np.max(np.abs(s[:, [0, 1, 0, 1, 0], [0, 1, 1, 2, 2]]))))
    return zz, spur


def build_slab_system(nb: int, nt: int, texture_amp: float = 0.0, texture_freq: float = 20.0,
                      kappa: float = 1e6, pressure: float = 10.0, device: int = 0) -> System:
    """SURVEY.md 8d Newton-steps/s scene for C2/C3: slab(nb, nt) with the
    make_patch_scene boundary conditions (bench.hpp:64-84): master bottom face
    clamped, slave body u_x = u_y = 0, uniform pressure on the slave top face
    along -z (lambda-ramped), E = 1000, nu = 0."""
    sl = S.slab_scene(nb, nt, texture_amp=texture_amp, texture_freq=texture_freq)
    sys_ = System(device)
    ib = sys_.add_body(sl.meshes[0], 1000.0, 0.0, "indenter")
    it = sys_.add_body(sl.meshes[1], 1000.0, 0.0, "pad")
    r3 = sys_.rest.reshape(-1, 3)
    b = sys_.bodies[ib]
    gv = b.vertex_offset + np.arange(b.mesh.vertices.shape[0])
    for v in gv[r3[gv, 2] < 1e-9]:
        sys_.fix_vertex(int(v), r3[v])
    t = sys_.bodies[it]
    gv = t.vertex_offset + np.arange(t.mesh.vertices.shape[0])
    for v in gv:
        sys_.fix_dof(int(v), 0, r3[v, 0])
        sys_.fix_dof(int(v), 1, r3[v, 1])
    gtris = t.vertex_offset + t.boundary.vertex_map[t.boundary.triangles]
    top = gtris[np.all(np.abs(r3[gtris, 2] - 0.202) < 1e-9, axis=1)]
    add_pressure_forces(top, sys_.rest, pressure, (0, 0, -1), sys_.f_ext)
    down = np.nonzero(np.all(np.abs(r3[gtris, 2] - 0.102) < 1e-9, axis=1))[0]
    sys_.add_contact_pair(it, ib, S.BarrierParams(kappa_face=kappa, eps_max=1e-3), down, None)
    return sys_


# ---------------------------------------------------------------------------
# Hertz sphere-on-block indentation (C1), bench.hpp:195-303

@dataclass
class HertzResult:
    oracle: S.HertzOracle
    params: S.BarrierParams
    block_tets: int = 0
    ball_tets: int = 0
    applied_force: float = 0.0
    peak: float = 0.0
    contact_radius: float = 0.0
    outside_max: float = 0.0
    peak_rel_err: float = 0.0
    contact_radius_rel_err: float = 0.0
    profile: np.ndarray | None = None  # (n, 3): radius, pressure, analytic pressure
    stats: RunStats | None = None
    face_samples: int = 0
    system: object = None  # the device System that ran the solve


def build_hertz_system(cfg: S.HertzConfig | None = None, device: int = 0, scene: S.HertzScene | None = None):
    """run_hertz set-up (bench.hpp:210-272) on a device System. Returns
    (System, HertzResult skeleton)."""
    sc = scene or S.hertz_scene(cfg)
    sys_ = System(device)
    ib = sys_.add_body(sc.block, sc.cfg.E, sc.cfg.nu, "block")
    ih = sys_.add_body(sc.ball, sc.cfg.E, sc.cfg.nu, "ball")
    for (v, ax), t in zip(sc.fixed.tolist(), sc.fixed_target.tolist()):
        sys_.fix_dof(v, ax, t)
    sys_.f_ext[:] = sc.f_ext
    sys_.add_contact_pair(ib, ih, sc.params, sc.slave_tris, None)
    res = HertzResult(sc.oracle, sys_.contacts[0][2], sc.block.tets.shape[0], sc.ball.tets.shape[0],
                      sc.applied_force)
    return sys_, res


def run_hertz(cfg: S.HertzConfig | None = None, settings: SolverSettings | None = None, device: int = 0,
              on_step=None) -> HertzResult:
    """bench.hpp:210-303 on the device: solve, then the pressure profile metrics."""
    cfg = cfg or S.HertzConfig()
    sys_, res = build_hertz_system(cfg, device)
    settings = settings or SolverSettings()
    settings.load_steps = cfg.load_steps
    res.stats = sys_.solve(settings, on_step)
    res.system = sys_
    field = sys_.contact_pressure_field(0)
    res.face_samples = int(field.size)
    r, p = field["radius"].astype(np.float64), field["pressure"].astype(np.float64)
    res.peak = max(0.0, float(p.max())) if p.size else 0.0
    order = np.argsort(r, kind="stable")
    res.profile = np.stack([r[order], p[order], res.oracle.pressure(r[order])], axis=1)
    act = p >= 0.05 * res.peak
    res.contact_radius = float(r[act].max()) if np.any(act) else 0.0
    out = r > 1.2 * res.oracle.alpha_H
    res.outside_max = max(0.0, float(p[out].max())) if np.any(out) else 0.0
    res.peak_rel_err = abs(res.peak - res.oracle.p0) / res.oracle.p0
    res.contact_radius_rel_err = abs(res.contact_radius - res.oracle.alpha_H) / res.oracle.alpha_H
    return res


def build_hertz_batch_system(batch: S.SceneBatch, device: int = 0, load_scale: bool = True) -> System:
    """C5 as one device System: the batch's Hertz scenes (block + shifted ball
    per scene, quarter-model BCs, pressure Q * q_scale[s] on each ball top),
    one packed contact pair, per-vertex scene ids. solve() then runs every
    scene's Newton loop on its own (batched reductions)."""
    base = batch.base
    sys_ = System(device)
    N = base.rest.size // 3
    nb = base.ball_offset
    bb, bh = S.extract_boundary_surface(base.block), S.extract_boundary_surface(base.ball)  # same topology per scene
    specs = []
    for k in range(batch.scenes.size):
        specs.append((base.block, base.cfg.E, base.cfg.nu, f"block{k}", bb))
        bv = batch.rest.reshape(-1, 3)[k * N + nb:(k + 1) * N]
        specs.append((S.TetMesh(bv.copy(), base.ball.tets), base.cfg.E, base.cfg.nu, f"ball{k}", bh))
    sys_.add_bodies(specs)
    cnt = batch.scenes.size
    dofs = (3 * (base.fixed[:, 0][None, :] + N * np.arange(cnt)[:, None]) + base.fixed[:, 1][None, :]).ravel()
    sys_.fixed[dofs] = 1
    sys_.dirichlet[dofs] = sys_.rest[dofs]
    q = batch.q_scale if load_scale else np.ones(cnt)
    sys_.f_ext[:] = (base.f_ext.reshape(1, -1) * q[:, None]).ravel()
    sys_.add_contact_surfaces(batch.slave, batch.master, base.params)
    sys_.set_vertex_scenes(batch.vscene)
    return sys_


def build_hertz_scene_system(batch: S.SceneBatch, k: int, device: int = 0, load_scale: bool = True) -> System:
    """Scene k of a batch as its own System (same meshes, BCs and loads)."""
    base = batch.base
    sys_ = System(device)
    N = base.rest.size // 3
    nb = base.ball_offset
    ib = sys_.add_body(base.block, base.cfg.E, base.cfg.nu, "block")
    bv = batch.rest.reshape(-1, 3)[k * N + nb:(k + 1) * N]
    ih = sys_.add_body(S.TetMesh(bv.copy(), base.ball.tets), base.cfg.E, base.cfg.nu, "ball")
    dofs = 3 * base.fixed[:, 0] + base.fixed[:, 1]
    sys_.fixed[dofs] = 1
    sys_.dirichlet[dofs] = sys_.rest[dofs]
    sys_.f_ext[:] = base.f_ext * (batch.q_scale[k] if load_scale else 1.0)
    sl = S.make_contact_surface(sys_.bodies[ib].boundary, 0, base.slave_tris)
    ms = S.make_contact_surface(sys_.bodies[ih].boundary, nb)
    sys_.add_contact_surfaces(sl, ms, base.params)
    return sys_
