"""Batched independent tactile scenes across GPUs: the
product path for "1024 independent tactile indentation scenes batched and
sharded across 1/2/4/8 B200" (BASELINE.json configs[4]).

One process per GPU (torchrun). Each rank

1. balances the job by per-scene contact sample counts (one LBVH + sampler
   pass over all scenes on its own GPU; dist.shard_scenes cuts contiguous
   ranges at equal prefix sums),
2. packs its scene range into one device System with per-vertex scene ids and
   runs the reference's load-stepped Newton loop (System::solve,
   solver.hpp:125-228) for every scene at once -- each scene converges,
   backtracks and re-samples on its own; there is no collective on this path,
3. returns per-scene results -- final positions, the per-load-step StepStats
   (solver.hpp:44-53, the StepCallback payload of solver.hpp:123) and the
   face-sample pressure records (contact_energy.hpp:225-242, the rows of
   bench.hpp:322-372's pressure CSV) -- which are gathered ONCE at the end to
   rank 0 over NCCL (torch.distributed.gather of one padded float64 row per
   scene; NCCL has no variable-size gather).

Every scene's trajectory is independent of the batch it runs in (per-scene
reductions, per-scene CTA PCG, per-scene re-sampling), so rank 0's gathered
results equal a single-rank run bitwise (tests/test_gpu_batch_dist.py)."""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import dist as D
from . import gmcp as _g
from . import scenes as S
from . import system as SY

STEP_FIELDS = ("newton_iters", "rebuilds", "backtracks", "residual", "energy", "min_gap")
_HEAD = 4  # scene id, n_dof, load steps, pressure records


@dataclass
class SceneResult:
    scene: int                # global scene id
    x: np.ndarray             # (3N,) final positions
    steps: np.ndarray         # (load_steps, 6) STEP_FIELDS per load step
    pressure: np.ndarray      # gmcp.PRESSURE_DTYPE records; `sample` is local to the scene

    def same_as(self, o: "SceneResult") -> bool:
        return (self.scene == o.scene and np.array_equal(self.x, o.x) and np.array_equal(self.steps, o.steps)
                and np.array_equal(self.pressure.view(np.uint8), o.pressure.view(np.uint8)))


def scene_sample_counts(n_scenes: int, device: int = 0, refine: float = 0.7) -> np.ndarray:
    """Contact samples of every scene of the job at rest (the shard balance
    weights): one batched broadphase + sampler pass on the device."""
    b = S.c5_batch(n_scenes, 0, n_scenes, refine=refine)
    ctx = _g.Context(device)
    ctx.set_params(b.params)
    ctx.set_surfaces(b.slave, b.master)
    ctx.set_positions(b.rest)
    ctx.set_vertex_scenes(b.vscene)
    ctx.broadphase(b.params.detection_radius)
    ctx.build_samples()
    smp = ctx.download_samples()
    ctx.close()
    scene_of_sample = b.vscene[smp["slave"][:, 0]]
    return np.bincount(scene_of_sample, minlength=n_scenes).astype(np.int64)


def solve_shard(n_scenes: int, first: int, count: int, settings: SY.SolverSettings | None = None,
                device: int = 0, refine: float = 0.7):
    """Solves scenes first .. first+count-1 of the job in one batched device
    System; returns ([SceneResult], RunStats, wall seconds)."""
    settings = settings or SY.SolverSettings()
    if count <= 0:  # more ranks than scenes
        return [], SY.RunStats(), 0.0
    b = S.c5_batch(n_scenes, first, count, refine=refine)
    sys_ = SY.build_hertz_batch_system(b, device=device)
    t0 = time.perf_counter()
    rs = sys_.solve(settings)
    wall = time.perf_counter() - t0
    st = sys_.scene_step_stats()
    press = sys_.contact_pressure_field(0)
    soff = sys_.pair_scene_offsets(0)
    N = b.base.rest.size // 3
    # face-sample records come in sample order: scene k's are one contiguous run
    cut = np.searchsorted(press["sample"], soff)
    out = []
    for k in range(count):
        pk = press[cut[k]:cut[k + 1]].copy()
        pk["sample"] -= soff[k]
        steps = np.stack([st[f][:, k].astype(np.float64) for f in STEP_FIELDS], axis=1)
        out.append(SceneResult(int(b.scenes[k]), sys_.x[3 * k * N:3 * (k + 1) * N].copy(), steps, pk))
    return out, rs, wall


def pack(results: list[SceneResult], width: int | None = None) -> np.ndarray:
    """One float64 row per scene: [scene, n_dof, load steps, n_pressure,
    x, steps, pressure records (7 doubles each: sample, position, radius, gap,
    pressure)], zero-padded to `width` (default: the longest row)."""
    rows = []
    for r in results:
        p = r.pressure
        prec = np.column_stack([p["sample"].astype(np.float64), p["position"], p["radius"], p["gap"],
                                p["pressure"]]) if p.size else np.zeros((0, 7))
        rows.append(np.concatenate([[r.scene, r.x.size, r.steps.shape[0], p.size], r.x, r.steps.ravel(),
                                    prec.ravel()]))
    w = max((row.size for row in rows), default=_HEAD) if width is None else width
    out = np.zeros((len(rows), w))
    for i, row in enumerate(rows):
        out[i, :row.size] = row
    return out


def unpack(rows: np.ndarray) -> list[SceneResult]:
    out = []
    for row in rows:
        scene, ndof, nsteps, npress = (int(v) for v in row[:_HEAD])
        o = _HEAD
        x = row[o:o + ndof].copy()
        o += ndof
        steps = row[o:o + 6 * nsteps].reshape(nsteps, 6).copy()
        o += 6 * nsteps
        pr = row[o:o + 7 * npress].reshape(npress, 7)
        p = np.zeros(npress, _g.PRESSURE_DTYPE)
        p["sample"] = pr[:, 0].astype(np.int64)
        p["position"] = pr[:, 1:4]
        p["radius"], p["gap"], p["pressure"] = pr[:, 4], pr[:, 5], pr[:, 6]
        out.append(SceneResult(scene, x, steps, p))
    return out


def gather_to_rank0(results: list[SceneResult], dist, device=None):
    """End-of-run gather (the only collective of the job): every rank's packed
    rows, padded to a common (rows, width), to rank 0 with one
    torch.distributed.gather (NCCL on the GPU box, gloo in the CPU tests).
    Returns (results in global scene order on rank 0, else None; bytes moved)."""
    import torch

    dev = device if device is not None else torch.device("cpu")
    local = pack(results)
    world = dist.get_world_size()
    shape = torch.tensor([local.shape[0], local.shape[1]], dtype=torch.int64, device=dev)
    dist.all_reduce(shape, op=dist.ReduceOp.MAX)
    kmax, w = int(shape[0]), int(shape[1])
    buf = torch.zeros((kmax, w), dtype=torch.float64, device=dev)
    if local.size:
        buf[:local.shape[0], :local.shape[1]] = torch.from_numpy(local).to(dev)
    rank = dist.get_rank()
    bufs = [torch.zeros_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, gather_list=bufs, dst=0)
    if rank != 0:
        return None, int(buf.numel() * 8)
    rows = np.concatenate([b.cpu().numpy() for b in bufs], axis=0)
    rows = rows[rows[:, 1] > 0]  # drop padding rows (n_dof > 0 for every real scene)
    res = sorted(unpack(rows), key=lambda r: r.scene)
    return res, int(world * buf.numel() * 8)


def run_batch(n_scenes: int = 1024, settings: SY.SolverSettings | None = None, dist=None, device: int = 0,
              refine: float = 0.7, counts: np.ndarray | None = None):
    """The C5 job on this rank's GPU (torchrun: one rank per GPU, `dist` =
    torch.distributed initialised, or None for one process). Returns
    (per-scene results on rank 0 / None elsewhere, info dict)."""
    import torch

    rank = dist.get_rank() if dist else 0
    world = dist.get_world_size() if dist else 1
    if counts is None:
        counts = scene_sample_counts(n_scenes, device, refine)
    lo, hi = D.shard_scenes(counts, world)[rank]
    res, rs, wall = solve_shard(n_scenes, lo, hi - lo, settings, device, refine)
    info = {"rank": rank, "scenes": (lo, hi), "wall_seconds": wall, "scene_newton_iters": int(rs.total_newton_iters),
            "samples": int(counts[lo:hi].sum())}
    if dist is None or world == 1:
        return res, info
    dev = torch.device("cuda", device) if dist.get_backend() == "nccl" else torch.device("cpu")
    t0 = time.perf_counter()
    gathered, nbytes = gather_to_rank0(res, dist, dev)
    info["gather_seconds"] = time.perf_counter() - t0
    info["gather_bytes"] = nbytes
    return gathered, info
