#!/usr/bin/env python
"""GMCP B200 benchmark (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[2], SURVEY.md 8d "C3"): GelSight-style pad
slab(155,124) pressed by a textured indenter (A = 2e-4, f = 20), sampled at
rest -> 1,008,248 mortar contact samples, evaluated at the indented state
(-1.5 mm) with a seeded +-1e-4 perturbation of every coordinate (dense
Gauss-Newton blocks). Synthetic geometry, generated here; all FP64.

A "step" is one contact assembly pass over the resident sample set: barrier
energy + gradient + Gauss-Newton Hessian blocks assembled into BCSR
(K7 run partials + K8 row gather + deterministic energy reduction).
value = samples processed per second over the whole job (all ranks).

Multi-GPU (torchrun): every rank runs its own independent scene (batched
tactile rollouts are independent scenes) -> weak scaling, no
collective on the hot path; NCCL only for the end-of-run result gather and the
max-over-ranks timing.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GMCP contact samples/s and Newton steps/s at 1/2/4/8 B200 vs CPU ref"
UNIT = "samples/s"
WORKLOAD = "C3: GelSight pad slab(155,124) + textured indenter (A=2e-4, f=20), ~1M mortar samples, FP64"


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle sampling while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        loaded = [float(r[0]) for r in self.rows if len(r) > 8 and r[8].isdigit() and int(r[8]) > 0]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[4:8]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(loaded or sm) if (loaded or sm) else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def build_scene(seed: int):
    from paper_2605_24339_b200 import scenes as S
    return S.slab_scene(155, 124, texture_amp=2e-4, texture_freq=20.0, seed=seed)


def algorithmic_bytes(types: np.ndarray, n_vertices: int, nnzb: int):
    """SoA sample record face 88 B / edge 68 B / point 56 B;
    positions 24 B/vertex; gradient write 24 B/vertex; BCSR values 72 B/block."""
    nf = int((types == 2).sum())
    ne = int((types == 1).sum())
    npnt = int((types == 0).sum())
    samples = 88 * nf + 68 * ne + 56 * npnt
    k7 = samples + 24 * n_vertices  # dominant kernel: reads records + positions
    pass_bytes = samples + 48 * n_vertices + 72 * nnzb
    return {"faces": nf, "edges": ne, "points": npnt, "k7": k7, "pass": pass_bytes}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profiled_instructions():
    """Warp instructions per launch of K7 from the committed ncu capture, or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get("k_run_partials_warp_instructions")
    except Exception:
        return None


def profiled_traffic():
    """dram__bytes (read + write) per launch of the dominant kernel from the
    committed ncu capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get("k_run_partials_dram_bytes")
    except Exception:
        return None


def pcg_roofline(ps: dict, pre: dict | None = None) -> dict:
    """HBM roofline of one PCG iteration, device time from CUDA events around
    the chunk graphs of every PCG solve in the timed Newton run. Algorithmic
    bytes per iteration:
      SpMV    the symmetric-half operand: 72 B per stored block (on or above
              the diagonal) + 8 B (column, stored index) per block of the merged
              pattern (76 B per block when the full BCSR is read) + per row 4 B
              row pointer and 24 B each of z, p_old, mask read and p_new, q
              written (124 B); large systems split p = z + beta p into
              k_pupdate (z, p_old read, p_new written: 72 B/row) and the SpMV
              then reads p_new and mask and writes q (76 B/row);
      update  24 B each of p, q, x, r read and x, r, z written (168 B), the
              vertex-pair block-Jacobi rows (3x6 = 144 B) + 4 B pair index
              (316 B/row; the partner's r and q rows are L2 hits of rows another
              thread streams, not counted);
      two-level (coarse space on): the restriction fused into the update reads
              mask + aggregate offset + vertex id (52 B/row); the coarse solve +
              prolongation reads the dense coarse inverse (8 n_pad^2 B) and per
              row vertex id, offset, mask and z, writes z (100 B/row)."""
    if not ps["iters"]:
        return None
    peak, src = peaks()
    half = ps.get("stored_blocks", 0) > 0
    split = half and ps["rows"] >= 32768  # large systems stream p = z + beta p in k_pupdate
    row = (76 + 72 if split else 124) + (316 if (pre is None or pre["pair_jacobi"]) else 168 + 72)
    coarse = bool(pre and pre["coarse"])
    if coarse:
        row += 52 + 100
    mat = 72 * ps["stored_blocks"] + 8 * ps["nnzb"] if half else 76 * ps["nnzb"]
    per_iter = mat + row * ps["rows"] + (8 * pre["coarse_padded"] ** 2 if coarse else 0)
    ms = ps["ms"] / ps["iters"]
    achieved = per_iter / (ms / 1e3) / 1e9
    kern = ("k_pupdate + " if split else "") + (
        "k_spmv_cg + k_update_agg + k_coarse_prolong" if coarse else "k_spmv_cg + k_update_cg_pair")
    return {"bound": "hbm", "kernels": kern + " (one PCG iteration)", "achieved": achieved,
            "peak": peak, "unit": "GB/s", "frac": achieved / peak, "algorithmic_bytes": per_iter,
            "us_per_iter": 1e3 * ms, "iters_timed": ps["iters"], "operand_blocks": ps["nnzb"], "rows": ps["rows"],
            "stored_blocks": ps.get("stored_blocks", 0),
            "preconditioner": pre, "peak_source": src,
            "clock": "CUDA events around each 16-iteration chunk graph on the solve stream"}


def cpu_scene_reference(name: str):
    """The reference's parse_scene + build_scene + System::solve (scene.hpp,
    solver.hpp) on one of the repo's scene files, oracle/_ref, 1 thread."""
    import ctypes as C
    lib = os.path.join(ROOT, "oracle", "_ref", "libgmcp_ref.so")
    if not os.path.exists(lib):
        return None
    L = C.CDLL(lib)
    path = os.path.join(ROOT, "scenes", name + ".scene").encode()
    n = C.c_int64()
    if L.ref_run_scene(C.c_char_p(path), C.byref(n), None, None, None, C.c_int32(0)) != 0:
        return None
    x, st, fo = np.zeros(n.value), np.zeros(6), np.zeros(24)
    if L.ref_run_scene(C.c_char_p(path), C.byref(n), C.c_void_p(x.ctypes.data), C.c_void_p(st.ctypes.data),
                       C.c_void_p(fo.ctypes.data), C.c_int32(8)) != 0:
        return None
    return {"newton_iters": int(st[0]), "rebuilds": int(st[1]), "wall_seconds": float(st[3]),
            "steps_per_s": float(st[0] / st[3]), "x": x}


def cpu_newton_reference(refine: float = 0.7):
    """The reference's own System::solve (solver.hpp:125-228) through run_hertz
    (bench.hpp:210-303) on C1, compiled from the reference sources (oracle/_ref;
    the Eigen shim's SimplicialLDLT stand-in with an RCM ordering), 1 thread:
    Newton iterations per second of the whole 10-step solve."""
    import ctypes as C
    lib = os.path.join(ROOT, "oracle", "_ref", "libgmcp_ref.so")
    if not os.path.exists(lib):
        return None
    L = C.CDLL(lib)
    v = np.zeros(14)
    rc = L.ref_run_hertz(C.c_double(refine), C.c_int32(10), C.c_void_p(v.ctypes.data))
    if rc != 0:
        return None
    return {"newton_iters": int(v[8]), "wall_seconds": float(v[11]), "steps_per_s": float(v[8] / v[11]),
            "peak": float(v[0]), "cores": 1, "kind": "reference",
            "sample": f"C1 Hertz (refine {refine}) full 10-load-step solve, reference System::solve via run_hertz, "
                      "oracle/_ref (shim SimplicialLDLT with RCM ordering), 1 thread"}


def cpu_baseline(scene, samples: dict, x: np.ndarray, seconds_budget: float = 20.0, threads: int | None = None):
    """Reference CPU path (oracle/_ref when built here, else the C restatement)
    timed on this host on a bounded sample of the same workload: whole-slab
    shards of the C3 sample set, one shard per host thread."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, Oracle
    if not os.path.exists(LIBS["restated"]):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "libgmcp_oracle.so"], check=True,
                       capture_output=True)
    kind = "reference" if os.path.exists(LIBS["reference"]) else "restated"
    orc = Oracle(kind)
    n = samples["type"].size
    threads = threads or 1
    # bounded sample: the first `take` samples (whole slave triangles, reference order)
    probe = orc.state_from_samples({k: v[: min(n, 20000)] for k, v in samples.items()}, x)
    t_probe, _ = probe.time_assembly(scene.params, x, 1)
    per_sample = t_probe / max(1, min(n, 20000))
    take = int(min(n, max(20000, seconds_budget * threads / max(per_sample, 1e-12) / 2)))
    shard = (take + threads - 1) // threads
    states = [orc.state_from_samples({k: v[i * shard:(i + 1) * shard] for k, v in samples.items()}, x)
              for i in range(threads)]
    res = [None] * threads

    def work(i):
        res[i] = states[i].time_assembly(scene.params, x, 2)

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    slowest = max(r[0] for r in res)
    total = sum(states[i].__len__() for i in range(threads))
    return {"value": total / slowest, "unit": UNIT, "cores": threads,
            "kind": "reference" if kind == "reference" else "port",
            "sample": f"{total} of {n} C3 samples ({threads} shard(s)), add_contact_gradient_hessian, best of 2, "
                      f"{wall:.1f} s wall", "triplets": int(sum(r[1] for r in res))}


def run_reference(args):
    rank, world, local = _dist()
    if rank != 0:
        return 0
    from paper_2605_24339_b200 import scenes as S
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, Oracle
    if not os.path.exists(LIBS["restated"]):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "libgmcp_oracle.so"], check=True,
                       capture_output=True)
    kind = "reference" if os.path.exists(LIBS["reference"]) else "restated"
    orc = Oracle(kind)
    scene = build_scene(12345)
    # CPU sampling of C3 by the oracle itself (no GPU on this arm)
    t0 = time.perf_counter()
    pairs = orc.candidate_pairs(scene.slave, scene.master, scene.rest, scene.params.detection_radius)
    st = orc.contact_state(scene.slave, scene.master, pairs, scene.rest, scene.params)
    samples = st.samples()
    t_build = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    x = scene.x_eval
    times = []
    n = samples["type"].size
    shard = (n + threads - 1) // threads
    states = [orc.state_from_samples({k: v[i * shard:(i + 1) * shard] for k, v in samples.items()}, x)
              for i in range(threads)]
    for step in range(args.warmup + args.steps):
        res = [None] * threads

        def work(i):
            res[i] = states[i].time_assembly(scene.params, x, 1)[0]

        ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = n / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "samples": int(n), "impl_path": f"oracle ({kind})",
                       "build_seconds": t_build},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                             "kind": "reference" if kind == "reference" else "port",
                             "sample": f"full C3 sample set sharded over {threads} threads, "
                                       f"add_contact_gradient_hessian per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-newton", action="store_true")
    ap.add_argument("--newton-iters", type=int, default=5)
    ap.add_argument("--no-batched", action="store_true")
    ap.add_argument("--batch-scenes", type=int, default=1024)
    ap.add_argument("--no-job", action="store_true", help="skip the full C5 solve + result gather")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    rank, world, local = _dist()
    import torch
    # GMCP_BENCH_SHARE_GPU=1 (functional check only, never a measurement): N
    # ranks share the visible GPUs round-robin over gloo, so the N>1 path runs
    # on a 1-GPU box; the ranks' kernels are independent (no collective on the
    # hot path), so nothing waits on a co-resident rank
    share = os.environ.get("GMCP_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2605_24339_b200 import gmcp as gm

    scene = build_scene(12345 + rank)
    ctx = gm.Context(local)
    ctx.set_params(scene.params)
    ctx.set_surfaces(scene.slave, scene.master)
    ctx.set_positions(scene.rest)
    t0 = time.perf_counter()
    ctx.broadphase(scene.params.detection_radius)
    n = ctx.build_samples()
    t_rebuild = time.perf_counter() - t0  # cold: the context's buffers are allocated here
    t0 = time.perf_counter()  # warm: the rebuild a Newton load step pays (same buffers)
    ctx.broadphase(scene.params.detection_radius)
    n = ctx.build_samples()
    t_rebuild_warm = time.perf_counter() - t0
    ctx.set_positions(scene.x_eval)
    ctx.set_step(scene.dx)
    g = np.zeros(scene.rest.size)
    e0 = ctx.gradient(g, hessian=True)  # builds the assembly plan (per rebuild)
    rowptr, cols, _ = ctx.download_hessian()
    samples = ctx.download_samples()
    ab = algorithmic_bytes(samples["type"], scene.rest.size // 3, int(cols.size))

    # warm-up (untimed)
    ctx.time_assembly(args.warmup, True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches
    with ClockSampler(local) as clk:
        time.sleep(0.25)
        ms_pass, ms_k7 = ctx.time_assembly(args.steps, True)  # CUDA events on the ctx stream, L2 flushed per step
        launches = ctx.launches - l0
        # keep the GPU busy long enough for the clock sampler to see it under load
        t_hold = time.perf_counter()
        while time.perf_counter() - t_hold < 1.0:
            ctx.time_assembly(20, False)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
        t = torch.tensor([ms_pass, ms_k7], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_pass, ms_k7 = float(t[0]), float(t[1])
    value = world * n / (ms_pass / 1e3)

    # end-to-end through the public API with host buffers (pinned), per step:
    # H2D x (3N doubles) and of the caller's gradient (3N doubles, accumulated
    # into as the reference's add_contact_gradient_hessian does), assembly, D2H
    # gradient (3N doubles) + energy: one C-ABI call (gmcp_add_gradient_hessian).
    xh = torch.empty(scene.rest.size, dtype=torch.float64, pin_memory=True).numpy()
    gh = torch.empty(scene.rest.size, dtype=torch.float64, pin_memory=True).numpy()
    xh[:] = scene.x_eval
    gh[:] = 0
    for _ in range(args.warmup):
        ctx.add_gradient(xh, gh, hessian=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.add_gradient(xh, gh, hessian=True)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    e2e = world * n * args.steps / e2e_s

    # drop-in end to end: the reference's add_contact_gradient_hessian(state,
    # params, x, grad, H) RETURNS H to the caller. Per step: the single-call
    # assembly above plus the download of the Gauss-Newton Hessian (BCSR:
    # row pointers, columns, 3x3 values) into host memory.
    ctx.add_gradient(xh, gh, hessian=True)
    rp_h, cl_h, vl_h = ctx.download_hessian()
    hbytes = int(rp_h.nbytes + cl_h.nbytes + vl_h.nbytes)
    pinned = (torch.empty(rp_h.size, dtype=torch.int32, pin_memory=True).numpy(),
              torch.empty(cl_h.size, dtype=torch.int32, pin_memory=True).numpy(),
              torch.empty(vl_h.size, dtype=torch.float64, pin_memory=True).numpy().reshape(-1, 3, 3))
    nd = max(3, args.steps // 5)
    for _ in range(2):
        ctx.add_gradient(xh, gh, hessian=True)
        ctx.download_hessian(pinned)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(nd):
        ctx.add_gradient(xh, gh, hessian=True)
        ctx.download_hessian(pinned)
    e2e_dropin_s = (time.perf_counter() - t0) / nd
    if dist:
        t = torch.tensor([e2e_dropin_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_dropin_s = float(t[0])
    e2e_dropin = {"value": world * n / e2e_dropin_s, "unit": UNIT, "ms_per_step": 1e3 * e2e_dropin_s,
                  "h2d_bytes_per_step": int(2 * scene.rest.size * 8),
                  "d2h_bytes_per_step": int(scene.rest.size * 8 + 40 + hbytes),
                  "path": "gmcp_add_gradient_hessian + gmcp_download_hessian into pinned host buffers: the Hessian "
                          "returned to the host as BCSR (include/gmcp/b200.hpp then expands it into Eigen triplets, "
                          "not timed here)"}

    # end-of-run result gather (NCCL): per-rank sample counts and energies
    if dist:
        from paper_2605_24339_b200 import dist as D
        rows = D.gather_results(np.array([[float(n), e0]]), dist, device=torch.device("cuda", local))
        total_samples = int(rows[:, 0].sum())
    else:
        total_samples = n

    # Newton steps/s: C3 with patch-test BCs, device-resident
    # System::solve; each timed iteration = assembly, residual, PCG to
    # tolerance, filter + cap, every line-search trial, rebuild check.
    newton = None
    if not args.no_newton:
        from paper_2605_24339_b200 import system as SY
        nsys = SY.build_slab_system(155, 124, texture_amp=2e-4, device=local)
        settings = SY.SolverSettings(pcg_tol=1e-10, pcg_max_iters=50000)  # the product default
        if dist:
            dist.barrier()
        ms_it, pcg_it = nsys.time_newton(settings, args.newton_iters + 1)
        ps = nsys.pcg_stats()
        ps.update(nsys.operand_info())
        pre = nsys.precond_info()
        lin = nsys.linear_stats()
        steady = ms_it[1:] if ms_it.size > 1 else ms_it
        t = float(np.mean(steady))
        if dist:
            tt = torch.tensor([t], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt[0])
        newton = {"steps_per_s": world * 1e3 / t, "ms_per_iter": t, "per_iter_ms": [round(float(v), 3) for v in ms_it],
                  "pcg_iters": [int(v) for v in pcg_it], "pcg_tol": settings.pcg_tol,
                  "first_iter_includes": "load-step rebuild + one-time elastic BCSR build (excluded from the mean)",
                  "dofs": int(nsys.rest.size), "samples": int(nsys.num_samples(0)),
                  "clock": "host steady_clock around each iteration (device synchronized)",
                  "preconditioner": pre, "true_residual_max": lin["max_rel2"],
                  "pcg_roofline": pcg_roofline(ps, pre)}
        del nsys
        # C1 (the CPU reference's own scene): device Newton steps/s and the whole
        # 10-step solve next to the reference System::solve on the host
        from paper_2605_24339_b200 import scenes as S
        c1cfg = S.HertzConfig(refine=0.7)  # C1: refine 0.7, the scene the CPU reference solves below
        hs, _ = SY.build_hertz_system(c1cfg, device=local)
        ms_h, pcg_h = hs.time_newton(SY.SolverSettings(), args.newton_iters + 3)
        del hs
        t0 = time.perf_counter()
        hr = SY.run_hertz(c1cfg, device=local)
        dev_solve = time.perf_counter() - t0
        newton["c1"] = {"scene": "C1 Hertz (refine 0.7), 3,759 dofs",
                        "steps_per_s": world * 1e3 / float(np.mean(ms_h[3:])),
                        "per_iter_ms": [round(float(v), 3) for v in ms_h], "pcg_iters": [int(v) for v in pcg_h],
                        "solve_seconds": dev_solve, "solve_newton_iters": int(hr.stats.total_newton_iters),
                        "solve_steps_per_s": hr.stats.total_newton_iters / dev_solve, "peak": hr.peak}
        del hr
        # C4 (scenes/fingertip.scene: two pads squeeze a clamped object, 2 contact
        # pairs, 20 load steps, rebuilds): parse_scene + build_scene + solve
        from paper_2605_24339_b200 import scene as SC
        t0 = time.perf_counter()
        c4_sys, c4_st = SC.run_scene(os.path.join(ROOT, "scenes", "fingertip.scene"), device=local)
        c4_s = time.perf_counter() - t0
        newton["c4"] = {"scene": "C4 fingertip (scenes/fingertip.scene), 2 contact pairs, 20 load steps",
                        "solve_seconds": c4_s, "solve_newton_iters": int(c4_st.total_newton_iters),
                        "solve_rebuilds": int(c4_st.total_rebuilds), "solve_steps_per_s": c4_st.total_newton_iters / c4_s,
                        "x": c4_sys.x.copy()}
        del c4_sys

    # C5: the 1024-scene batched job (C1 Hertz scenes) on the
    # product path (paper_2605_24339_b200/batch.py): scenes sharded across
    # ranks by sample-count prefix sums (dist.shard_scenes), each shard packed
    # into one context / System per GPU; no collective on the hot path; one
    # NCCL gather of the per-scene results at the end.
    batched = None
    if not args.no_batched:
        from paper_2605_24339_b200 import batch as B
        from paper_2605_24339_b200 import dist as D
        from paper_2605_24339_b200 import scenes as S
        counts = B.scene_sample_counts(args.batch_scenes, local)
        first, last = D.shard_scenes(counts, world)[rank]
        count = last - first
        b = S.c5_batch(args.batch_scenes, first, count)
        bctx = gm.Context(local)
        bctx.set_params(b.params)
        bctx.set_surfaces(b.slave, b.master)
        bctx.set_positions(b.rest)
        bctx.set_vertex_scenes(b.vscene)
        torch.cuda.synchronize()
        tb0 = time.perf_counter()
        bctx.broadphase(b.params.detection_radius)
        nb_s = bctx.build_samples()
        t_brebuild = time.perf_counter() - tb0
        bctx.set_positions(b.x_eval)
        gb = np.zeros(b.rest.size)
        bctx.gradient(gb, hessian=True)
        bctx.time_assembly(args.warmup, True)
        if dist:
            dist.barrier()
        ms_b, _ = bctx.time_assembly(args.steps, True)
        tot = float(nb_s)
        if dist:
            t = torch.tensor([ms_b, tot], device="cuda", dtype=torch.float64)
            t2 = t.clone()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.all_reduce(t2, op=dist.ReduceOp.SUM)
            ms_b, tot = float(t[0]), float(t2[1])
        del bctx
        # batched Newton: the shard as one device System, every scene
        # with its own residual / step / line search / convergence; timed loop
        # passes 3..8 (pass 1-2: set-up and the singular first load-step solve)
        newton_b = None
        job = None
        if not args.no_newton:
            from paper_2605_24339_b200 import system as SY
            bsys = SY.build_hertz_batch_system(b, device=local)
            if dist:
                dist.barrier()
            ms_b_it, pcg_b = bsys.time_newton(SY.SolverSettings(load_steps=10), 8)
            act = bsys.timed_active_scenes(len(ms_b_it))
            steps_b, t_b = float(act[2:].sum()), float(ms_b_it[2:].sum()) / 1e3
            if dist:
                t = torch.tensor([t_b, steps_b], device="cuda", dtype=torch.float64)
                t2 = t.clone()
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dist.all_reduce(t2, op=dist.ReduceOp.SUM)
                t_b, steps_b = float(t[0]), float(t2[1])
            newton_b = {"scene_newton_steps_per_s": steps_b / t_b, "passes_timed": int(len(ms_b_it) - 2),
                        "per_pass_ms": [round(float(v), 2) for v in ms_b_it],
                        "pcg_iters": [int(v) for v in pcg_b], "scenes_per_pass": [int(v) for v in act],
                        "definition": "scene-Newton-iterations (one scene's assemble + PCG + filter + line search) "
                                      "per second, all scenes of the shard in one batched device solve"}
            del bsys
            # the whole job end to end: every scene's 10-step solve, then the
            # per-scene results (final x, StepStats per load step, pressure
            # records) gathered to rank 0 (one NCCL gather)
            if not args.no_job:
                if dist:
                    dist.barrier()
                torch.cuda.synchronize()
                tj = time.perf_counter()
                res, info = B.run_batch(args.batch_scenes, SY.SolverSettings(), dist=dist, device=local,
                                        counts=counts)
                torch.cuda.synchronize()
                wall = time.perf_counter() - tj
                its = float(info["scene_newton_iters"])
                if dist:
                    t = torch.tensor([wall, info["wall_seconds"]], device="cuda", dtype=torch.float64)
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    wall, solve_s = float(t[0]), float(t[1])
                    t2 = torch.tensor([its], device="cuda", dtype=torch.float64)
                    dist.all_reduce(t2, op=dist.ReduceOp.SUM)
                    its = float(t2[0])
                else:
                    solve_s = info["wall_seconds"]
                job = {"what": f"{args.batch_scenes} scenes x 10 load steps, solved and gathered to rank 0",
                       "wall_seconds": wall, "solve_seconds_max_rank": solve_s, "scene_newton_iters": int(its),
                       "scene_newton_steps_per_s": its / wall,
                       "gather_seconds": info.get("gather_seconds", 0.0), "gather_bytes": info.get("gather_bytes", 0),
                       "scenes_gathered": len(res) if res is not None else None,
                       "x_checksum": float(sum(float(r.x.sum()) for r in res)) if res else None}
        batched = {"workload": f"C5: {args.batch_scenes} independent C1 Hertz scenes (refine 0.7) sharded across "
                               f"{world} GPU(s) by sample-count prefix sums, packed per GPU with scene ids",
                   "samples_per_s": tot / (ms_b / 1e3), "ms_per_step": ms_b, "samples_total": int(tot),
                   "scenes_per_gpu": count, "samples_rank0": int(nb_s),
                   "scaling": "strong (fixed job, scenes sharded)",
                   "rebuild_seconds_rank0": t_brebuild,
                   "step": "energy + gradient + Gauss-Newton BCSR assembly over the packed batch, L2 flushed",
                   "newton": newton_b, "job": job}

    peak, peak_src = peaks()
    achieved_k7 = ab["k7"] / (ms_k7 / 1e3) / 1e9
    achieved_pass = ab["pass"] / (ms_pass / 1e3) / 1e9
    # north_star's "contact assembly + PCG" target, per steady Newton iteration
    # of C3: one assembly pass (bytes and event time above) plus that
    # iteration's PCG (mean steady iteration count x the event-timed bytes and
    # time of one PCG iteration).
    roofline_newton = None
    if newton and newton["pcg_roofline"] and len(newton["pcg_iters"]) > 1:
        pr = newton["pcg_roofline"]
        its = float(np.mean(newton["pcg_iters"][1:]))
        nb_ = ab["pass"] + its * pr["algorithmic_bytes"]
        nms = ms_pass + its * pr["us_per_iter"] / 1e3
        roofline_newton = {"bound": "hbm", "what": "contact assembly pass + PCG to tolerance, per steady C3 Newton "
                                                   "iteration", "achieved": nb_ / (nms / 1e3) / 1e9, "peak": peak,
                           "unit": "GB/s", "frac": nb_ / (nms / 1e3) / 1e9 / peak, "algorithmic_bytes": nb_,
                           "ms": nms, "pcg_iters_mean": its}
    e2e_solve = None
    if rank == 0 and newton and not args.no_cpu_baseline:
        ref = cpu_newton_reference()
        if ref:
            newton["cpu_baseline"] = {"value": ref["steps_per_s"], "unit": "Newton steps/s", "cores": 1,
                                      "kind": ref["kind"], "sample": ref["sample"]}
            c1 = newton["c1"]
            e2e_solve = {"what": "full load-stepped solves through the public API (host scene in, host x out): "
                                 "device System::solve vs the reference System::solve on 1 host thread",
                         "c1": {"device_seconds": c1["solve_seconds"], "reference_seconds": ref["wall_seconds"],
                                "speedup": ref["wall_seconds"] / c1["solve_seconds"],
                                "device_newton_iters": c1["solve_newton_iters"],
                                "reference_newton_iters": ref["newton_iters"], "device_peak": c1["peak"],
                                "reference_peak": ref["peak"]}}
        c4 = newton.get("c4")
        r4 = cpu_scene_reference("fingertip") if c4 else None
        if r4:
            x4 = c4.pop("x")
            newton["cpu_baseline_c4"] = {"value": r4["steps_per_s"], "unit": "Newton steps/s", "cores": 1,
                                         "kind": "reference", "sample": "C4 fingertip full 20-load-step solve, "
                                         "reference parse_scene + build_scene + System::solve (oracle/_ref), 1 thread"}
            e2e_solve = e2e_solve or {"what": "full load-stepped solves, device vs reference"}
            e2e_solve["c4"] = {"device_seconds": c4["solve_seconds"], "reference_seconds": r4["wall_seconds"],
                               "speedup": r4["wall_seconds"] / c4["solve_seconds"],
                               "device_newton_iters": c4["solve_newton_iters"],
                               "reference_newton_iters": r4["newton_iters"],
                               "device_rebuilds": c4["solve_rebuilds"], "reference_rebuilds": r4["rebuilds"],
                               "max_abs_x_diff": float(np.abs(x4 - r4["x"]).max())}
    if newton and "c4" in newton:
        newton["c4"].pop("x", None)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(scene, samples, scene.x_eval, args.cpu_seconds, threads=1)
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": f"failed: {exc}"}
    if rank == 0:
        clocks = clk.summary()
        traffic = profiled_traffic()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_pass, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "samples_per_gpu": n, "samples_total": total_samples,
                       "faces": ab["faces"], "edges": ab["edges"], "points": ab["points"],
                       "contact_bcsr_blocks": int(cols.size), "vertices": int(scene.rest.size // 3),
                       "l2": "flushed between timed steps (256 MB write > 126 MB L2)",
                       "step": "energy + gradient + Gauss-Newton BCSR assembly (K7+K8+reduce)",
                       "rebuild_seconds_broadphase_plus_sampler": t_rebuild,
                       "rebuild_seconds_warm": t_rebuild_warm,
                       "parallelism": f"{world} independent scene(s), one per GPU"},
            "roofline": {"bound": "hbm", "kernel": "k_run_partials (K7)", "achieved": achieved_k7, "peak": peak,
                         "unit": "GB/s", "frac": achieved_k7 / peak, "traffic": traffic,
                         "algorithmic_bytes": ab["k7"], "ms": ms_k7, "peak_source": peak_src},
            # K7 is issue-bound, not HBM-bound: its warp instructions (ncu) over the
            # event-timed launch against the issue peak (148 SMs x 4 schedulers x 1 warp
            # instruction per cycle at the measured SM clock)
            "roofline_issue": ({"bound": "issue", "kernel": "k_run_partials (K7)",
                                "achieved": insts / (ms_k7 / 1e3) / 1e9,
                                "peak": 148 * 4 * (clocks.get("sm_mhz") or 1965.0) / 1e3,
                                "unit": "G warp-instructions/s",
                                "frac": insts / (ms_k7 / 1e3) / (148 * 4 * (clocks.get("sm_mhz") or 1965.0) * 1e6),
                                "instructions": insts} if (insts := profiled_instructions()) else None),
            "roofline_pass": {"achieved": achieved_pass, "peak": peak, "unit": "GB/s", "frac": achieved_pass / peak,
                              "algorithmic_bytes": ab["pass"], "ms": ms_pass},
            "roofline_newton": roofline_newton,
            "e2e_dropin": e2e_dropin,
            "e2e_solve": e2e_solve,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(2 * scene.rest.size * 8),
                    "d2h_bytes_per_step": int(scene.rest.size * 8 + 40),
                    "path": "gmcp.Context.add_gradient(x, grad, hessian=True) = one C-ABI call "
                            "gmcp_add_gradient_hessian (reference add_contact_gradient_hessian(state, params, x, "
                            "grad, H)): H2D x + caller grad, assembly, D2H grad += g_c + energy/status; pinned "
                            "host buffers; host wall clock around the loop"},
            "newton": newton,
            "batched": batched,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
