"""Multi-GPU plumbing for batched independent scenes.

Independent tactile scenes share nothing, so the hot path has no collective:
each rank (one process per GPU) runs its contiguous shard of scenes, and the
only communication is the end-of-run gather of per-scene results to rank 0
(NCCL over NVLink on the GPU box; gloo in the CPU tests). NCCL 2.27/2.28 has
no variable-size gather, so results are padded to the largest shard and
gathered with all_gather (one collective per run, not per iteration).
"""
from __future__ import annotations

import numpy as np


def shard_scenes(sample_counts, world: int):
    """Contiguous scene ranges [(lo, hi)] per rank, balanced by the prefix
    sum of per-scene sample counts (every rank gets >= 1 scene when possible)."""
    counts = np.asarray(sample_counts, dtype=np.float64)
    n = counts.size
    if world <= 0:
        raise ValueError("world must be positive")
    if n == 0:
        return [(0, 0)] * world
    cum = np.concatenate([[0.0], np.cumsum(counts)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        b = int(np.searchsorted(cum, target, side="left"))
        b = max(b, bounds[-1] + (1 if bounds[-1] < n - (world - r) else 0))
        b = min(b, n - (world - r)) if n >= world else min(b, n)
        bounds.append(max(b, bounds[-1]))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def gather_results(local: np.ndarray, dist, device=None):
    """Gathers each rank's (k_r, d) float64 result rows to every rank (rank 0
    uses them); returns the concatenation in rank order. `dist` is
    torch.distributed, already initialised."""
    import torch

    world = dist.get_world_size()
    local = np.ascontiguousarray(local, dtype=np.float64)
    if local.ndim == 1:
        local = local[:, None]
    dev = device if device is not None else torch.device("cpu")
    k = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    ks = [torch.zeros_like(k) for _ in range(world)]
    dist.all_gather(ks, k)
    kmax = int(max(int(t.item()) for t in ks))
    buf = torch.zeros((kmax, local.shape[1]), dtype=torch.float64, device=dev)
    if local.shape[0]:
        buf[: local.shape[0]] = torch.from_numpy(local).to(dev)
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    return np.concatenate([o[: int(kk.item())].cpu().numpy() for o, kk in zip(out, ks)], axis=0)


def max_over_ranks(value: float, dist, device=None) -> float:
    import torch

    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
