"""CPU coverage of the N>1 path: scene sharding and the end-of-run result
gather, run as a world_size-2 gloo job on 127.0.0.1."""
import os
import socket

import numpy as np
import pytest

from paper_2605_24339_b200 import dist as D


def test_shard_balanced_contiguous_complete():
    rng = np.random.default_rng(0)
    counts = rng.integers(3000, 5000, size=1024)
    for world in (1, 2, 4, 8):
        sh = D.shard_scenes(counts, world)
        assert sh[0][0] == 0 and sh[-1][1] == 1024
        assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
        loads = [counts[lo:hi].sum() for lo, hi in sh]
        assert max(loads) / (counts.sum() / world) < 1.02
        assert all(hi > lo for lo, hi in sh)


def test_shard_more_ranks_than_scenes():
    sh = D.shard_scenes([5, 5, 5], 4)
    assert sh[-1][1] == 3 and all(hi >= lo for lo, hi in sh)
    assert sum(hi - lo for lo, hi in sh) == 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    counts = np.arange(10, 30)
    lo, hi = D.shard_scenes(counts, world)[rank]
    # per-scene "result" rows: (scene id, energy-like value)
    local = np.stack([np.arange(lo, hi), np.arange(lo, hi) * 0.5 + rank * 0], axis=1).astype(float)
    allres = D.gather_results(local, dist)
    t = D.max_over_ranks(1.0 + rank, dist)
    if rank == 0:
        q.put((allres, t))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allres, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(allres[:, 0], np.arange(20))
    assert np.allclose(allres[:, 1], np.arange(20) * 0.5)
    assert t == 2.0
