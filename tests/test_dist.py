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


def _synthetic_results(lo, hi):
    from paper_2605_24339_b200 import batch as B
    from paper_2605_24339_b200 import gmcp as G
    out = []
    for s in range(lo, hi):
        rng = np.random.default_rng(s)
        p = np.zeros(3 + s % 4, G.PRESSURE_DTYPE)
        p["sample"] = np.arange(p.size) * 7 + s
        p["position"] = rng.standard_normal((p.size, 3))
        p["radius"], p["gap"], p["pressure"] = rng.random(p.size), rng.random(p.size), rng.random(p.size) * 1e9
        out.append(B.SceneResult(s, rng.standard_normal(30 + 3 * (s % 2)), rng.standard_normal((4, 6)), p))
    return out


def _batch_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2605_24339_b200 import batch as B
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    counts = np.arange(9) + 10
    lo, hi = D.shard_scenes(counts, world)[rank]
    res, nbytes = B.gather_to_rank0(_synthetic_results(lo, hi), dist)
    if rank == 0:
        q.put((B.pack(res), nbytes))
    dist.barrier()
    dist.destroy_process_group()


def test_pack_unpack_round_trip():
    from paper_2605_24339_b200 import batch as B
    res = _synthetic_results(0, 7)
    back = B.unpack(B.pack(res))
    assert all(a.same_as(b) for a, b in zip(res, back)) and len(back) == 7


def test_gloo_world2_scene_result_gather():
    """The C5 end-of-run gather (batch.gather_to_rank0) over a world-2 gloo job:
    rank 0 receives every scene's positions, step stats and pressure records
    bitwise, in global scene order."""
    import torch.multiprocessing as mp
    from paper_2605_24339_b200 import batch as B
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows, nbytes = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = B.unpack(rows)
    want = _synthetic_results(0, 9)
    assert [r.scene for r in got] == list(range(9))
    assert all(a.same_as(b) for a, b in zip(want, got))
    assert nbytes > 0
