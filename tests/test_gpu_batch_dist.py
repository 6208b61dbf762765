"""C5 product path (paper_2605_24339_b200/batch.py): scenes
sharded over ranks by sample-count prefix sums, each shard solved as one
batched device System, per-scene results (final x, per-load-step StepStats,
pressure records) gathered once to rank 0.

On the one-GPU test box the world-2 job runs as two processes sharing cuda:0
with the gloo backend for the gather (a functional check of the N>1 path: the
ranks' kernels are independent, nothing waits on a co-resident rank). Rank
0's gathered results must equal a single-rank run of the whole job BITWISE,
since every scene's trajectory is independent of the batch it runs in."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_SCENES = 6
STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, counts, q):
    import torch
    import torch.distributed as dist
    from paper_2605_24339_b200 import batch as B
    from paper_2605_24339_b200 import system as SY
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res, info = B.run_batch(N_SCENES, SY.SolverSettings(load_steps=STEPS), dist=dist, device=0, counts=counts)
    if rank == 0:
        q.put((B.pack(res), info["scenes"]))
    else:
        q.put((None, info["scenes"]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_batch_equals_single_rank_bitwise():
    import torch.multiprocessing as mp
    from paper_2605_24339_b200 import batch as B
    from paper_2605_24339_b200 import system as SY
    counts = B.scene_sample_counts(N_SCENES, 0)
    assert counts.min() > 0
    single, info1 = B.run_batch(N_SCENES, SY.SolverSettings(load_steps=STEPS), counts=counts)
    assert [r.scene for r in single] == list(range(N_SCENES)) and info1["scenes"] == (0, N_SCENES)
    for r in single:
        assert r.steps.shape == (STEPS, 6) and np.all(r.steps[:, 0] >= 1)  # every step iterated
        assert r.pressure.size > 0 and np.all(r.steps[:, 5] > 0)          # contact, positive gaps
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, counts, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rows = next(g[0] for g in got if g[0] is not None)
    shards = sorted(g[1] for g in got)
    assert shards[0][0] == 0 and shards[0][1] == shards[1][0] and shards[1][1] == N_SCENES
    gathered = B.unpack(rows)
    assert [r.scene for r in gathered] == list(range(N_SCENES))
    for a, b in zip(single, gathered):
        assert a.same_as(b), f"scene {a.scene} differs between the 1-rank and the 2-rank job"
