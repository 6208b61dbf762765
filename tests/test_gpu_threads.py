"""Independent contexts driven from different host threads at the same time
(INTEGRATION.md threading contract; SURVEY.md 8b "independent contexts may
run on different host threads"). Each C-ABI call binds its context's device
and its own CUB temp storage, so concurrent rebuilds (radix sorts, scans)
and assemblies of two contexts must give exactly the single-thread results.
ctypes releases the GIL for the duration of every C-ABI call."""
import threading

import numpy as np
import pytest

from paper_2605_24339_b200 import scenes as S

pytestmark = pytest.mark.gpu


def _run(sl, reps=6):
    from paper_2605_24339_b200 import gmcp as gm
    ctx = gm.Context(0)
    ctx.set_params(sl.params)
    ctx.set_surfaces(sl.slave, sl.master)
    out = None
    for _ in range(reps):
        ctx.set_positions(sl.rest)
        ctx.broadphase(sl.params.detection_radius)
        n = ctx.build_samples()
        ctx.set_positions(sl.x_eval)
        g = np.zeros_like(sl.rest)
        e = ctx.gradient(g, hessian=True)
        rowptr, cols, vals = ctx.download_hessian()
        res = (n, e, g, cols.copy(), vals.copy())
        if out is not None:  # repeatable inside the thread too
            assert res[0] == out[0] and res[1] == out[1] and np.array_equal(res[2], out[2])
        out = res
    ctx.close()
    return out


def test_two_contexts_two_threads_bitwise():
    scenes = [S.slab_scene(40, 32, texture_amp=2e-4, seed=1), S.slab_scene(36, 29, seed=2)]
    serial = [_run(sl, reps=1) for sl in scenes]
    got = [None, None]
    errs = []

    def work(k):
        try:
            got[k] = _run(scenes[k])
        except Exception as ex:  # surfaced below
            errs.append(ex)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for a, b in zip(serial, got):
        assert a[0] == b[0] and a[1] == b[1]
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
