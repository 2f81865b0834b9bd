"""Independent problems on one GPU: two handles, each on its own stream and driven by its own host
thread, run concurrently (the serving mode `scripts/concurrent_bench.py` measures) and must give
bit-identical filter and smoother results to the same problems run one after the other.  This pins
that handles share no device state (K1 scheduling counters, culling lists, side streams, library
handles, workspaces) — DESIGN §7."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import make_workload  # noqa: E402


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _results(h, T):
    from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, runner
    return runner.collect(h, T, CAKF_FILTER), runner.collect(h, T, CAKF_SMOOTH)


def test_two_handles_concurrent_equal_sequential():
    from paper_2405_08971_b200 import runner
    wls = [make_workload("cfg2", T=4, max_iter=24, max_rank=64, seed=s) for s in (0, 1)]
    trans = [runner.transitions(wl)[0] for wl in wls]

    # sequential: one handle at a time on the current stream
    ref = []
    for wl, tr in zip(wls, trans):
        h = runner.make_handle(wl, "f32", stream=torch.cuda.current_stream().cuda_stream)
        runner.run(h, tr, runner.stage_inputs(wl, "f32"), smooth=True)
        torch.cuda.synchronize()
        ref.append(_results(h, wl.T))
        del h

    # concurrent: own stream + own host thread per handle, two passes each (second reuses the state)
    streams = [torch.cuda.Stream() for _ in wls]
    hs = [runner.make_handle(wl, "f32", stream=s.cuda_stream) for wl, s in zip(wls, streams)]
    ins = [runner.stage_inputs(wl, "f32") for wl in wls]
    errs = []

    def drive(p):
        try:
            for _ in range(2):
                runner.run(hs[p], trans[p], ins[p], smooth=True)
        except Exception as e:  # surfaced below
            errs.append(e)

    ths = [threading.Thread(target=drive, args=(p,)) for p in range(len(wls))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    for p, wl in enumerate(wls):
        got = _results(hs[p], wl.T)
        for (rm, rv), (gm, gv) in zip(ref[p], got):
            for a, b in zip(rm + rv, gm + gv):
                np.testing.assert_array_equal(a, b)
    # the two problems differ, so a cross-talk would not cancel out
    assert not np.array_equal(ref[0][1][0][-1], ref[1][1][0][-1])


_FRESH = r'''
import sys, threading
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, runner
from synth import make_workload
torch.cuda.set_device(0)
wls = [make_workload("sphere24", T=3, max_iter=12, max_rank=20, seed=s) for s in (0, 1)]
trans = [runner.transitions(wl)[0] for wl in wls]
ins = [runner.stage_inputs(wl, "f32") for wl in wls]
streams = [torch.cuda.Stream() for _ in wls]
out, errs = [None, None], []
go = threading.Barrier(2)

def drive(p):
    try:
        torch.cuda.set_device(0)
        go.wait()          # both threads make their FIRST library calls at the same time
        h = runner.make_handle(wls[p], "f32", stream=streams[p].cuda_stream)
        runner.run(h, trans[p], ins[p], smooth=True)
        out[p] = [runner.collect(h, wls[p].T, w) for w in (CAKF_FILTER, CAKF_SMOOTH)]
        h.destroy()
    except Exception as e:
        errs.append(repr(e))

ths = [threading.Thread(target=drive, args=(p,)) for p in range(2)]
for t in ths: t.start()
for t in ths: t.join()
assert not errs, errs
for p, wl in enumerate(wls):   # sequential re-run in the same process
    h = runner.make_handle(wl, "f32", stream=torch.cuda.current_stream().cuda_stream)
    runner.run(h, trans[p], ins[p], smooth=True)
    ref = [runner.collect(h, wl.T, w) for w in (CAKF_FILTER, CAKF_SMOOTH)]
    for (rm, rv), (gm, gv) in zip(ref, out[p]):
        for a, b in zip(rm + rv, gm + gv):
            np.testing.assert_array_equal(a, b)
print("fresh-concurrent ok")
'''


def test_fresh_handles_first_calls_concurrent():
    """the library's one-time setup (function attributes, occupancy, tensor-map entry point,
    env switches) must be safe when two fresh handles make their first calls from two host threads at
    once.  A fresh interpreter guarantees nothing was initialised beforehand."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _FRESH, root], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fresh-concurrent ok" in r.stdout
