"""Steady-state launch list: cfg3 filter steps k0..k0+1 (rank r_in = 512) and the whole smoother, bracketed by
cudaProfilerStart/Stop so that `ncu --profile-from-start off --metrics gpu__time_duration.sum` sees only them.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/steady.csv python scripts/launch_list_steady.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_08971_b200 import runner
from synth import make_workload

k0 = int(os.environ.get("STEADY_K0", "40"))
wl = make_workload("cfg3")
trans, _ = runner.transitions(wl)
h = runner.make_handle(wl, "f32")
inputs = runner.stage_inputs(wl, "f32")
h.reset()
for k, ((A, Q), (idx, y, nv, order)) in enumerate(zip(trans, inputs)):
    if k == k0:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    h.predict(A, Q)
    h.update(idx, y, nv, order)
    h.truncate()
    if k == k0 + 1:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
torch.cuda.synchronize()
torch.cuda.profiler.start()
h.smooth()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", [h.get_stats(k)["rank_in"] for k in (k0, k0 + 1)])
