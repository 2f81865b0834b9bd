"""Where the end-to-end (host buffers) pass spends its time beyond the device-resident pass, cfg3 fp32:
device-resident inputs vs pinned host inputs (same handle, warm), and the 49 cakf_get read-backs."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2405_08971_b200 import CAKF_SMOOTH, runner
from synth import make_workload

wl = make_workload("cfg3")
trans, _ = runner.transitions(wl)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
h = runner.make_handle(wl, "f32", stream=stream.cuda_stream)
dev_in = runner.stage_inputs(wl, "f32")
host_in = []
for (idx, y, nv, order) in runner.host_inputs(wl, "f32"):
    host_in.append(tuple(None if a is None else torch.from_numpy(a).pin_memory() for a in (idx, y, nv, order)))
outm = [torch.empty(wl.D, dtype=torch.float32).pin_memory() for _ in range(wl.T + 1)]
outv = [torch.empty(wl.D, dtype=torch.float32).pin_memory() for _ in range(wl.T + 1)]


def timed(fn, reps=2):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), 1e3 * (time.perf_counter() - w0)))
    return ts


def gets():
    for k in range(wl.T + 1):
        h.get(k, CAKF_SMOOTH, outm[k], outv[k])


runner.run(h, trans, dev_in)   # warm
res = {
    "device_inputs_pass_ms": timed(lambda: runner.run(h, trans, dev_in)),
    "host_inputs_pass_ms": timed(lambda: runner.run(h, trans, host_in)),
    "gets_ms": timed(gets),
    "host_inputs_pass_plus_gets_ms": timed(lambda: (runner.run(h, trans, host_in), gets())),
}
print(json.dumps(res))
