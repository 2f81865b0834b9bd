"""Host enqueue vs device time of one cfg3 pass: perf_counter around the enqueue only, then the stream sync,
then the device-wide sync (does any library side stream outlive the main stream's end event?)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_08971_b200 import runner
from synth import make_workload

wl = make_workload("cfg3")
trans, _ = runner.transitions(wl)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
h = runner.make_handle(wl, "f32", stream=stream.cuda_stream)
dev_in = runner.stage_inputs(wl, "f32")
runner.run(h, trans, dev_in)
torch.cuda.synchronize()
out = []
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    runner.run(h, trans, dev_in)
    e1.record(stream)
    t1 = time.perf_counter()
    stream.synchronize()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    out.append({"enqueue_ms": 1e3 * (t1 - t0), "stream_sync_wait_ms": 1e3 * (t2 - t1),
                "device_sync_extra_ms": 1e3 * (t3 - t2), "event_ms": e0.elapsed_time(e1), "wall_ms": 1e3 * (t3 - t0)})
# host enqueue of the filter alone vs the smoother alone
torch.cuda.synchronize()
t0 = time.perf_counter(); runner.run(h, trans, dev_in, smooth=False); t1 = time.perf_counter()
torch.cuda.synchronize(); t2 = time.perf_counter()
h.smooth(); t3 = time.perf_counter(); torch.cuda.synchronize(); t4 = time.perf_counter()
out.append({"filter_enqueue_ms": 1e3 * (t1 - t0), "filter_wall_ms": 1e3 * (t2 - t0),
            "smooth_enqueue_ms": 1e3 * (t3 - t2), "smooth_wall_ms": 1e3 * (t4 - t2),
            "launches_per_pass": h.kernel_launches() if hasattr(h, "kernel_launches") else None})
print(json.dumps(out, indent=1))
