"""cfg4 (N_X = 501,000, D = 1,002,000, N = 376,500, r = 1024) for a few steps on one GPU:
timing per phase, finiteness, variance sanity, and sampled K1 / K2 rows vs the oracle."""
import json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, binding, runner
from synth import make_workload

T = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = make_workload("cfg4", T=T)
stream = torch.cuda.Stream()   # a dedicated stream: the handle runs on it and the events bracket its work
torch.cuda.set_stream(stream)
t0 = time.time()
trans, Sinf = runner.transitions(wl)
h = runner.make_handle(wl, "f32", stream=stream.cuda_stream)
inputs = runner.stage_inputs(wl, "f32")
h.profile(True)
runner.run(h, trans, inputs, smooth=True)   # warm
h.profile_read(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
runner.run(h, trans, inputs, smooth=True)
e1.record()
torch.cuda.synchronize()
prof = h.profile_read(reset=True)
ms = e0.elapsed_time(e1)
ok = True
for k in range(T + 1):
    for which in (CAKF_FILTER, CAKF_SMOOTH):
        m, v = h.get(k, which)
        ok &= bool(np.all(np.isfinite(m)) and np.all(np.isfinite(v)))
        ok &= bool(np.all(v <= np.repeat(np.diag(Sinf), wl.n_space) * (1 + 1e-5) + 1e-3))
        ok &= bool(np.all(v >= -1e-3 * np.repeat(np.diag(Sinf), wl.n_space)))
st = [h.get_stats(k) for k in range(T + 1)]
print(json.dumps({"workload": "cfg4", "T": T, "D": wl.D, "N": wl.n_obs(1), "ms_per_pass": ms,
                  "time_steps_per_s": T / (ms / 1e3), "finite_and_bounded": ok,
                  "ranks": [s["rank_out"] for s in st], "cull": h.cull_stats(),
                  "phase_ms": {c: round(prof[c][0], 1) for c in prof}, "wall_s": time.time() - t0}))
