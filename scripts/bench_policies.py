"""cfg5-style policy sweep on cfg3: time-steps/s of the full filter + smoother pass
for CG, random and coordinate actions, sequential (one K1 per action) and block-executed
(block_actions = b: one multi-RHS K2 per b actions).  One warm-up pass, one timed pass each."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2405_08971_b200 import runner
from synth import make_workload
from synth.workloads import farthest_point_order

res = []
for policy, b in [("cg", 1), ("random", 1), ("random", 16), ("random", 64), ("coord", 1), ("coord", 16)]:
    wl = make_workload("cfg3", policy=policy, block_actions=b)
    if policy == "coord":
        o = farthest_point_order(wl.coords[wl.obs_idx[0]], wl.max_iter)
        wl.coord_order = [o.copy() for _ in range(wl.T)]
    trans, _ = runner.transitions(wl)
    h = runner.make_handle(wl, "f32")
    inputs = runner.stage_inputs(wl, "f32")
    runner.run(h, trans, inputs)
    torch.cuda.synchronize()
    h.profile(True)
    h.profile_read(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    runner.run(h, trans, inputs)
    e1.record()
    torch.cuda.synchronize()
    prof = h.profile_read(reset=True)
    ms = e0.elapsed_time(e1)
    res.append({"policy": policy, "block_actions": b, "max_iter": wl.max_iter, "max_rank": wl.max_rank,
                "time_steps_per_s": wl.T / (ms / 1e3), "ms_per_pass": round(ms, 1),
                "k1_or_block_k2_ms": round(prof["k1_matvec"][0], 1), "stages_ms": round(prof["loop_stages"][0], 1)})
    print(json.dumps(res[-1]), flush=True)
    h.destroy()
json.dump({"workload": "cfg3", "dtype": "f32", "results": res}, open("gpurun_out/policies.json", "w"), indent=1)
