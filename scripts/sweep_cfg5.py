"""BASELINE.json configs[4] (cfg5): policy / iteration / rank sweep at cfg3's shape (D = 231,360, T = 48):
{CG, random, coordinate} actions x {16, 32, 64, 128, 256} iterations per step x rank cap {128, 256, 512, 1024}
(App. C.3.1).  Per run: time-steps/s of the full filter + smoother pass
(one warm-up pass, one timed pass, no per-launch events) and the quality side of the trade-off on the held-out
test subgrid: RMSE of the smoother mean of f_0 against the noise-free synthetic field, and the mean marginal
predictive variance there.  One JSON line per run to --out (written as it goes).

    python scripts/sweep_cfg5.py [--out gpurun_out/r2_cfg5_sweep.jsonl] [--policies cg,random,coord]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_08971_b200 import CAKF_SMOOTH, runner  # noqa: E402
from synth import make_workload  # noqa: E402
from synth.workloads import farthest_point_order, temperature_field  # noqa: E402


def quality(h, wl):
    X = wl.coords[wl.test_idx]
    lat, lon = np.arcsin(np.clip(X[:, 2], -1, 1)), np.arctan2(X[:, 1], X[:, 0])
    se, var = [], []
    for k in range(1, wl.T + 1):
        m, v = h.get(k, CAKF_SMOOTH)
        se.append((m[wl.test_idx].astype(np.float64) - temperature_field(wl.times[k - 1], lat, lon)) ** 2)
        var.append(v[wl.test_idx].astype(np.float64))
    return float(np.sqrt(np.mean(np.concatenate(se)))), float(np.mean(np.concatenate(var)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/r2_cfg5_sweep.jsonl")
    ap.add_argument("--policies", default="cg,random,coord")
    ap.add_argument("--iters", default="16,32,64,128,256")
    ap.add_argument("--ranks", default="128,256,512,1024")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    args = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()   # non-default: the handle runs on it and the events bracket its work
    torch.cuda.set_stream(stream)
    with open(args.out, "a") as fo:
        for policy in args.policies.split(","):
            for iters in (int(x) for x in args.iters.split(",")):
                for rank in (int(x) for x in args.ranks.split(",")):
                    rec = {"workload": "cfg3", "policy": policy, "max_iter": iters, "max_rank": rank, "dtype": args.dtype}
                    try:
                        wl = make_workload("cfg3", policy=policy, max_iter=iters, max_rank=rank)
                        if policy == "coord":
                            o = farthest_point_order(wl.coords[wl.obs_idx[0]], iters)
                            wl.coord_order = [o.copy() for _ in range(wl.T)]
                        trans, _ = runner.transitions(wl)
                        h = runner.make_handle(wl, args.dtype, stream=stream.cuda_stream)
                        inputs = runner.stage_inputs(wl, args.dtype)
                        runner.run(h, trans, inputs)
                        torch.cuda.synchronize()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        runner.run(h, trans, inputs)
                        e1.record(stream)
                        torch.cuda.synchronize()
                        ms = e0.elapsed_time(e1)
                        rmse, mvar = quality(h, wl)
                        rec.update({"time_steps_per_s": wl.T / (ms / 1e3), "ms_per_pass": round(ms, 1),
                                    "test_rmse_smoother": rmse, "test_mean_var_smoother": mvar,
                                    "rank_out_last": h.get_stats(wl.T)["rank_out"]})
                        h.destroy()
                        del inputs
                    except Exception as e:   # record and go on (e.g. memory at the largest points)
                        rec["error"] = repr(e)[:300]
                    torch.cuda.empty_cache()
                    print(json.dumps(rec), flush=True)
                    fo.write(json.dumps(rec) + "\n")
                    fo.flush()


if __name__ == "__main__":
    main()
