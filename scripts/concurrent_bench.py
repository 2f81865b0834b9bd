"""P independent cfg3 problems per GPU, one handle + one stream + one host thread each.

The filter's truncation eigensolver (cuSOLVER Dsyevd at c = 576, ~5 ms of tridiagonalisation
latency per call with the GPU mostly idle) and the CG stage kernels (latency-bound grid-wide
reductions) leave SMs idle inside one pass; a second independent problem on its own stream fills
them with its K1 launches.  This measures the aggregate throughput (time-steps/s over all P
problems) with CUDA events: one event on the main stream that every problem stream waits on, and
one after the main stream has waited on every problem stream.

Usage: python scripts/concurrent_bench.py [--P 2] [--steps 2] [--warmup 3] [--config cfg3]
Prints one JSON line.  Each handle is an independent problem (same synthetic workload), so P
problems = P x T time steps per pass.
"""
import argparse
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    args = ap.parse_args()
    import torch

    from paper_2405_08971_b200 import runner
    from synth import make_workload

    torch.cuda.set_device(0)
    wl = make_workload(args.config)
    trans, _ = runner.transitions(wl)
    main_st = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in range(args.P)]
    handles = [runner.make_handle(wl, "f32", stream=s.cuda_stream) for s in streams]
    inputs = [runner.stage_inputs(wl, "f32") for _ in range(args.P)]

    def drive(p, n):
        for _ in range(n):
            runner.run(handles[p], trans, inputs[p], smooth=True)

    def run_all(n):
        ths = [threading.Thread(target=drive, args=(p, n)) for p in range(args.P)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()

    run_all(args.warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main_st)
    for s in streams:
        s.wait_event(e0)
    run_all(args.steps)
    for s in streams:
        ev = torch.cuda.Event()
        ev.record(s)
        main_st.wait_event(ev)
    e1.record(main_st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ts = args.P * args.steps * wl.T
    print(json.dumps({"what": "P independent filter+smoother passes per GPU, one stream + host thread each",
                      "config": args.config, "P": args.P, "steps": args.steps, "warmup": args.warmup,
                      "ms_total": ms, "time_steps_per_s": ts / (ms / 1e3),
                      "ms_per_pass_per_problem": ms / args.steps}))


if __name__ == "__main__":
    main()
